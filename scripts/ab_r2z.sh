set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2z_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2z_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2z_bench.log 2>&1; echo rc=$? >> gpurun_out/r2z_bench.log
