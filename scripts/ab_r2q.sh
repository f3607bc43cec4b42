set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py tests/test_gpu_smoke.py -q -p no:cacheprovider > gpurun_out/r2q_tests.log 2>&1; echo rc=$? >> gpurun_out/r2q_tests.log
