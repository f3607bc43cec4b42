set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hss.py tests/test_gpu_slabs.py -q -p no:cacheprovider -x > gpurun_out/r3b_tests.log 2>&1; echo rc=$? >> gpurun_out/r3b_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r3b_prof.json > gpurun_out/r3b_bench.log 2>&1
BBOT_DOWN_SL=0 timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r3b_prof_nosl.json > gpurun_out/r3b_bench_nosl.log 2>&1
