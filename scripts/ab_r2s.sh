set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
python scripts/diag_exec_modes.py C2 > gpurun_out/r2s_diag.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2s_prof.json > gpurun_out/r2s_bench.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py tests/test_gpu_smoke.py tests/test_gpu_edge.py -q -p no:cacheprovider > gpurun_out/r2s_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_tests.log
