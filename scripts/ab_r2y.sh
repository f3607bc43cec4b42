set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
BBOT_NAGG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bb_apply or direction or amg or kcycle" > gpurun_out/r2y_tests_nagg.log 2>&1; echo rc=$? >> gpurun_out/r2y_tests_nagg.log
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2y_prof.json > gpurun_out/r2y_bench.log 2>&1
BBOT_NAGG=1 timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2y_prof_nagg.json > gpurun_out/r2y_bench_nagg.log 2>&1
