set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hss.py tests/test_gpu_smoke.py tests/test_gpu_edge.py -q -p no:cacheprovider -x > gpurun_out/r2u_tests.log 2>&1; echo rc=$? >> gpurun_out/r2u_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2u_prof.json > gpurun_out/r2u_bench.log 2>&1
BBOT_TAIL_SMEM=0 timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2u_prof_nosmem.json > gpurun_out/r2u_bench_nosmem.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"LapView|k_tailA|k_pcg_xr" --launch-skip 400 --launch-count 12 -o gpurun_out/r2u_full python scripts/profile_step.py --config C4 --warm 0 > gpurun_out/r2u_ncu.log 2>&1
