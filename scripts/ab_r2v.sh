set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -p no:cacheprovider -x > gpurun_out/r2v_tests.log 2>&1; echo rc=$? >> gpurun_out/r2v_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2v_prof.json > gpurun_out/r2v_bench.log 2>&1
BBOT_DOWN_SPLIT=1 timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2v_prof_ds.json > gpurun_out/r2v_bench_ds.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_up_dot|k_pcg_pq|k_gm_orth|k_gm_dots" --launch-skip 300 --launch-count 16 -o gpurun_out/r2v_full python scripts/profile_step.py --config C4 --warm 0 > gpurun_out/r2v_ncu.log 2>&1
