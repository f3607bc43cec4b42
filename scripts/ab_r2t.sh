set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1
BBOT_SELL_SPLIT=1 timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2t_prof_split.json > gpurun_out/r2t_bench_split.log 2>&1
BBOT_EAGER=1 timeout 300 python scripts/profile_step.py --config C4 --warm 0 > gpurun_out/r2t_pstep.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_tailA|k_up_dot|k_down|k_up|k_pcg_pq|k_restrict|k_pcg_xr" --launch-count 20 -o gpurun_out/r2t_full python scripts/profile_step.py --config C4 --warm 0 > gpurun_out/r2t_ncu.log 2>&1
