set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3b_build.log 2>&1
timeout 600 python scripts/sweep_inner.py --config C4 --eps 1e-3,3e-3,1e-2,5e-2 > gpurun_out/r3b_sweep_C4.log 2>&1
timeout 300 python scripts/sweep_inner.py --config C2 --eps 1e-3,3e-3,1e-2,5e-2 --omega 0.6667,0.8 > gpurun_out/r3b_sweep_C2.log 2>&1
timeout 300 python scripts/sweep_inner.py --config C2 --newton 5 --eps 1e-3,3e-3,1e-2,5e-2 > gpurun_out/r3b_sweep_C2n5.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"k_up_dot|k_pcg_pq|k_down|k_pcg_xr|k_tailA|k_restrict|k_up<|k_spmv|k_post|k_resid" --launch-count 24 --set full --import-source on --clock-control none -o gpurun_out/r3b_full_C4 python scripts/profile_apply.py --config C4 > gpurun_out/r3b_ncu_full.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3b_launches_C4.csv python scripts/profile_step.py --config C4 > gpurun_out/r3b_launches.log 2>&1
ls -la gpurun_out
