set -x
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"k_up_dot|k_pcg_pq|k_down_sb|k_pcg_xr|k_tailA|k_up_res|k_down_nx" --launch-count 16 --set full --import-source on --clock-control none -o gpurun_out/r4l_full_C4_A python scripts/profile_apply.py --config C4 > gpurun_out/r4l_ncu_full.log 2>&1
BBOT_EAGER=1 timeout 1800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4l_launches_C4.csv python scripts/profile_step.py --config C4 > gpurun_out/r4l_launches.log 2>&1
