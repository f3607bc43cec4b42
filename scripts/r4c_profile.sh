set -x
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"k_up_dot|k_pcg_pq|k_down_sb" --launch-count 6 --set full --import-source on --clock-control none -o gpurun_out/r4c_full_C4_A python scripts/profile_apply.py --config C4 > gpurun_out/r4c_ncu_full.log 2>&1
ncu -i gpurun_out/r4c_full_C4_A.ncu-rep --page raw --csv > gpurun_out/r4c_raw.csv 2>/dev/null
ncu -i gpurun_out/r4c_full_C4_A.ncu-rep --page details > gpurun_out/r4c_details.txt 2>/dev/null
