set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3c_build.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"LapView|k_pcg_xr|k_tailA" --launch-count 10 --set full --import-source on --clock-control none -o gpurun_out/r3c_full_C4_A python scripts/profile_apply.py --config C4 > gpurun_out/r3c_ncu_full.log 2>&1
BBOT_EAGER=1 timeout 1800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3c_launches_C4.csv python scripts/profile_step.py --config C4 > gpurun_out/r3c_launches.log 2>&1
