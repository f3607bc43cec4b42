set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r4h_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r4h_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4h_smoke.log 2>&1; echo rc=$? >> gpurun_out/r4h_smoke.log
python bench.py > gpurun_out/r4h_bench.log 2>&1; echo rc=$? >> gpurun_out/r4h_bench.log
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"k_up_dot|k_pcg_pq|k_down_sb|k_pcg_xr|k_tailA|k_up_res|k_down_nx" --launch-count 16 --set full --import-source on --clock-control none -o gpurun_out/r4h_full_C4_A python scripts/profile_apply.py --config C4 > gpurun_out/r4h_ncu_full.log 2>&1
BBOT_EAGER=1 timeout 1800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4h_launches_C4.csv python scripts/profile_step.py --config C4 > gpurun_out/r4h_launches.log 2>&1
tail -3 gpurun_out/r4h_gpu_tests.log
