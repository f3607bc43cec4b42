set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2x_prof.json > gpurun_out/r2x_bench.log 2>&1
BBOT_TAILT_ROWS=65536 timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2x_prof_tt.json > gpurun_out/r2x_bench_tt.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"LapView" --launch-count 6 --set full --import-source on --clock-control none -o gpurun_out/r2x_full python scripts/profile_apply.py --config C4 > gpurun_out/r2x_ncu.log 2>&1
timeout 2100 python scripts/ipm_run.py --config C3 > gpurun_out/r2x_ipm_C3.log 2>&1
