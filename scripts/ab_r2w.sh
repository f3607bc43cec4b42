set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --side-config C2 --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2w_prof.json > gpurun_out/r2w_bench.log 2>&1
BBOT_EAGER=1 timeout 300 python scripts/profile_apply.py --config C4 > gpurun_out/r2w_papply.log 2>&1
BBOT_EAGER=1 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k regex:"LapView|SellView|k_restrict|k_pcg_xr" --launch-count 16 --set full --import-source on --clock-control none -o gpurun_out/r2w_full python scripts/profile_apply.py --config C4 > gpurun_out/r2w_ncu.log 2>&1
