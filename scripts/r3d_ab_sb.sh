set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3d_build.log 2>&1
timeout 300 python scripts/ab_lap_sb.py --config C2 > gpurun_out/r3d_ab_C2.log 2>&1
timeout 900 python scripts/ab_lap_sb.py --config C4 > gpurun_out/r3d_ab_C4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_smoke.py -q -x > gpurun_out/r3d_tests.log 2>&1; echo rc=$? >> gpurun_out/r3d_tests.log
