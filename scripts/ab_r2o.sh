set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_harmonic.py tests/test_gpu_hss.py tests/test_gpu_slabs.py -x -q -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo rc=$? >> gpurun_out/r2o_tests.log
for v in main minb6 head; do
  if [ $v = main ]; then L=paper_2209_00315_b200/libbbot.so; else L=paper_2209_00315_b200/variants/libbbot_$v.so; fi
  BBOT_LIB=$PWD/$L timeout 600 python bench.py --steps 3 --warmup 2 --side-config '' --no-cpu-baseline --ipm-config '' --e2e-steps 1 --profile-out gpurun_out/r2o_prof_$v.json > gpurun_out/r2o_bench_$v.log 2>&1
done
