#!/bin/bash
# A/B of the GPU-only tail knobs on the bench workload (C2): prints ms/step and krylov ms per setting
for cfg in "4096 16384 0" "4096 16384 1" "4096 0 0" "4096 0 1" "1024 0 1" "8192 16384 8" "0 0 1"; do
  set -- $cfg
  out=$(BBOT_TAIL_ROWS=$1 BBOT_TAILT_ROWS=$2 BBOT_TAIL_CL=$3 timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-profile 2>&1 | tail -1)
  python -c "
import json,sys
j=json.loads(sys.argv[1]); print('TAIL_ROWS=$1 TAILT_ROWS=$2 CL=$3', round(j['ms_per_step'],1), j['timing'])" "$out" || echo "$cfg failed: $out"
done
