#!/bin/bash
# A/B of GPU-only tuning knobs on the C4 headline step: prints ms/step per setting
for cfg in "BBOT_TAIL_CL=1" "BBOT_TAIL_CL=2" "BBOT_TAIL_CL=4" "BBOT_UP_SPLIT=1"; do
  out=$(env $cfg timeout 400 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-profile --side-config '' --ipm-config '' 2>&1 | tail -1)
  python -c "
import json,sys
j=json.loads(sys.argv[1]); print('$cfg', round(j['ms_per_step'],1), j['timing'], j['solve']['inner_A_its_max'])" "$out" || echo "$cfg failed: $out"
done
