#!/bin/bash
# A/B of the reduction block budget (BBOT_RED_BLOCKS_PER_SM) on the C4 headline and the C2 side step
for v in 64 128 256; do
  out=$(BBOT_RED_BLOCKS_PER_SM=$v timeout 500 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --ipm-config '' 2>&1 | grep '^{' | tail -1)
  python -c "
import json,sys
j=json.loads(sys.argv[1]); k={r['kernel'].split('<')[0].replace('void bbot::','').replace('bbot::',''):round(r['ms'],1) for r in j['kernels'][:8]}
print('blocks/SM $v', round(j['ms_per_step'],1), 'C2', round(j['side_point']['ms_per_step'],1), k)" "$out" || echo "$v failed"
done
