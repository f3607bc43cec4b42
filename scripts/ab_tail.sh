#!/bin/bash
# A/B of the k_tailA block size on the C4 headline step
for v in 1024 512 256; do
  out=$(BBOT_TAILA_BS=$v timeout 500 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --ipm-config '' --side-config '' 2>&1 | grep '^{' | tail -1)
  python -c "
import json,sys
j=json.loads(sys.argv[1]); k={r['kernel'].split('(')[0].replace('void bbot::','').replace('bbot::',''):round(r['ms'],1) for r in j['kernels'][:6]}
print('tail bs $v', round(j['ms_per_step'],1), j['timing']['t_krylov_ms'], k)" "$out" || echo "$v failed"
done
