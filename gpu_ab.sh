#!/bin/bash
# A/B of env knobs on the headline bench (device + e2e), one line each
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for v in "DG_TMA_AT=1" "DG_TMA_AT=0" "DG_TMA_AT=1" "DG_TMA_AT=0"; do
  echo "== $v" >> $out
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --only 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_launch']*1e3,1) for k,v in d['rooflines'].items() if k.startswith('gemm')})
" >> $out
done
