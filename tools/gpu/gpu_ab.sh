#!/bin/bash
# A/B of env knobs on the headline bench (device + e2e), one line each: ./gpu_ab.sh "ENV=a" "ENV=b" ...
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
for v in "$@"; do
  echo "== $v" >> $out
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --only 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_launch']*1e3,1) for k,v in d['rooflines'].items()})
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
" >> $out
done
