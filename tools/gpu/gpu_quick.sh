#!/bin/bash
# GPU parity tests + headline bench (device, e2e, per-class)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --only 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4)); print({k: round(v['ms_per_launch']*1e3,1) for k,v in d['rooflines'].items()}); print(d['kernel_share'])
" > gpurun_out/quick.txt
