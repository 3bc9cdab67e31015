#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/e2e_var.txt
for i in 1 2 3; do
  for v in "DG_X=1" "DG_CUDA_GRAPH=0" "DG_PLAN_CACHE=0"; do
    env $v timeout 300 python bench.py --steps 20 --warmup 5 --only --no-cpu 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v', round(d['value']), round(e['value']), round(e['ms_per_step'],3), e['step_wall_ms'])" >> gpurun_out/e2e_var.txt
  done
done
