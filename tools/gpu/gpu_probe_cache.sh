#!/bin/bash
mkdir -p gpurun_out
for v in "" "DG_CUDA_GRAPH=0" "DG_PLAN_CACHE=0"; do
  echo "=== $v cycle4" >> gpurun_out/probe.txt
  env $v timeout 300 python tools/e2e_steps.py 24 4 >> gpurun_out/probe.txt 2>&1
done
echo "=== timing cycle4" >> gpurun_out/probe.txt
DG_PLAN_TIMING=1 timeout 300 python tools/e2e_steps.py 8 4 >> gpurun_out/probe.txt 2>&1
echo "=== default nocycle" >> gpurun_out/probe.txt
DG_PLAN_TIMING=1 timeout 300 python tools/e2e_steps.py 12 >> gpurun_out/probe.txt 2>&1
