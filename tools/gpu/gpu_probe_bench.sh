#!/bin/bash
mkdir -p gpurun_out
DG_PLAN_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --only --no-cpu > gpurun_out/pb.log 2> gpurun_out/pb_timing.txt
