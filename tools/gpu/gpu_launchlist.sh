#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x --clock-control none --csv \
  --log-file gpurun_out/step_launches.csv python tools/profile_step.py --steps 1 --warmup 2 > gpurun_out/step_launches.log 2>&1
