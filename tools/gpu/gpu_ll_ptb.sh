#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum --clock-control none --csv \
  --log-file gpurun_out/step_launches_ptb.csv python tools/profile_step.py --config ptb64 --steps 1 --warmup 1 > /dev/null 2>&1
