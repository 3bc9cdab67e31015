#!/bin/bash
mkdir -p gpurun_out
for c in ${CONFIGS:-tree tagger}; do
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
  --log-file gpurun_out/step_launches_$c.csv python tools/profile_step.py --config $c --steps 1 --warmup 2 > gpurun_out/step_launches_$c.log 2>&1
done
