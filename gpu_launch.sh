#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 --warmup 1 > gpurun_out/ncu_stdout.txt 2>&1
