#!/bin/bash
mkdir -p gpurun_out
python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 --warmup 1 > gpurun_out/ncu_stdout.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
