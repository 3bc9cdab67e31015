#!/bin/bash
mkdir -p gpurun_out
python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_group_kernel -s 60 -c 1 -o gpurun_out/prof_dx python tools/profile_step.py --steps 1 --warmup 1 > gpurun_out/ncu_full_stdout.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
