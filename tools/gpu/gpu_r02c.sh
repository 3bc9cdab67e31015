#!/bin/bash
mkdir -p gpurun_out
./tools/gpu/gpu_tests.sh
timeout 600 python bench.py --steps 20 --warmup 5 --only --no-cpu > gpurun_out/bench_20.log 2>&1; echo "rc=$?" >> gpurun_out/bench_20.log
DG_CUDA_GRAPH=0 timeout 600 python bench.py --steps 20 --warmup 5 --only --no-cpu > gpurun_out/bench_20_nograph.log 2>&1; echo "rc=$?" >> gpurun_out/bench_20_nograph.log
DG_PLAN_CACHE=0 timeout 600 python bench.py --steps 20 --warmup 5 --only --no-cpu > gpurun_out/bench_20_nocache.log 2>&1; echo "rc=$?" >> gpurun_out/bench_20_nocache.log
timeout 300 python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
