#!/bin/bash
# tests + headline bench at the driver's K/W and the default + round profile
mkdir -p gpurun_out
./tools/gpu/gpu_tests.sh
timeout 600 python bench.py --steps 20 --warmup 5 --only --no-cpu > gpurun_out/bench_20.log 2>&1; echo "rc=$?" >> gpurun_out/bench_20.log
timeout 600 python bench.py --steps 10 --warmup 3 --only --no-cpu > gpurun_out/bench_10.log 2>&1; echo "rc=$?" >> gpurun_out/bench_10.log
timeout 300 python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
./tools/profile_round.sh
