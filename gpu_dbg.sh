#!/bin/bash
mkdir -p gpurun_out
./tools/gemm_bench > gpurun_out/gemm_bench.txt 2>&1
python tools/debug_grads.py > gpurun_out/debug_grads.txt 2>&1
python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
