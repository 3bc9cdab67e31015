#!/bin/bash
mkdir -p gpurun_out
DG_GEMM_LOG=1 timeout 300 python tools/profile_step.py --steps 1 --warmup 1 > gpurun_out/gemmlog.txt 2>&1
