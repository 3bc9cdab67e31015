#!/bin/bash
mkdir -p gpurun_out
DG_EARLY_DW_LOG=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --only > gpurun_out/edw_log.txt 2>&1
./tools/gpu/gpu_earlydw.sh
