#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tma_gemm_pers" -s 2 -c 1 -o gpurun_out/full_pers ./tools/tma_bench t > gpurun_out/full_pers.log 2>&1
echo "rc=$?" >> gpurun_out/full_pers.log
