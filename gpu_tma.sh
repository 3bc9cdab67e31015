#!/bin/bash
mkdir -p gpurun_out
timeout 200 ./tools/tma_bench > gpurun_out/tma_bench.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_gemm_kernel -s 8 -c 1 -o gpurun_out/tma_fwd ./tools/tma_bench > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_gemm_kernel -s 54 -c 1 -o gpurun_out/tma_dx ./tools/tma_bench > /dev/null 2>&1
