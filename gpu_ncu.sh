#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 7 -c 1 -o gpurun_out/tc_fwd ./tools/gemm_bench > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 30 -c 1 -o gpurun_out/tc_dx ./tools/gemm_bench > /dev/null 2>&1
