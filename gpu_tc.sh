#!/bin/bash
mkdir -p gpurun_out
timeout 300 ./tools/gemm_bench > gpurun_out/gemm_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/gemm_bench.txt
