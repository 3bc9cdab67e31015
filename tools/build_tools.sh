#!/bin/bash
# diagnostic binaries (not part of the product build)
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/gemm_bench.cu paper_1701_03980_b200/csrc/gemm.cu paper_1701_03980_b200/csrc/tcgemm.cu paper_1701_03980_b200/csrc/kernels.cu -o tools/gemm_bench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/tma_bench.cu paper_1701_03980_b200/csrc/tmagemm.cu paper_1701_03980_b200/csrc/tcgemm.cu paper_1701_03980_b200/csrc/kernels.cu -o tools/tma_bench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/umma_probe.cu -o tools/umma_probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/launch_probe.cu -o tools/launch_probe
