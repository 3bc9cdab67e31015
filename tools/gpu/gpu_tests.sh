#!/bin/bash
# GPU tests only (optionally a -k filter as $1)
mkdir -p gpurun_out
if [ -n "$1" ]; then K="-k $1"; else K=""; fi
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider $K -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
