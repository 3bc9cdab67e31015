#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_semantics.py -m gpu -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
./tools/gpu/gpu_ab.sh "DG_X=1" "DG_X=2"
