#!/bin/bash
# full GPU tests + bench all configs
mkdir -p gpurun_out
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_all.log 2>&1
