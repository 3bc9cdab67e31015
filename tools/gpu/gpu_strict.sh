#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --config tagger --only --no-cpu > gpurun_out/bench_tagger.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --only --no-cpu > gpurun_out/bench_20.log 2>&1
