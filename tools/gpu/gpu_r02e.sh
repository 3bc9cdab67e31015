#!/bin/bash
# strict parity report of the parity tests + recurrence step A/B probe
mkdir -p gpurun_out
rm -f gpurun_out/strict_report.tsv
./tools/rnn_step_probe > gpurun_out/rnn_step_probe.txt 2>&1
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
