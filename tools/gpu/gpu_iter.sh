#!/bin/bash
# iteration check: recurrence-heavy GPU tests, timeline, headline bench
mkdir -p gpurun_out
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1200 python -m pytest tests/test_gpu_initial_state.py tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_semantics.py -m gpu -q -x --timeout 600 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
DG_RNN_TRACE=2 timeout 300 python tools/rnn_trace.py 2>&1 | grep -v "^\[rnn\]" > gpurun_out/rnn_trace.txt
./tools/gpu/gpu_ab.sh "DG_X=1"
