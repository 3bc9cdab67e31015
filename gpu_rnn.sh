#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/rnn_trace.py > gpurun_out/rnn_trace.txt 2>&1; echo "rc=$?" >> gpurun_out/rnn_trace.txt
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
