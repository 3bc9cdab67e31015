#!/bin/bash
mkdir -p gpurun_out
DG_RNN_TRACE=2 timeout 200 python tools/rnn_trace.py > gpurun_out/rnn_trace.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rnn_fwd_cl -s 2 -c 1 -o gpurun_out/rnn_fwd python tools/profile_step.py --steps 1 --warmup 1 > gpurun_out/ncu1.txt 2>&1
