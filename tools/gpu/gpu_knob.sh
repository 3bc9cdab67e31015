#!/bin/bash
# recurrence timeline per DG_RNN_KNOB value: ./gpu_knob.sh 0 1 4 ...
mkdir -p gpurun_out; : > gpurun_out/knob.txt
for k in "$@"; do
  echo "== knob $k" >> gpurun_out/knob.txt
  DG_RNN_KNOB=$k DG_RNN_TRACE=2 timeout 300 python tools/rnn_trace.py 2>&1 | grep -v "^\[rnn\]" >> gpurun_out/knob.txt
done
