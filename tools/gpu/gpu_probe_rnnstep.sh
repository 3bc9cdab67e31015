#!/bin/bash
mkdir -p gpurun_out
./tools/rnn_step_probe > gpurun_out/rnn_step_probe.txt 2>&1
