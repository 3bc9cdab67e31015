#!/bin/bash
mkdir -p gpurun_out
./tools/launch_probe > gpurun_out/launch_probe.txt 2>&1
DG_PLAN_TIMING=2 timeout 300 python tools/host_phases.py tagger > gpurun_out/op_timing_tagger.txt 2>&1
DG_PLAN_TIMING=1 timeout 300 python tools/host_phases.py tagger > gpurun_out/plan_timing_tagger.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
