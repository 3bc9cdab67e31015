#!/bin/bash
mkdir -p gpurun_out
DG_SAN_EARLY=1 timeout 300 python tools/sanitize.py tagger > gpurun_out/san7_plain.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 DG_SAN_EARLY=1 timeout 300 python tools/sanitize.py tagger > gpurun_out/san7_blocking.txt 2>&1
DG_SAN_EARLY=1 timeout 1200 compute-sanitizer --tool racecheck --print-limit 3 python tools/sanitize.py tagger > gpurun_out/san7_race.txt 2>&1
DG_SAN_EARLY=1 timeout 1200 compute-sanitizer --tool racecheck --print-limit 3 python tools/sanitize.py ptb > gpurun_out/san7_race_ptb.txt 2>&1
