#!/bin/bash
mkdir -p gpurun_out
DG_SAN_NODES=1 timeout 300 python tools/sanitize.py tagger > gpurun_out/san5_plain.txt 2>&1
DG_SAN_NODES=1 timeout 1200 compute-sanitizer --tool racecheck --print-limit 3 python tools/sanitize.py tagger > gpurun_out/san5_race.txt 2>&1
DG_SAN_NODES=1 DG_PLAN_CACHE=0 DG_SCHED_CACHE=0 timeout 1200 compute-sanitizer --tool racecheck --print-limit 3 python tools/sanitize.py tagger > gpurun_out/san5_race_nocache.txt 2>&1
