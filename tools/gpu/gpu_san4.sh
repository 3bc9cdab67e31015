#!/bin/bash
mkdir -p gpurun_out
DG_SAN_DUMP=1 timeout 300 python tools/sanitize.py tagger > gpurun_out/san4_plain.txt 2>&1
DG_SAN_DUMP=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python tools/sanitize.py tagger > gpurun_out/san4_race.txt 2>&1
