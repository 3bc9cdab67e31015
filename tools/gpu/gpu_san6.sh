#!/bin/bash
mkdir -p gpurun_out
python tools/replay_probe.py > gpurun_out/san6.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/replay_probe.py >> gpurun_out/san6.txt 2>&1
