#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/sanitize.py > gpurun_out/san_plain.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py > gpurun_out/san_$t.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_$t.txt
done
