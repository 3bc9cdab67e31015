#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/san3.txt
echo "== plain" >> gpurun_out/san3.txt; timeout 300 python tools/sanitize.py tagger >> gpurun_out/san3.txt 2>&1
for v in "DG_X=1" "DG_PDL=0" "DG_RNN=0" "DG_TC=0"; do
  echo "== racecheck $v" >> gpurun_out/san3.txt
  env $v timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python tools/sanitize.py tagger >> gpurun_out/san3.txt 2>&1
done
echo "== memcheck PDL on" >> gpurun_out/san3.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python tools/sanitize.py tagger >> gpurun_out/san3.txt 2>&1
