#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize.py); summaries to gpurun_out/san_*.txt
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for w in ptb tiny tree tagger gru ptb_big; do
    timeout 900 $S --tool $tool --print-limit 20 python tools/sanitize.py $w > gpurun_out/san_${tool}_${w}.txt 2>&1
    echo "rc=$?" >> gpurun_out/san_${tool}_${w}.txt
  done
done
grep -H -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|Error|error" gpurun_out/san_*.txt | grep -v "^.*: *$" > gpurun_out/san_summary.txt
