#!/bin/bash
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for w in ptb ptb_big; do
  timeout 900 $S --tool racecheck --print-limit 20 python tools/sanitize.py $w > gpurun_out/san_racecheck_${w}.txt 2>&1
  echo "rc=$?" >> gpurun_out/san_racecheck_${w}.txt
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_san.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_san.log
