#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/ab_window.txt; : > $out
for i in 1 2; do
for m in 1 3; do
  echo "W$m" >> $out; DG_WINDOW=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --only 2>&1 | grep '^{' >> $out
done
done
