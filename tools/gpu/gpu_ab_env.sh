#!/bin/bash
# A/B of one environment switch on the headline bench: AB_ENV="VAR=value", AB_N alternations
mkdir -p gpurun_out
out=gpurun_out/ab_env.txt; : > $out
for i in $(seq 1 ${AB_N:-4}); do
  echo "A" >> $out; env $AB_ENV timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --only 2>&1 | grep '^{' >> $out
  echo "B" >> $out; timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --only 2>&1 | grep '^{' >> $out
done
