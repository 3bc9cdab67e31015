#!/bin/bash
# persistent split-K work units: correctness + timing vs the cluster / workspace kernels
mkdir -p gpurun_out
out=gpurun_out/tma_pers_split.txt; : > $out
for mn in 4 2; do
  echo "== DG_TMA_PERS_MIN=$mn" >> $out
  DG_TMA_PERS_MIN=$mn timeout 120 ./tools/tma_bench 2>&1 | grep -E "check|time" >> $out
done
echo "== DG_TMA_PERS=0" >> $out
DG_TMA_PERS=0 timeout 120 ./tools/tma_bench t 2>&1 | grep -E "^time" >> $out
if [ -n "$PYT" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tma.log
rm -f gpurun_out/ab_pers2.txt
for i in 1 2; do
  DG_TMA_PERS_SPLIT=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --only >> gpurun_out/ab_pers2.txt 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --only >> gpurun_out/ab_pers2.txt 2>&1
done
fi
