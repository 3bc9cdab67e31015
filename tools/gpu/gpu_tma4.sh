#!/bin/bash
# automatic cluster / workspace split-K choice on the PTB GEMM shapes + parity + A/B bench
mkdir -p gpurun_out
out=gpurun_out/tma_gsplit2.txt; : > $out
timeout 120 ./tools/tma_bench 2>&1 | grep -E "check|time" >> $out; echo "rc=$?" >> $out
echo "== forced workspace split (bit 21)" >> $out
DG_TMA_DBG=0x200000 timeout 120 ./tools/tma_bench t 2>&1 | grep -E "^time" >> $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tma.log
for i in 1 2; do
  DG_TMA_GSPLIT=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --only >> gpurun_out/ab_gsplit.txt 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --only >> gpurun_out/ab_gsplit.txt 2>&1
done
