#!/bin/bash
# workspace split-K vs cluster split-K on the PTB GEMM shapes, forced split factors
mkdir -p gpurun_out
out=gpurun_out/tma_gsplit.txt; : > $out
timeout 120 ./tools/tma_bench 2>&1 | grep -E "check|time" >> $out; echo "rc=$?" >> $out
echo "== cluster (TMA_NO_WS)" >> $out
TMA_NO_WS=1 timeout 120 ./tools/tma_bench t 2>&1 | grep -E "^time" >> $out
for S in 1 2 3 4 5 6 8; do
  echo "== forced S=$S" >> $out
  DG_TMA_DBG=$((S << 16)) timeout 120 ./tools/tma_bench t 2>&1 | grep -E "^time" >> $out
done
if [ -n "$PYT" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider $PYT > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tma.log
fi
