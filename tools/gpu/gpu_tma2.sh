#!/bin/bash
# TMA GEMM breakdown on the PTB output-layer shapes: normal timing, then with
# DG_TMA_DBG bits removing one pipeline role at a time, then the CTA-0 timeline
mkdir -p gpurun_out
out=gpurun_out/tma_breakdown.txt; : > $out
timeout 120 ./tools/tma_bench 2>&1 | grep -E "check|time" >> $out; echo "rc=$?" >> $out
for d in 2 1 17 4 8 2048 0x20000 0x40000 0x80000; do
  echo "== DG_TMA_DBG=$d" >> $out
  DG_TMA_DBG=$d timeout 120 ./tools/tma_bench t 2>&1 | grep -E "^time" >> $out
done
echo "== timeline" >> $out
TMA_PROF=1 DG_TMA_DBG=1024 timeout 120 ./tools/tma_bench t 2>&1 | grep -vE "with lo" >> $out
