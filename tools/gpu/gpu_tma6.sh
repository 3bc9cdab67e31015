#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tma_pers_dbg.txt; : > $out
timeout 60 ./tools/tma_bench 2>&1 | grep -E "check fwd" >> $out
for d in 0 2 8 10; do
  echo "== DG_TMA_DBG=$d" >> $out
  DG_TMA_DBG=$d timeout 60 ./tools/tma_bench t 2>&1 | grep -E "^time  fwd" >> $out
done
echo "== DG_TMA_TSTORE=0" >> $out
DG_TMA_TSTORE=0 timeout 60 ./tools/tma_bench t 2>&1 | grep -E "^time  fwd" >> $out
echo "== timeline" >> $out
TMA_PROF=1 DG_TMA_DBG=1024 timeout 60 ./tools/tma_bench t 2>&1 | grep -A8 "prof fwd 2176" | grep -E "epi|mma" >> $out
