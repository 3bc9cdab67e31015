#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tma_pers_split_dbg.txt; : > $out
timeout 120 ./tools/tma_bench 2>&1 | grep -E "check|time" >> $out
echo "== DG_TMA_PERS_SPLIT=0" >> $out
DG_TMA_PERS_SPLIT=0 timeout 60 ./tools/tma_bench t 2>&1 | grep -E "^time" >> $out
echo "== DG_TMA_TSTORE=0" >> $out
DG_TMA_TSTORE=0 timeout 60 ./tools/tma_bench t 2>&1 | grep -E "^time  dW 256" >> $out
