#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tma_pers_split_dbg.txt; : > $out
DG_TMA_PERS_SPLIT=1 TMA_PROF=1 TMA_PROF_RED=1 DG_TMA_DBG=1024 timeout 60 ./tools/tma_bench t 2>&1 | grep -A12 "prof dW 256" | grep -E "split reduce|epi acc_full" >> $out
