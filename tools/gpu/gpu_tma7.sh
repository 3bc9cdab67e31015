#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tma_pers_epi.txt; : > $out
for d in 1024 1025 1032; do
echo "== timeline $d" >> $out
TMA_PROF_EPI=1 TMA_PROF=1 DG_TMA_DBG=$d timeout 60 ./tools/tma_bench t 2>&1 | grep -A10 "prof fwd 2176" | grep -E "epi|time|mma acc" >> $out
done
