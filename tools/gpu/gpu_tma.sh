#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tma_ep3.txt; : > $out
timeout 120 ./tools/tma_bench 2>&1 | grep -v "with lo" >> $out; echo "rc=$?" >> $out
for d in 1024 7168; do
echo "== $d" >> $out
TMA_PROF=1 DG_TMA_DBG=$d timeout 120 ./tools/tma_bench t 2>&1 | grep -E "phases|time" >> $out
done
