#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tma_pers_min2.txt; : > $out
DG_TMA_PERS_MIN=2 timeout 120 ./tools/tma_bench 2>&1 | grep -E "check|time" >> $out
