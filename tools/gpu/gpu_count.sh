#!/bin/bash
mkdir -p gpurun_out
python tools/count_launches.py > gpurun_out/count.txt 2>&1
DG_AFFCELL=0 python tools/count_launches.py >> gpurun_out/count.txt 2>&1
