#!/bin/bash
./tools/gpu/gpu_iter.sh
cp gpurun_out/ab.txt gpurun_out/ab_iter.txt
./tools/gpu/gpu_ab_src.sh A cur
