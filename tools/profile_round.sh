#!/bin/bash
# Round profile: launch list of the bench command + full captures of the
# dominant kernels.  Run under gpurun; outputs in gpurun_out/ (summarised into
# profiles/ by tools/summarize_profiles.py).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench_stdout.txt 2>&1
# dominant kernels of the step: tcgen05 GEMM (output-layer dX / dW / fwd) and
# the grouped SIMT GEMM of the recurrent levels
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 6 -c 3 \
    -o gpurun_out/full_tc python tools/profile_step.py --steps 1 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_group_kernel -s 120 -c 2 \
    -o gpurun_out/full_simt python tools/profile_step.py --steps 1 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:cell_ -s 40 -c 2 \
    -o gpurun_out/full_cell python tools/profile_step.py --steps 1 --warmup 1 > /dev/null 2>&1
