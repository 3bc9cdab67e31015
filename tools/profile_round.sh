#!/bin/bash
# Round profile: launch list of the bench command + full captures of the
# dominant kernels.  Run under gpurun; outputs in gpurun_out/ (summarised into
# profiles/ by tools/summarize_profiles.py).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --only > gpurun_out/ncu_bench_stdout.txt 2>&1
P="python tools/profile_step.py --steps 1 --warmup 1"
# TMA tcgen05 GEMMs (output layer fwd / dX / dW), persistent LSTM kernels, pnls
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_gemm_kernel -s 8 -c 4 \
    -o gpurun_out/full_tma $P > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rnn_ -s 2 -c 4 \
    -o gpurun_out/full_rnn $P > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"row_reg_kernel|row_kernel" -s 2 -c 2 \
    -o gpurun_out/full_row $P > /dev/null 2>&1
