#!/bin/bash
# Round profile: launch list of the bench command + full captures of the
# dominant kernels (one ncu --set full capture per kernel class).  Run under
# gpurun; outputs in gpurun_out/ (summarised into profiles/ by
# tools/summarize_profiles.py <tag>, which also writes profiles/traffic.json).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --only > gpurun_out/ncu_bench_stdout.txt 2>&1
P="python tools/profile_step.py --steps 1 --warmup 1"
full() {  # name, kernel regex, skip, count
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c "$4" \
      -o "gpurun_out/$1" $P > "gpurun_out/$1.log" 2>&1
}
full full_rnnf rnn_fwd_cl 2 2
full full_rnnb rnn_bwd_cl 2 2
full full_tma tma_gemm_kernel 8 6
full full_pers tma_gemm_pers 1 1
full full_row row_reg_kernel 2 2
full full_bw "scatter_rows|gather_rows|colsum_partial|update_dense|update_rows" 5 10
