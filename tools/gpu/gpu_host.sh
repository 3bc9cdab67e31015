#!/bin/bash
# host-side phase timings (real and dry-run) + bench line
mkdir -p gpurun_out
rm -f gpurun_out/host_real.txt gpurun_out/host_dry.txt
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-budget 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ptb64 tree tagger ptb16; do
  timeout 300 python tools/host_phases.py $c >> gpurun_out/host_real.txt 2>&1
  DG_DRYRUN=1 timeout 300 python tools/host_phases.py $c >> gpurun_out/host_dry.txt 2>&1
done
