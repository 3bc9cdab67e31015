#!/bin/bash
# strict parity report (all GPU tests, no -x), recurrence timeline, CUDA-graph A/B
mkdir -p gpurun_out
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
DG_RNN_TRACE=2 timeout 300 python tools/rnn_trace.py > gpurun_out/rnn_trace.txt 2>&1
./tools/gpu/gpu_ab.sh "DG_X=1" "DG_CUDA_GRAPH=1" "DG_X=1" "DG_CUDA_GRAPH=1"
for c in tagger tree; do
  for v in "DG_X=1" "DG_CUDA_GRAPH=1"; do
    echo "== $c $v" >> gpurun_out/ab.txt
    env $v timeout 300 python bench.py --steps 20 --warmup 5 --config $c --only --no-cpu 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/ab.txt
  done
done
