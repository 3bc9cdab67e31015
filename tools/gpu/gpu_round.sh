#!/bin/bash
# round evidence: GPU tests + smoke, full default bench line (all configs, CPU baseline), reference arm,
# launch list + full captures (tools/profile_round.sh), per-config step launch lists
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
./tools/profile_round.sh
CONFIGS="tree tagger" ./tools/gpu/gpu_launchlist2.sh
