#!/bin/bash
# one GPU session: smoke, gpu tests, bench (+ A/B without the TMA GEMM), host/device phase profile
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-budget 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
DG_TMA=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_notma.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_notma.log
timeout 300 python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
