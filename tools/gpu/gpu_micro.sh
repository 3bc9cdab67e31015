#!/bin/bash
# micro batches + scatter combine: parity, kernel paths, A/B bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_semantics.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_micro.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_micro.log
rm -f gpurun_out/ab_micro.txt
for i in 1 2; do
  DG_MICRO=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --only >> gpurun_out/ab_micro.txt 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --only >> gpurun_out/ab_micro.txt 2>&1
done
