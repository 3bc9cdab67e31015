#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
rm -f gpurun_out/strict_report.tsv
DG_STRICT_REPORT=$PWD/gpurun_out/strict_report.tsv timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_semantics.py tests/test_gpu_cfsm.py tests/test_gpu_builders.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_rowcs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rowcs.log
out=gpurun_out/ab_env.txt; : > $out
for i in 1 2 3; do echo "B" >> $out; timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --only 2>&1 | grep '^{' >> $out; done
