#!/bin/bash
# host-side phase timings (real and dry-run) + GPU parity subset
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/e2e_steps.py 30 > gpurun_out/e2e_steps.txt 2>&1
for c in ptb64 tree tagger ptb16; do
  timeout 300 python tools/host_phases.py $c >> gpurun_out/host_real.txt 2>&1
  DG_DRYRUN=1 timeout 300 python tools/host_phases.py $c >> gpurun_out/host_dry.txt 2>&1
done
timeout 300 python tools/profile_step.py > gpurun_out/host_phases.txt 2>&1
