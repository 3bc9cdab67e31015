#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_split2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split2.log
AB_ENV="DG_TMA_PERS_SPLIT=0" AB_N=3 ./tools/gpu/gpu_ab_env.sh
