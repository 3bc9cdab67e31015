#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
DG_EARLY_DW=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --only > gpurun_out/edw_off.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --only > gpurun_out/edw_on.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_semantics.py tests/test_gpu_dp.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_edw.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_edw.log
AB_ENV="DG_EARLY_DW=0" AB_N=3 ./tools/gpu/gpu_ab_env.sh
