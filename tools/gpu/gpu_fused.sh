#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_small.py tests/test_gpu_gru.py tests/test_gpu_cfsm.py tests/test_gpu_builders.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
DG_AFFCELL=0 timeout 600 python -m pytest tests/test_gpu_fused_small.py -m gpu -q -x -p no:cacheprovider >> gpurun_out/pytest_fused.log 2>&1; echo "unfused rc=$?" >> gpurun_out/pytest_fused.log
