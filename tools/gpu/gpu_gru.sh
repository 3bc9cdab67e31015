#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gru.py tests/test_gpu_builders.py tests/test_gpu_parity.py -m gpu -q -x -k "gru or GRU or builder or transduce or workload or cfsm" -p no:cacheprovider > gpurun_out/pytest_gru.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gru.log
DG_GRU_FUSE=0 timeout 600 python -m pytest tests/test_gpu_gru.py -m gpu -q -x -p no:cacheprovider >> gpurun_out/pytest_gru.log 2>&1; echo "unfused rc=$?" >> gpurun_out/pytest_gru.log
timeout 600 python -m pytest tests/test_gpu_cfsm.py -m gpu -q -x -p no:cacheprovider >> gpurun_out/pytest_gru.log 2>&1; echo "cfsm rc=$?" >> gpurun_out/pytest_gru.log
DG_PNLS2=0 timeout 600 python -m pytest tests/test_gpu_cfsm.py -m gpu -q -x -p no:cacheprovider >> gpurun_out/pytest_gru.log 2>&1; echo "cfsm unfused rc=$?" >> gpurun_out/pytest_gru.log
