#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/san2.txt
for i in 1 2; do echo "== plain $i" >> gpurun_out/san2.txt; timeout 300 python tools/sanitize.py >> gpurun_out/san2.txt 2>&1; done
echo "== cluster off" >> gpurun_out/san2.txt; DG_RNN_CLUSTER=0 timeout 300 python tools/sanitize.py >> gpurun_out/san2.txt 2>&1
echo "== rnn off" >> gpurun_out/san2.txt; DG_RNN=0 timeout 300 python tools/sanitize.py >> gpurun_out/san2.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python tools/sanitize.py > gpurun_out/san_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.txt
