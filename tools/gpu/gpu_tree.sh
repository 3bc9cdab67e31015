#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/tree_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_builders.py tests/test_gpu_semantics.py tests/test_gpu_acceptance.py tests/test_frontend.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_tree.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tree.log
for c in tree tagger; do for v in "DG_X=1" "DG_AFFCELL=0"; do
  echo "== $c $v" >> gpurun_out/tree_ab.txt
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --config $c --only --no-cpu 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'])" >> gpurun_out/tree_ab.txt
done; done
