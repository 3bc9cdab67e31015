#!/bin/bash
# same-box A/B of csrc variants: ./gpu_ab_src.sh A B ... ; variant X = the csrc
# files under abtmp/X/ over a copy of the repo ("cur" = the repo as shipped)
mkdir -p gpurun_out; : > gpurun_out/ab_src.txt
for v in "$@"; do
  d=/tmp/ab_$v; rm -rf $d; mkdir -p $d
  cp -r paper_1701_03980_b200 tools bench.py Makefile __graft_entry__.py oracle include $d/ 2>/dev/null
  if [ "$v" != "cur" ]; then cp abtmp/$v/* $d/paper_1701_03980_b200/csrc/; (cd $d && make -j32 > /dev/null 2>&1 || echo "build $v failed" >> $GRAFT_REPO_ROOT/gpurun_out/ab_src.txt); fi
  echo "== $v" >> gpurun_out/ab_src.txt
  (cd $d && DG_RNN_TRACE=2 timeout 300 python tools/rnn_trace.py 2>&1 | grep -v "^\[rnn\]" | head -4) >> gpurun_out/ab_src.txt
  (cd $d && timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --only 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_launch']*1e3,1) for k,v in d['rooflines'].items()})
") >> gpurun_out/ab_src.txt
done
