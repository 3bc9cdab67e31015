#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/host_ph.txt
for c in ptb64 tagger tree tiny; do
  timeout 300 python tools/host_phases.py $c >> gpurun_out/host_ph.txt 2>&1
  DG_DRYRUN=1 timeout 300 python tools/host_phases.py $c | sed 's/^/dry /' >> gpurun_out/host_ph.txt 2>&1
done
python - >> gpurun_out/host_ph.txt 2>&1 <<'PY'
import cProfile, pstats, sys, io
sys.path.insert(0, '.')
import bench, paper_1701_03980_b200 as dy
for name in ("tagger", "tree"):
    cfg = bench.CONFIGS[name]
    data, units, tg = bench.make_data(cfg, 60, 0, 1)
    pools = dy.new_poolset(128, 128, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    task = bench.make_task(dy, model, cfg, tg)
    tr = dy.Trainer(model, "adam")
    def run(lo, hi):
        for i in range(lo, hi):
            cg.renew(); loss = bench.call_loss(task, cg, data[i]); cg.backward(loss); float(cg.value(loss).data[0]); tr.update()
    run(0, 10)
    pr = cProfile.Profile(); pr.enable(); run(10, 60); pr.disable()
    s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18); print("==", name); print(s.getvalue()[:4000])
PY
