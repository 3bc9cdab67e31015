"""Median host time per phase of one training step (construct / forward plan+launch /
backward plan+launch / update) for a bench config; run with DG_DRYRUN=1 to
isolate the planner from device waits.  Diagnostic only."""
import os, sys, time
sys.path.insert(0, "/root/repo")
import bench
import paper_1701_03980_b200 as dy
name = sys.argv[1] if len(sys.argv) > 1 else "ptb64"
cfg = bench.CONFIGS[name]
N = 43
data, units, tg = bench.make_data(cfg, N, 0, 1)
pools = dy.new_poolset(1024, 1024, 64)
cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
task = bench.make_task(dy, model, cfg, tg)
tr = dy.Trainer(model, "adam")
ts = []
for i in range(N):
    t0 = time.perf_counter()
    cg.renew(); loss = bench.call_loss(task, cg, data[i])
    t1 = time.perf_counter()
    cg.forward_to(loss)
    t2 = time.perf_counter()
    cg.backward(loss)
    t3 = time.perf_counter()
    tr.update()
    t4 = time.perf_counter()
    ts.append((t1-t0, t2-t1, t3-t2, t4-t3, t4-t0))
import numpy as np
a = np.median(np.array(ts[3:]), axis=0) * 1e3
print(name, "construct %.3f fwd %.3f bwd %.3f update %.3f total %.3f ms" % tuple(a))
