"""Per-step wall time of the public-API training loop (PTB MB=64), to find
host-side outliers in e2e.  Diagnostic only."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1701_03980_b200 as dy  # noqa: E402

cfg = bench.CONFIGS["ptb64"]
K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
CYCLE = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # >0: reuse this many batches cyclically (plan-cache hits)
data, units, _ = bench.make_data(cfg, K + 3, 0, 1)
if CYCLE:
    data = [data[i % CYCLE] for i in range(K + 3)]
pools = dy.new_poolset(1024, 1024, 64)
cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
task = bench.make_task(dy, model, cfg)
tr = dy.Trainer(model, "adam")
gcs = []
gc.callbacks.append(lambda phase, info: gcs.append((phase, info.get("generation"), time.perf_counter())))
for i in range(3):
    cg.renew(); loss = task.loss(cg, data[i]); cg.backward(loss); float(cg.value(loss).data[0]); tr.update()
torch.cuda.synchronize()
ts = []
for i in range(K):
    t0 = time.perf_counter()
    cg.renew()
    loss = task.loss(cg, data[3 + i])
    t1 = time.perf_counter()
    cg.backward(loss)
    t2 = time.perf_counter()
    float(cg.value(loss).data[0])
    t3 = time.perf_counter()
    tr.update()
    t4 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0, len(data[3 + i][0]), max(len(s) for s in data[3 + i])))
torch.cuda.synchronize()
a = np.array(ts) * 1e3
print("per step ms: construct  backward(plan+launch)  value-wait  update  total  | T_max")
for r, t in zip(a, ts):
    print("  %.3f  %.3f  %.3f  %.3f  %.3f  | %d" % (r[0], r[1], r[2], r[3], r[4], t[6]))
print("median", np.median(a[:, :5], axis=0).round(3), "gc events", len(gcs), [g[1] for g in gcs if g[0] == "start"])
