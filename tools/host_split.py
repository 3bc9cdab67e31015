"""Host time split of one public-API training step (construct / node-table
flush / dg_forward / dg_backward / value / update).  Diagnostic only."""
import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_1701_03980_b200 as dy
from paper_1701_03980_b200 import _native
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "ptb64"]
N = 33
data, units, tg = bench.make_data(cfg, N, 0, 1)
pools = dy.new_poolset(1024, 1024, 64)
cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
task = bench.make_task(dy, model, cfg, tg)
tr = dy.Trainer(model, "adam")
lib = _native.lib()
ts = []
for i in range(N):
    t0 = time.perf_counter()
    cg.renew(); loss = bench.call_loss(task, cg, data[i])
    t1 = time.perf_counter()
    h = cg._prepare()
    t2 = time.perf_counter()
    _native.check(lib.dg_forward(h, loss.index)); cg._advance(loss.index)
    t3 = time.perf_counter()
    _native.check(lib.dg_backward(h, loss.index)); cg._advance(loss.index)
    t4 = time.perf_counter()
    float(cg.value(loss).data[0])
    t5 = time.perf_counter()
    tr.update()
    t6 = time.perf_counter()
    ts.append((t1-t0, t2-t1, t3-t2, t4-t3, t5-t4, t6-t5))
torch.cuda.synchronize()
a = np.median(np.array(ts[3:]), axis=0) * 1e3
print("construct %.3f prepare %.3f dg_forward %.3f dg_backward %.3f value %.3f update %.3f (ms)" % tuple(a))
