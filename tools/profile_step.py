"""Diagnostics for one workload: host-side phase timings of the API step and
(under ncu) the per-kernel launch list.  Not a benchmark."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03980_b200 as dy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="ptb64")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--warmup", type=int, default=2)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
data, units, tg = bench.make_data(cfg, args.steps + args.warmup, 0, 1)
pools = dy.new_poolset(1024, 1024, 64)
cg = dy.ComputationGraph(pools)
model = dy.Model(pools, seed=1)
task = bench.make_task(dy, model, cfg, tg)
tr = dy.Trainer(model, "adam")
acc = {}


def tick(name, t0):
    acc.setdefault(name, []).append(time.perf_counter() - t0)
    return time.perf_counter()


for i in range(args.steps + args.warmup):
    torch.cuda.synchronize()
    t = time.perf_counter()
    cg.renew()
    loss = bench.call_loss(task, cg, data[i])
    t = tick("construct", t)
    cg._prepare()
    t = tick("flush", t)
    cg.backward(loss)
    t = tick("backward_host", t)
    tr.update()
    t = tick("update_host", t)
    torch.cuda.synchronize()
    t = tick("device_drain", t)
    float(cg.value(loss).data[0])
    t = tick("value", t)
for k, v in acc.items():
    v = v[args.warmup:]
    print(f"{k:14s} {1e3 * np.mean(v):8.3f} ms")
print("launches", cg._counters()[5], "plan", cg.plan_stats())
