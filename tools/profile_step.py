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

# ---- live device-only per-class timing: stall the GPU with a spin kernel so
# the host enqueues the whole step first, then read the CUDA-event windows
classes = ("gemm_fwd", "gemm_dx", "gemm_dw", "pnls_fwd", "pnls_bwd", "elementwise", "gather", "scatter_add",
           "bias_colsum", "other", "rnn_fwd", "rnn_bwd")
cg.profile_enable(classes)
tot = {c: 0.0 for c in classes}
cnt = {c: 0 for c in classes}
n_meas = 3
for i in range(n_meas):
    torch.cuda.synchronize()
    cg.profile_reset()
    cg.renew()
    loss = bench.call_loss(task, cg, data[i % len(data)])
    cg._prepare()
    torch.cuda._sleep(int(40e6))  # ~20 ms spin
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    cg.backward(loss)
    tr.update()
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1)
    for c in classes:
        r = cg.profile_read(c)
        tot[c] += r["ms"]
        cnt[c] += r["launches"]
    print(f"device-only step {step_ms:.3f} ms")
for c in classes:
    if cnt[c]:
        print(f"  {c:12s} {tot[c] / n_meas:8.3f} ms/step  {cnt[c] / n_meas:6.1f} launches  "
              f"{1e3 * tot[c] / max(1, cnt[c]):7.1f} us/launch")
