"""Timeline of the persistent LSTM kernels (DG_RNN_TRACE=1): per-step arrival
stamps of every CTA for one PTB MB=64 training step.  Diagnostic only."""
import os
import sys

os.environ.setdefault("DG_RNN_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1701_03980_b200 as dy  # noqa: E402
from paper_1701_03980_b200 import _native  # noqa: E402

cfg = bench.CONFIGS["ptb64"]
data, units, _ = bench.make_data(cfg, 4, 0, 1)
pools = dy.new_poolset(1024, 1024, 64)
cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
task = bench.make_task(dy, model, cfg)
tr = dy.Trainer(model, "adam")
for d in data:
    cg.renew()
    loss = task.loss(cg, d)
    cg.backward(loss)
    tr.update()
torch.cuda.synchronize()
T = max(len(s) for s in data[-1]) - 1
buf = np.zeros(2 * 148 * 256, np.uint64)
_native.check(_native.lib().dg_rnn_trace(buf.ctypes.data, buf.size))
buf = buf.reshape(2, 148, 256).astype(np.int64)
for kind, name in ((0, "fwd"), (1, "bwd")):
    b = buf[kind]
    live = b[:, 0] > 0
    b = b[live]
    t0 = b[:, 0].min()
    arr = b[:, 2:2 + T] - t0
    order = arr[:, -1] if kind == 0 else arr[:, 0]
    steps = np.abs(np.diff(arr.max(axis=0)))
    print(f"== {name} (last launch, {live.sum()} CTAs): weights resident {(b[:, 1] - b[:, 0]).mean() / 1e3:.1f} us, "
          f"per-step {np.median(steps) / 1e3:.2f} us (min {steps.min() / 1e3:.2f}, max {steps.max() / 1e3:.2f}), "
          f"total {order.max() / 1e3:.1f} us, arrival skew {np.median(arr.max(axis=0) - arr.min(axis=0)) / 1e3:.2f} us")

if os.environ.get("DG_RNN_TRACE") == "2":
    # per-step phases of CTA 0 of the last forward launch (slots 64 + 4t + k)
    b = buf[0, 0]
    ph = b[64:64 + 4 * min(T, 47)].reshape(-1, 4).astype(np.int64)
    d = np.diff(np.concatenate([ph, np.roll(ph[:, :1], -1, axis=0)], axis=1), axis=1)[:-1]
    print("fwd CTA0 per-step phases (us): wait, fma, reduce+cell, push+rest ->", np.round(np.median(d, axis=0) / 1e3, 2))
    n = min(T, 47) - 1
    cell_end = ph[:n, 3]
    arrive = b[2:2 + n].astype(np.int64)  # after the push and the step barrier
    nxt = ph[1:n + 1, 0]
    print("  push+rest split (us): push+barrier", np.round(np.median(arrive - cell_end) / 1e3, 2),
          "stores+next step top", np.round(np.median(nxt - arrive) / 1e3, 2))

if os.environ.get("DG_RNN_TRACE") == "2":
    b = buf[0]
    live = b[:, 0] > 0
    b = b[live].astype(np.int64)
    t0 = b[:, 0]
    ph = np.stack([b[:, 252] - t0, b[:, 253] - t0, b[:, 254] - t0, b[:, 1] - t0, t0 - t0.min()], axis=1)
    print("fwd prologue (us, median over CTAs): weights", np.round(np.median(ph[:, 0]) / 1e3, 2), "| +init sync",
          np.round(np.median(ph[:, 1]) / 1e3, 2), "| +h_-1", np.round(np.median(ph[:, 2]) / 1e3, 2),
          "| +cluster sync", np.round(np.median(ph[:, 3]) / 1e3, 2), "| CTA start skew max",
          np.round(ph[:, 4].max() / 1e3, 2))

