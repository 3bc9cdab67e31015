"""Diagnostic: per-node gradient comparison GPU vs oracle for one PTB MB16 step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_03980_b200 import workloads as W  # noqa: E402
from tests.helpers import gpu_ctx, oracle_ctx  # noqa: E402

sents = W.ptb_corpus(21, 32)
batch = W.minibatches(sents, 16)[0]
res = {}
for name, ctx in (("gpu", gpu_ctx(seed=3, mb=1024)), ("orc", oracle_ctx(seed=3)), ("o64", None)):
    if name == "o64":
        dy, cg, m = oracle_ctx(seed=3, dtype=np.float64)
        task = W.RNNLM(dy, m, 10_000, 128, 256, 2)
        for x, v in zip(list(m.parameters) + list(m.lookups), init):
            x.values[...] = v
    else:
        dy, cg, m = ctx
        task = W.RNNLM(dy, m, 10_000, 128, 256, 2)
        if name == "orc":
            init = [np.array(x.values, copy=True) for x in list(m.parameters) + list(m.lookups)]
    cg.renew()
    loss = task.loss(cg, batch)
    cg.backward(loss)
    kinds = [nd.kind for nd in cg.nodes] if hasattr(cg, "nodes") else list(cg.kinds)
    grads = {}
    for i, k in enumerate(kinds):
        if k in ("affine", "cmult", "add", "tanh", "logistic", "pick_range", "lookup_batch", "sum_batches",
                 "pickneglogsoftmax_batch"):
            e = type(loss)(cg, i, cg.generation)
            grads[i] = np.asarray(cg.gradient(e).data, dtype=np.float64)
    res[name] = (kinds, grads, {p.name: np.array(p.gradient if isinstance(p.gradient, np.ndarray) else p.gradient.data,
                                                 dtype=np.float64) for p in m.parameters})
kinds = res["gpu"][0]
worst = []
for i, g in res["gpu"][1].items():
    r = res["orc"][1][i]
    r64 = res["o64"][1][i]
    scale = max(1e-30, np.abs(r).max())
    err = np.abs(g - r)
    ref_err = np.abs(r - r64)
    j = int(np.argmax(err - 2 * ref_err))
    worst.append((float((err[j] - 2 * ref_err[j]) / scale), i, kinds[i], j, g[j], r[j], r64[j]))
worst.sort(reverse=True)
for w in worst[:15]:
    print("rel-excess %.3e node %d %s elem %d gpu %.9e orc %.9e o64 %.9e" % w)
for pname, g in res["gpu"][2].items():
    r, r64 = res["orc"][2][pname], res["o64"][2][pname]
    err = np.abs(g - r) - 2 * np.abs(r - r64)
    j = int(np.argmax(err))
    print(pname, "worst excess", err[j], "at", j, g[j], r[j], r64[j], "scale", np.abs(r).max())
