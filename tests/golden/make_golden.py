"""Generate golden fixtures from the REAL reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/ops.npz and tests/golden/workloads.npz.  The reference is
imported read-only from /root/reference (it does not exist on the GPU box, so
the fixtures are committed).  Inputs are seeded; outputs are whatever the
reference computes in fp32 (PoolSet dtype float32, core/arena.py:76).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")

import dyncore as ref  # noqa: E402

from tests.golden import cases  # noqa: E402
from paper_1701_03980_b200 import workloads as W  # noqa: E402


def mk(seed=1, mb=64):
    pools = ref.new_poolset(mb, mb, mb)
    return ref.ComputationGraph(pools), ref.Model(pools, seed=seed)


def gen_ops():
    out = {}
    for name, build in cases.OP_CASES.items():
        cg, model = mk(seed=7)
        outs, ins = build(ref, cg, model)
        loss = cases.scalarize(ref, cg, outs)
        cg.backward(loss)
        out[f"{name}/loss"] = cg.value(loss).data.astype(np.float32)
        out[f"{name}/value"] = cg.value(outs).data.astype(np.float32)
        for k, e in enumerate(ins):
            out[f"{name}/grad{k}"] = cg.gradient(e).data.astype(np.float32)
        for p in model.parameters:
            out[f"{name}/pgrad/{p.name}"] = p.gradient.data.copy()
        for lp in model.lookups:
            out[f"{name}/lgrad/{lp.name}"] = lp.gradient.copy()
            out[f"{name}/touched/{lp.name}"] = np.array(sorted(lp.touched), dtype=np.int64)
        out[f"{name}/forward_calls"] = np.array([cg.forward_calls])
        out[f"{name}/alloc"] = np.array([cg.pools.forward.alloc_count, cg.pools.backward.alloc_count])
    return out


def gen_workloads():
    out = {}
    for name, (make_task, data, rule, steps) in cases.workload_cases().items():
        cg, model = mk(seed=1, mb=512)
        task = make_task(ref, model)
        for p in model.parameters:
            out[f"{name}/init/{p.name}"] = p.values.data.copy()
        for lp in model.lookups:
            out[f"{name}/init/{lp.name}"] = lp.values.copy()
        tr = ref.Trainer(model, rule)
        for s in range(steps):
            cg.renew()
            loss = cases.call_loss(task, cg, data[s])
            cg.backward(loss)
            out[f"{name}/loss{s}"] = cg.value(loss).data.astype(np.float32)
            for p in model.parameters:
                if name != "tiny" or s == 0:  # keep the fixture small
                    out[f"{name}/grad{s}/{p.name}"] = p.gradient.data.copy()
            for lp in model.lookups:
                rows = np.array(sorted(lp.touched), dtype=np.int64)
                out[f"{name}/touched{s}/{lp.name}"] = rows
                out[f"{name}/lgrad{s}/{lp.name}"] = lp.gradient[rows].copy()
            tr.update()
        for p in model.parameters:
            out[f"{name}/final/{p.name}"] = p.values.data.copy()
        for lp in model.lookups:
            out[f"{name}/final/{lp.name}"] = lp.values.copy()
    return out


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **gen_ops())
    np.savez_compressed(os.path.join(HERE, "workloads.npz"), **gen_workloads())
    for f in ("ops.npz", "workloads.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))
