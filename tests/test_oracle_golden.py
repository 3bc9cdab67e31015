"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures come from tests/golden/make_golden.py (reference imported from
/root/reference in the build container).  The oracle restates the same fp32
algorithm, so agreement is expected to the last few ulps.
"""

import os

import numpy as np
import pytest

from oracle import engine as orc
from tests.golden import cases

GOLD = os.path.join(os.path.dirname(__file__), "golden")
OPS = np.load(os.path.join(GOLD, "ops.npz"))
WL = np.load(os.path.join(GOLD, "workloads.npz"))


def close(a, b, rtol=1e-5, atol_frac=1e-6):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(1.0, float(np.abs(b).max(initial=0.0)))
    assert a.shape == b.shape, (a.shape, b.shape)
    assert np.all(np.abs(a - b) <= rtol * np.abs(b) + atol_frac * scale), np.abs(a - b).max()


@pytest.mark.parametrize("name", sorted(cases.OP_CASES))
def test_oracle_op_cases(name):
    pools = orc.new_poolset()
    cg, model = orc.ComputationGraph(pools), orc.Model(pools, seed=7)
    out, ins = cases.OP_CASES[name](orc, cg, model)
    loss = cases.scalarize(orc, cg, out)
    cg.backward(loss)
    close(cg.value(loss).data, OPS[f"{name}/loss"])
    close(cg.value(out).data, OPS[f"{name}/value"])
    for k, e in enumerate(ins):
        close(cg.gradient(e).data, OPS[f"{name}/grad{k}"])
    for p in model.parameters:
        close(p.gradient, OPS[f"{name}/pgrad/{p.name}"])
    for lp in model.lookups:
        close(lp.gradient, OPS[f"{name}/lgrad/{lp.name}"])
        assert sorted(lp.touched) == list(OPS[f"{name}/touched/{lp.name}"])
    assert cg.forward_calls == int(OPS[f"{name}/forward_calls"][0])


@pytest.mark.parametrize("name", sorted(cases.workload_cases()))
def test_oracle_workload_traces(name):
    make_task, data, rule, steps = cases.workload_cases()[name]
    pools = orc.new_poolset()
    cg, model = orc.ComputationGraph(pools), orc.Model(pools, seed=1)
    task = make_task(orc, model)
    for p in model.parameters:
        assert np.array_equal(p.values, WL[f"{name}/init/{p.name}"])
    for lp in model.lookups:
        assert np.array_equal(lp.values, WL[f"{name}/init/{lp.name}"])
    tr = orc.Trainer(model, rule)
    for s in range(steps):
        cg.renew()
        loss = cases.call_loss(task, cg, data[s])
        cg.backward(loss)
        close(cg.value(loss).data, WL[f"{name}/loss{s}"])
        for p in model.parameters:
            key = f"{name}/grad{s}/{p.name}"
            if key in WL:
                close(p.gradient, WL[key])
        for lp in model.lookups:
            rows = WL[f"{name}/touched{s}/{lp.name}"]
            assert sorted(lp.touched) == list(rows)  # bit-exact touched set
            close(lp.gradient[rows], WL[f"{name}/lgrad{s}/{lp.name}"])
        tr.update()
    for p in model.parameters:
        close(p.values, WL[f"{name}/final/{p.name}"])
    for lp in model.lookups:
        close(lp.values, WL[f"{name}/final/{lp.name}"])
