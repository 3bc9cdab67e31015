"""The fused class-factored softmax term (executor U_PNLS2 + kernels.cu
pnls2_*_kernel): values and gradients of the class / word score rows and of
every picked negative log softmax node vs the oracle, including several
terms sharing one h (shared class scores: the conflict rounds path) and a
term whose class and word rows differ in width (builders.py:282-378)."""
import numpy as np
import pytest

from tests.helpers import gpu_ctx, oracle_ctx, parity

pytestmark = pytest.mark.gpu

HID = 8
CLASSES = {f"w{i}": i % 3 for i in range(17)}  # class sizes 6, 6, 5


def _run(dy, cg, model, shared):
    ops = dy.ops
    cf = dy.ClassFactoredSoftmax(model, HID, CLASSES, "cf")
    rng = np.random.default_rng(4)
    cg.renew()
    hs = [ops.input(cg, dy.Tensor(dy.Shape((HID,)), rng.standard_normal(HID).astype(np.float32)))
          for _ in range(1 if shared else 5)]
    words = ["w0", "w4", "w8", "w13", "w16"]
    terms, loss = [], None
    for k, w in enumerate(words):
        h = hs[0 if shared else k]
        t = cf.neg_log_softmax(cg, h, w)
        terms.append(t)
        loss = t if loss is None else ops.add(loss, t)
    cg.backward(loss)
    out = {}
    for k, t in enumerate(terms):
        out[f"term{k}"] = (np.asarray(cg.value(t).data, np.float64), np.asarray(cg.gradient(t).data, np.float64))
    for k, h in enumerate(hs):
        out[f"h{k}"] = (np.asarray(cg.value(h).data, np.float64), np.asarray(cg.gradient(h).data, np.float64))
    pg = {p.name: np.asarray(p.gradient.data if hasattr(p.gradient, "data") else p.gradient, np.float64)
          for p in model.parameters}
    return out, pg


@pytest.mark.parametrize("shared", [False, True])
def test_fused_cfsm_terms_match_oracle(shared):
    dyg, cgg, mg = gpu_ctx(seed=6, mb=64)
    dyo, cgo, mo = oracle_ctx(seed=6)
    got, gp = _run(dyg, cgg, mg, shared)
    ref, rp = _run(dyo, cgo, mo, shared)
    for k in ref:
        parity(got[k][0], ref[k][0], what=f"value {k}")
        parity(got[k][1], ref[k][1], what=f"gradient {k}")
    for k in rp:
        parity(gp[k], rp[k], what=f"param grad {k}")
