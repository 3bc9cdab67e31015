"""The fused GRU step (executor match_gru + kernels.cu gru_*_kernel) keeps
every node of the reference pattern (builders.py:102-110): values and
gradients of each internal expression on the device vs the oracle, with a
per-row or broadcast (batch-1) previous state, batched and batch 1."""
import numpy as np
import pytest

from tests.helpers import gpu_ctx, oracle_ctx, parity

pytestmark = pytest.mark.gpu

H, X = 24, 10


def _gru_steps(dy, cg, model, B, h_b1, steps=3, seed=3):
    ops = dy.ops
    wx = model.add_parameters((3 * H, X), "wx")
    wh = model.add_parameters((3 * H, H), "wh")
    b = model.add_parameters((3 * H,), "b")
    rng = np.random.default_rng(seed)
    cg.renew()
    pb, pwx, pwh = ops.parameter(cg, b), ops.parameter(cg, wx), ops.parameter(cg, wh)
    hb = 1 if h_b1 else B
    h = ops.input(cg, dy.Tensor(dy.Shape((H,), hb), (0.3 * rng.standard_normal(H * hb)).astype(np.float32)))
    ones = dy.Tensor(dy.Shape((H,)), np.ones(H, dtype=np.float32))
    watch = {"h0": h}
    for t in range(steps):
        x = ops.input(cg, dy.Tensor(dy.Shape((X,), B), rng.standard_normal(X * B).astype(np.float32)))
        zr = ops.affine(pb, pwx, x, pwh, h)
        z = ops.logistic(ops.pick_range(zr, 0, H))
        r = ops.logistic(ops.pick_range(zr, H, 2 * H))
        cx = ops.pick_range(ops.affine(pb, pwx, x), 2 * H, 3 * H)
        rh = ops.cmult(r, h)
        ch = ops.pick_range(ops.matmul(pwh, rh), 2 * H, 3 * H)
        cand = ops.tanh(ops.add(cx, ch))
        keep = ops.add(ops.input(cg, ones), ops.scalar_mul(z, -1.0))
        h = ops.add(ops.cmult(keep, h), ops.cmult(z, cand))
        watch.update({f"z{t}": z, f"r{t}": r, f"cx{t}": cx, f"rh{t}": rh, f"ch{t}": ch, f"cand{t}": cand,
                      f"keep{t}": keep, f"h{t}": h, f"x{t}": x})
    loss = ops.sum_batches(ops.pickneglogsoftmax_batch(h, [int(v) for v in rng.integers(0, H, B)]))
    cg.backward(loss)
    vals = {k: np.asarray(cg.value(e).data, dtype=np.float64) for k, e in watch.items()}
    grads = {k: np.asarray(cg.gradient(e).data, dtype=np.float64) for k, e in watch.items()}
    pg = {p.name: np.asarray(p.gradient.data if hasattr(p.gradient, "data") else p.gradient, dtype=np.float64)
          for p in model.parameters}
    return vals, grads, pg


@pytest.mark.parametrize("B,h_b1", [(4, False), (4, True), (1, False)])
def test_fused_gru_nodes_match_oracle(B, h_b1):
    dyg, cgg, mg = gpu_ctx(seed=9, mb=64)
    dyo, cgo, mo = oracle_ctx(seed=9)
    gv, gg, gp = _gru_steps(dyg, cgg, mg, B, h_b1)
    rv, rg, rp = _gru_steps(dyo, cgo, mo, B, h_b1)
    for k in rv:
        parity(gv[k], rv[k], what=f"value {k}")
        parity(gg[k], rg[k], what=f"gradient {k}")
    for k in rp:
        parity(gp[k], rp[k], what=f"param grad {k}")
