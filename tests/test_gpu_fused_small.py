"""Fused small levels with an activation instead of a gated cell (executor
act_level + cellgemm.cu level_fwd): simple-RNN steps tanh(affine(b, Wx, x,
Wh, h)) (builders.py:90-91) and TreeRNN composes tanh(matmul(W,
concatenate([e1, e2]))) (builders.py:183-210).  Values and gradients of every
node (affine / matmul, concatenate, activation) vs the oracle."""
import numpy as np
import pytest

from tests.helpers import gpu_ctx, oracle_ctx, parity

pytestmark = pytest.mark.gpu

H, X = 20, 12


def _simple(dy, cg, model, B, h_b1):
    ops = dy.ops
    wx = model.add_parameters((H, X), "wx")
    wh = model.add_parameters((H, H), "wh")
    b = model.add_parameters((H,), "b")
    rng = np.random.default_rng(2)
    cg.renew()
    pb, pwx, pwh = ops.parameter(cg, b), ops.parameter(cg, wx), ops.parameter(cg, wh)
    hb = 1 if h_b1 else B
    h = ops.input(cg, dy.Tensor(dy.Shape((H,), hb), (0.4 * rng.standard_normal(H * hb)).astype(np.float32)))
    watch = {"h0": h}
    for t in range(4):
        x = ops.input(cg, dy.Tensor(dy.Shape((X,), B), rng.standard_normal(X * B).astype(np.float32)))
        a = ops.affine(pb, pwx, x, pwh, h)
        h = ops.tanh(a)
        watch.update({f"a{t}": a, f"h{t + 1}": h, f"x{t}": x})
    loss = ops.sum_batches(ops.pickneglogsoftmax_batch(h, [int(v) for v in rng.integers(0, H, B)]))
    return watch, loss


def _treernn(dy, cg, model, B, h_b1):
    ops = dy.ops
    W = model.add_parameters((H, 2 * H), "W")
    E = model.add_lookup_parameters(30, H, "E")
    cg.renew()
    pw = ops.parameter(cg, W)
    leaves = [ops.lookup(cg, E, i) for i in (3, 7, 11, 5, 2)]
    watch = {f"leaf{i}": e for i, e in enumerate(leaves)}
    level, k = leaves, 0
    while len(level) > 1:
        nxt = []
        for i in range(0, len(level) - 1, 2):
            c = ops.concatenate([level[i], level[i + 1]])
            m = ops.matmul(pw, c)
            t = ops.tanh(m)
            watch.update({f"c{k}": c, f"m{k}": m, f"t{k}": t})
            k += 1
            nxt.append(t)
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    loss = ops.pickneglogsoftmax(level[0], 4)
    return watch, loss


@pytest.mark.parametrize("case,B,h_b1", [("simple", 3, False), ("simple", 3, True), ("simple", 1, False),
                                          ("treernn", 1, False)])
def test_fused_activation_levels_match_oracle(case, B, h_b1):
    build = _simple if case == "simple" else _treernn
    out = []
    for dy, cg, model in (gpu_ctx(seed=4, mb=64), oracle_ctx(seed=4)):
        watch, loss = build(dy, cg, model, B, h_b1)
        cg.backward(loss)
        vals = {k: np.asarray(cg.value(e).data, np.float64) for k, e in watch.items()}
        grads = {k: np.asarray(cg.gradient(e).data, np.float64) for k, e in watch.items()}
        pg = {p.name: np.asarray(p.gradient.data if hasattr(p.gradient, "data") else p.gradient, np.float64)
              for p in model.parameters}
        out.append((vals, grads, pg, float(cg.value(loss).data[0])))
    (gv, gg, gp, gl), (rv, rg, rp, rl) = out
    parity(gl, rl, what="loss")
    for k in rv:
        parity(gv[k], rv[k], what=f"value {k}")
        parity(gg[k], rg[k], what=f"gradient {k}")
    for k in rp:
        parity(gp[k], rp[k], what=f"param grad {k}")
