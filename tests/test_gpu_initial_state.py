"""Gradients of LSTM initial states on the device vs the oracle.

The backward recurrence kernel (rnn.cu) produces dh_{-1} / dc_{-1} itself:
per-row targets in place, batch-1 targets as per-slice row sums that are
summed right away for computed / parameter nodes and on `gradient()` for
INPUT leaves (executor.cpp LazyGrad).  The reference computes every node's
gradient during backward (graph.py:139-164), so `gradient()` of the initial
state inputs and the parameter gradients of a learned initial state must
match it (rtol 1e-4) however they are produced."""
import numpy as np
import pytest

from tests.helpers import gpu_ctx, oracle_ctx, parity, pgrad

pytestmark = pytest.mark.gpu

V, E, H, L, T = 50, 16, 32, 2, 5


def _run(dy, cg, model, mode, B, seed=7):
    ops = dy.ops
    emb = model.add_lookup_parameters(V, E, "E")
    rnn = dy.RNNBuilder(model, L, E, H, "lstm", "rnn")
    W = model.add_parameters((V, H), "W")
    bo = model.add_parameters((V,), "bo")
    h0p = [model.add_parameters((H,), f"h0.{l}") for l in range(L)]
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, V, size=(T + 1, B))
    init = rng.standard_normal((L, 2, B, H)).astype(np.float32) * 0.5
    cg.renew()
    s0 = rnn.initial_state(cg)
    if mode == "rows":  # per-row initial states (batch-B inputs)
        s0.hs = [ops.input(cg, dy.Tensor(dy.Shape((H,), B), init[l, 0].reshape(-1).copy())) for l in range(L)]
        s0.cs = [ops.input(cg, dy.Tensor(dy.Shape((H,), B), init[l, 1].reshape(-1).copy())) for l in range(L)]
    elif mode == "param":  # learned batch-1 h_{-1}: its gradient lands in a parameter
        s0.hs = [ops.parameter(cg, p) for p in h0p]
    xs = [ops.lookup_batch(cg, emb, [int(v) for v in ids[t]]) for t in range(T)]
    outs = s0.transduce(xs)
    we, be = ops.parameter(cg, W), ops.parameter(cg, bo)
    loss = None
    for t, h in enumerate(outs):
        nll = ops.sum_batches(ops.pickneglogsoftmax_batch(ops.affine(be, we, h), [int(v) for v in ids[t + 1]]))
        loss = nll if loss is None else ops.add(loss, nll)
    cg.backward(loss)
    grads = {}
    for l in range(L):
        grads[f"h{l}"] = np.asarray(cg.gradient(s0.hs[l]).data, dtype=np.float64)
        grads[f"c{l}"] = np.asarray(cg.gradient(s0.cs[l]).data, dtype=np.float64)
    params = {p.name: pgrad(p) for p in model.parameters}
    return grads, params, cg.value(loss).data[0]


@pytest.mark.parametrize("mode,B", [("zeros", 8), ("zeros", 1), ("rows", 8), ("param", 8), ("zeros", 20)])
def test_initial_state_gradients_match_oracle(mode, B):
    dyg, cgg, mg = gpu_ctx(seed=5, mb=64)
    dyo, cgo, mo = oracle_ctx(seed=5)
    got, gp, gl = _run(dyg, cgg, mg, mode, B)
    ref, rp, rl = _run(dyo, cgo, mo, mode, B)
    parity(gl, rl, what="loss")
    for k in ref:
        parity(got[k], ref[k], what=f"gradient({k})")
    for k in rp:
        parity(gp[k], rp[k], what=f"param grad {k}")


def test_lazy_initial_state_gradient_is_summed_once():
    dyg, cgg, mg = gpu_ctx(seed=5, mb=64)
    ops = dyg.ops
    emb = mg.add_lookup_parameters(V, E, "E")
    rnn = dyg.RNNBuilder(mg, 1, E, H, "lstm", "rnn")
    cgg.renew()
    s0 = rnn.initial_state(cgg)
    xs = [ops.lookup_batch(cgg, emb, list(range(t, t + 8))) for t in range(T)]
    out = s0.transduce(xs)[-1]
    loss = ops.sum_batches(ops.pickneglogsoftmax_batch(out, list(range(8))))
    cgg.backward(loss)
    a = np.asarray(cgg.gradient(s0.hs[0]).data).copy()
    b = np.asarray(cgg.gradient(s0.hs[0]).data).copy()
    assert np.array_equal(a, b)
    assert np.abs(a).max() > 0
    cgg.backward(loss)  # a second backward: fresh slots, same gradient
    c = np.asarray(cgg.gradient(s0.hs[0]).data)
    np.testing.assert_array_equal(a, c)
