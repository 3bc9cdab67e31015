"""Host-only checks of the native graph core (csrc/dgcore.c): the composite
LSTM-cell builder must write exactly the nodes and records the node-by-node
path writes (builders.py RNNBuilder._lstm), irregular inputs must take the
node-by-node path and raise its errors, and the construction helpers keep the
reference semantics (tuple(map(int, ids)) for batched lookups)."""

import ctypes

import numpy as np
import pytest

import paper_1701_03980_b200 as dy
from paper_1701_03980_b200 import ops
from paper_1701_03980_b200._dgcore import int_tuple

HDR = 13


def _records(cg):
    hdr, n, ins, n_ins, ai, n_ai, af, n_af = cg._core.pack(0)

    def arr(ptr, count, ctype, dtype):
        if count == 0:
            return np.zeros(0, dtype)
        return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), (count,)).copy()

    return (arr(hdr, n * HDR, ctypes.c_int32, np.int32), arr(ins, n_ins, ctypes.c_int32, np.int32),
            arr(ai, n_ai, ctypes.c_int64, np.int64), arr(af, n_af, ctypes.c_float, np.float32))


def _aux(a):
    if isinstance(a, dy.Tensor):
        return ("tensor", tuple(a.shape.dims), a.shape.batch, np.asarray(a.data).tobytes())
    if isinstance(a, tuple):
        return tuple(_aux(v) for v in a)
    if hasattr(a, "handle"):  # parameters of the two (separately built) models
        return ("param", tuple(a.shape.dims) if hasattr(a, "shape") else (a.rows, a.dim))
    return a


def _nodes(cg):
    return [(n.kind, tuple(n.inputs), tuple(n.shape.dims), n.shape.batch, _aux(n.aux)) for n in cg.nodes]


def _build(native, H=8, X=6, batch_x=4, batch_state=1, steps=3, transduce=False):
    pools = dy.new_poolset(64, 64, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    rnn = dy.RNNBuilder(model, 2, X, H, "lstm")
    E = model.add_lookup_parameters(20, X)
    saved = cg._core
    if not native:
        cg._core = None  # builders fall back to one ops call per node
    try:
        state = rnn.initial_state(cg)
        if batch_state > 1:
            zero = dy.Tensor(dy.Shape((H,), batch_state), np.zeros(H * batch_state, np.float32))
            state.hs = [ops.input(cg, zero) for _ in state.hs]
            state.cs = [ops.input(cg, zero) for _ in state.cs]
        xs = []
        for t in range(steps):
            x = ops.lookup_batch(cg, E, [(t + r) % 20 for r in range(batch_x)]) if batch_x > 1 else ops.lookup(cg, E, t)
            if transduce:
                xs.append(x)
            else:
                state = state.add_input(x)
        out = state.transduce(xs) if transduce else state.output()
    finally:
        cg._core = saved
    return cg, out


@pytest.mark.parametrize("transduce", [False, True])
@pytest.mark.parametrize("batch_x,batch_state", [(1, 1), (4, 1), (4, 4), (1, 4)])
def test_native_lstm_cell_matches_node_by_node_path(batch_x, batch_state, transduce):
    cg_n, out_n = _build(True, batch_x=batch_x, batch_state=batch_state, transduce=transduce)
    cg_p, out_p = _build(False, batch_x=batch_x, batch_state=batch_state, transduce=transduce)
    assert _nodes(cg_n) == _nodes(cg_p)
    if transduce:
        assert [e.index for e in out_n] == [e.index for e in out_p]
    else:
        assert out_n.index == out_p.index
    for a, b in zip(_records(cg_n), _records(cg_p)):
        np.testing.assert_array_equal(a, b)


def test_native_lstm_irregular_inputs_raise_like_ops():
    pools = dy.new_poolset(64, 64, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    b = ops.parameter(cg, model.add_parameters((32,), "b"))
    wx = ops.parameter(cg, model.add_parameters((32, 5), "wx"))
    wh = ops.parameter(cg, model.add_parameters((32, 8), "wh"))
    x = ops.input(cg, dy.Tensor(dy.Shape((6,)), np.zeros(6, np.float32)))  # wrong width
    h = ops.input(cg, dy.Tensor(dy.Shape((8,)), np.zeros(8, np.float32)))
    with pytest.raises(Exception) as native_err:
        cg._core.lstm(b, wx, x, wh, h, h, 8)
    with pytest.raises(Exception) as ops_err:
        ops.affine(b, wx, x, wh, h)
    assert type(native_err.value) is type(ops_err.value)


def test_native_lstm_rejects_stale_expressions():
    pools = dy.new_poolset(64, 64, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    b = ops.parameter(cg, model.add_parameters((32,), "b"))
    cg.renew()
    with pytest.raises(dy.errors.StaleExpression):
        cg._core.lstm(b, b, b, b, b, b, 8)


def test_int_tuple_is_tuple_map_int():
    assert int_tuple([1, 2, 3]) == (1, 2, 3)
    assert int_tuple((1, 2.0, np.int64(3))) == (1, 2, 3)
    assert all(type(v) is int for v in int_tuple(np.arange(5)))
    t = (4, 5)
    assert int_tuple(t) is t
    assert int_tuple(()) == ()
    with pytest.raises(ValueError):
        int_tuple(["x"])


def _small_graph():
    pools = dy.new_poolset(64, 64, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    E = model.add_lookup_parameters(12, 5)
    W = model.add_parameters((7, 10), "W")
    a, b = ops.lookup(cg, E, 3), ops.lookup(cg, E, 11)
    z = ops.matmul(ops.parameter(cg, W), ops.concatenate([a, b]))
    loss = ops.pickneglogsoftmax(z, 4)
    bz = ops.concatenate([ops.lookup_batch(cg, E, [1, 2]), ops.lookup_batch(cg, E, [3, 4])])
    return cg, loss, bz


@pytest.mark.parametrize("kinds", [("lookup",), ("concatenate",), ("pickneglogsoftmax",)])
def test_native_fast_kinds_match_python_rules(kinds):
    from paper_1701_03980_b200 import ops as ops_mod

    cg_n, _, _ = _small_graph()
    saved = {k: ops_mod.FAST_KINDS.pop(k) for k in kinds}
    try:
        cg_p, _, _ = _small_graph()
    finally:
        ops_mod.FAST_KINDS.update(saved)
    assert _nodes(cg_n) == _nodes(cg_p)
    for a, b in zip(_records(cg_n), _records(cg_p)):
        np.testing.assert_array_equal(a, b)


def test_native_fast_kinds_raise_reference_errors():
    pools = dy.new_poolset(64, 64, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    E = model.add_lookup_parameters(4, 3)
    with pytest.raises(dy.errors.IndexOutOfBounds):
        ops.lookup(cg, E, 4)
    x = ops.lookup(cg, E, 1)
    with pytest.raises(dy.errors.IndexOutOfBounds):
        ops.pickneglogsoftmax(x, 3)
    xb = ops.lookup_batch(cg, E, [0, 1])
    with pytest.raises(dy.errors.ShapeError):
        ops.concatenate([x, xb])


def _tree_graph(native):
    from paper_1701_03980_b200 import workloads as W

    pools = dy.new_poolset(64, 64, 64)
    cg, model = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    td = W.tree_corpus(3, 2, vocab=50)
    enc = dy.TreeLSTM(model, {f"w{i}": i for i in range(50)}, 6, 5, "enc")
    saved = cg._core
    if not native:
        cg._core = None
    try:
        outs = [enc.encode(cg, W.to_treenode(dy, t)) for t in td.trees]
    finally:
        cg._core = saved
    return cg, outs


def test_native_tree_lstm_matches_node_by_node_path():
    cg_n, out_n = _tree_graph(True)
    cg_p, out_p = _tree_graph(False)
    assert _nodes(cg_n) == _nodes(cg_p)
    assert [(h.index, c.index) for h, c in out_n] == [(h.index, c.index) for h, c in out_p]
    for a, b in zip(_records(cg_n), _records(cg_p)):
        np.testing.assert_array_equal(a, b)
