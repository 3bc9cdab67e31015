"""Reference test semantics re-run on the CUDA executor (fp32 variants of
pkg/tests/test_graph.py, test_ops.py, test_trainers.py, test_params.py)."""

import math

import numpy as np
import pytest

import paper_1701_03980_b200 as dc
from paper_1701_03980_b200 import ops
from paper_1701_03980_b200.errors import NonScalarLoss, PoolExhausted, StaleExpression
from tests.helpers import gpu_ctx

pytestmark = pytest.mark.gpu


def make_ctx(mb=4.0, seed=1, init_zero=False):
    pools = dc.new_poolset(mb, mb, mb)
    return dc.ComputationGraph(pools), dc.Model(pools, seed=seed, init_zero=init_zero)


def vec(values, batch=1):
    return dc.from_values(dc.Shape((len(values) // batch,), batch), values)


# -- graph semantics (tests/test_graph.py) ----------------------------------


def test_input_value_and_defensive_copy():
    cg, _ = make_ctx()
    x = ops.input(cg, vec([1.0, 2.0]))
    kept = cg.value(x)
    cg.renew()
    assert np.allclose(kept.data, [1, 2])
    with pytest.raises(StaleExpression):
        cg.value(x)


def test_incremental_forward_never_recomputes():
    cg, _ = make_ctx()
    x = ops.input(cg, vec([1.0, 2.0]))
    cg.value(x)
    calls = cg.forward_calls
    y = ops.tanh(x)
    assert np.allclose(cg.value(y).data, np.tanh([1.0, 2.0]), atol=1e-6)
    assert cg.forward_calls == calls + 1
    cg.value(y)
    assert cg.forward_calls == calls + 1


def test_forward_to_and_watermark():
    cg, _ = make_ctx()
    x = ops.input(cg, vec([0.5]))
    y = ops.logistic(x)
    z = ops.tanh(y)
    cg.forward_to(y)
    assert cg.watermark == y.index
    assert cg.forward_calls == 2
    assert np.allclose(cg.value(z).data, np.tanh(1 / (1 + np.exp(-0.5))), atol=1e-6)


def test_non_scalar_loss():
    cg, _ = make_ctx()
    with pytest.raises(NonScalarLoss):
        cg.backward(ops.input(cg, vec([1.0, 2.0])))


def test_two_backward_calls_accumulate_twice():
    cg, model = make_ctx()
    p = model.add_parameters((2,), "p")
    p.set_value([1.0, 2.0])
    pe = ops.parameter(cg, p)
    loss = ops.matmul(ops.input(cg, dc.from_values(dc.Shape((1, 2)), [1.0, 1.0])), ops.cmult(pe, pe))
    cg.backward(loss)
    g1 = p.gradient.data.copy()
    cg.backward(loss)
    assert np.allclose(p.gradient.data, 2 * g1)
    assert np.allclose(g1, [2.0, 4.0])


def test_pnls_gradient_known_answer():
    cg, model = make_ctx()
    x = ops.input(cg, vec([0.0, 0.0]))
    loss = ops.pickneglogsoftmax(x, 0)
    cg.backward(loss)
    assert np.allclose(cg.value(loss).data, [math.log(2)], atol=1e-6)
    assert np.allclose(cg.gradient(x).data, [-0.5, 0.5], atol=1e-6)


def test_shared_node_sums_both_branches():
    cg, model = make_ctx()
    x = ops.input(cg, vec([0.3, -0.7]))
    t = ops.tanh(x)
    s = ops.add(t, t)
    loss = ops.matmul(ops.input(cg, dc.from_values(dc.Shape((1, 2)), [1.0, 1.0])), s)
    cg.backward(loss)
    expect = 2 * (1 - np.tanh([0.3, -0.7]) ** 2)
    assert np.allclose(cg.gradient(x).data, expect, atol=1e-6)


def test_pool_exhausted_and_alloc_counts():
    cg, model = make_ctx(mb=0.01)
    x = ops.input(cg, vec([1.0] * 1000, 4))
    with pytest.raises(PoolExhausted):
        cg.value(ops.tanh(ops.tanh(ops.tanh(x))))


def test_forward_alloc_count_100_nodes_one_alias():
    # acceptance C4 (tests/test_acceptance.py:408-415): +99 allocations for a
    # 100-node graph whose first node is a parameter alias
    cg, model = make_ctx()
    p = model.add_parameters((4,), "p")
    before = cg.pools.forward.alloc_count
    e = ops.parameter(cg, p)
    for _ in range(99):
        e = ops.tanh(e)
    cg.value(e)
    assert cg.pools.forward.alloc_count - before == 99
    assert cg.forward_calls == 100


# -- ops known answers (tests/test_ops.py) ----------------------------------


def test_op_known_answers():
    cg, model = make_ctx()
    a = ops.input(cg, vec([1.0, 2.0, 3.0, 4.0], 2))
    b = ops.input(cg, vec([10.0, 10.0]))
    assert np.allclose(cg.value(ops.add(a, b)).data, [11, 12, 13, 14])
    A = model.add_parameters((2, 2), "A")
    A.set_value(np.array([[1.0, 2.0], [3.0, 4.0]]).reshape(-1, order="F"))
    y = ops.matmul(ops.parameter(cg, A), ops.input(cg, vec([1.0, 1.0])))
    assert np.allclose(cg.value(y).data, [3, 7])
    assert np.allclose(cg.value(ops.logistic(ops.input(cg, vec([0.0])))).data, [0.5])
    assert np.allclose(cg.value(ops.tanh(ops.input(cg, vec([1.0])))).data, [0.7615941559557649], atol=1e-6)
    sm = ops.softmax(ops.input(cg, vec([1000.0, 1000.0])))
    assert np.allclose(cg.value(sm).data, [0.5, 0.5])
    assert cg.value(ops.pickneglogsoftmax(ops.input(cg, vec([50.0, 0.0])), 0)).data[0] < 1e-6
    s = ops.sum_batches(ops.input(cg, vec([1.0, 2.0, 3.0], 3)))
    assert np.allclose(cg.value(s).data, [6.0])


def test_touched_only_looked_up_rows():
    cg, model = make_ctx()
    E = model.add_lookup_parameters(4, 3, "E")
    x = ops.lookup(cg, E, 1)
    loss = ops.pickneglogsoftmax(x, 0)
    cg.backward(loss)
    assert E.touched == {1}
    g = E.gradient
    assert np.all(g[[0, 2, 3]] == 0)


def test_touched_includes_non_ancestors_excludes_later():
    cg, model = make_ctx()
    E = model.add_lookup_parameters(10, 3, "E")
    a = ops.lookup(cg, E, 2)
    ops.lookup(cg, E, 7)  # not an ancestor of the loss, still touched
    loss = ops.pickneglogsoftmax(a, 1)
    ops.lookup(cg, E, 9)  # created after the loss: not touched
    cg.backward(loss)
    assert E.touched == {2, 7}
    assert np.all(E.gradient[7] == 0)


def test_lookup_batch_repeated_ids_accumulate():
    cg, model = make_ctx()
    E = model.add_lookup_parameters(5, 2, "E")
    x = ops.lookup_batch(cg, E, [3, 1, 3])
    w = ops.input(cg, vec([1.0, 2.0, 3.0, 4.0, 5.0, 6.0], 3))
    loss = ops.sum_batches(ops.matmul(ops.input(cg, dc.from_values(dc.Shape((1, 2)), [1.0, 1.0])), ops.cmult(x, w)))
    cg.backward(loss)
    g = E.gradient
    assert np.allclose(g[3], [1.0 + 5.0, 2.0 + 6.0])
    assert np.allclose(g[1], [3.0, 4.0])
    assert E.touched == {1, 3}


# -- trainers (tests/test_trainers.py), fp32 --------------------------------


def one_param_model(theta):
    cg, model = make_ctx(init_zero=True)
    p = model.add_parameters((len(theta),), "p")
    p.set_value(theta)
    return cg, model, p


def test_sgd_step():
    _, model, p = one_param_model([1.0, 1.0])
    tr = dc.Trainer(model, "sgd", lr=0.1)
    p.gradient.data[:] = [0.5, 0.0]
    tr.update()
    assert np.allclose(p.values.data, [0.95, 1.0])
    assert np.all(p.gradient.data == 0)


def test_adagrad_step():
    _, model, p = one_param_model([0.0])
    tr = dc.Trainer(model, "adagrad", lr=1.0, adagrad_eps=0.0)
    p.gradient.data[:] = [3.0]
    tr.update()
    assert np.allclose(tr.sq[id(p)], [9.0])
    assert np.allclose(p.values.data, [-1.0])


def test_adam_first_step():
    _, model, p = one_param_model([0.0])
    tr = dc.Trainer(model, "adam")
    p.gradient.data[:] = [1.0]
    tr.update()
    assert np.isclose(p.values.data[0], -0.000999999995, atol=1e-9)
    assert tr.t == 1


def test_momentum_step():
    _, model, p = one_param_model([0.0])
    tr = dc.Trainer(model, "momentum", lr=0.1, momentum=0.9)
    p.gradient.data[:] = [1.0]
    tr.update()
    assert np.allclose(tr.vel[id(p)], [-0.1])
    assert np.allclose(p.values.data, [-0.1])


def test_sgd_half_norm_halves_exactly():
    cg, model = make_ctx(init_zero=True)
    p = model.add_parameters((3,), "p")
    theta0 = np.array([0.7, -1.3, 2.9], dtype=np.float32)
    p.set_value(theta0)
    ones_row = dc.from_values(dc.Shape((1, 3)), [1.0, 1.0, 1.0])
    pe = ops.parameter(cg, p)
    loss = ops.scalar_mul(ops.matmul(ops.input(cg, ones_row), ops.cmult(pe, pe)), 0.5)
    cg.backward(loss)
    assert np.allclose(p.gradient.data, theta0)
    dc.Trainer(model, "sgd", lr=0.5).update()
    assert np.array_equal(p.values.data, theta0 * np.float32(0.5))


def _train_lookup(rule, sparse, steps):
    cg, model = make_ctx(seed=4)
    E = model.add_lookup_parameters(2, 2, "E")
    tr = dc.Trainer(model, rule, sparse=sparse)
    for rows in steps:
        cg.renew()
        loss = None
        for row in rows:
            term = ops.pickneglogsoftmax(ops.lookup(cg, E, row), row % 2)
            loss = term if loss is None else ops.add(loss, term)
        cg.backward(loss)
        tr.update()
    return E.values.copy()


@pytest.mark.parametrize("rule", ["sgd", "adagrad"])
def test_sparse_dense_equivalence(rule):
    steps = [(0, 1), (0,), (0, 0, 1), (1,)]
    assert np.allclose(_train_lookup(rule, False, steps), _train_lookup(rule, True, steps), atol=1e-6)


@pytest.mark.parametrize("rule", ["adam", "momentum"])
def test_sparse_freezes_untouched_rows(rule):
    steps = [(0, 1), (0,)]
    after1 = _train_lookup(rule, True, steps[:1])
    sparse = _train_lookup(rule, True, steps)
    dense = _train_lookup(rule, False, steps)
    assert np.array_equal(sparse[1], after1[1])
    assert not np.array_equal(dense[1], after1[1])


def test_update_clears_touched():
    cg, model = make_ctx()
    E = model.add_lookup_parameters(3, 2, "E")
    tr = dc.Trainer(model, "sgd")
    cg.backward(ops.pickneglogsoftmax(ops.lookup(cg, E, 2), 0))
    assert E.touched == {2}
    tr.update()
    assert E.touched == set()
    assert np.all(E.gradient == 0)


def test_adam_kernel_matches_oracle_on_injected_gradients():
    """Adam in isolation: identical gradients into both sides, 5 steps."""
    from oracle import engine as orc

    rng = np.random.default_rng(0)
    grads = [rng.standard_normal(257).astype(np.float32) for _ in range(5)]
    _, model, p = one_param_model(np.zeros(257))
    tr = dc.Trainer(model, "adam")
    om = orc.Model(orc.new_poolset(), init_zero=True)
    op = om.add_parameters((257,), "p")
    otr = orc.Trainer(om, "adam")
    for g in grads:
        p.gradient.data[:] = g
        tr.update()
        op.gradient[:] = g
        otr.update()
    assert np.allclose(p.values.data, op.values, rtol=1e-5, atol=1e-8)


# -- persistence (tests/test_params.py) --------------------------------------


def test_dyn1_roundtrip(tmp_path):
    dy, cg, model = gpu_ctx(seed=3, mb=8)
    W_ = model.add_parameters((3, 4), "W")
    E = model.add_lookup_parameters(5, 2, "E")
    tr = dy.Trainer(model, "sgd")
    x = ops.concatenate([ops.lookup(cg, E, 1), ops.lookup(cg, E, 3)])
    loss = ops.pickneglogsoftmax(ops.affine(ops.input(cg, vec([0.0, 0.0, 0.0])), ops.parameter(cg, W_), x), 1)
    before = E.values.copy()
    cg.backward(loss)
    tr.update()
    after = E.values.copy()
    assert not np.array_equal(after[[1, 3]], before[[1, 3]]), "the looked-up rows must have trained"
    assert np.array_equal(np.delete(after, [1, 3], 0), np.delete(before, [1, 3], 0))
    path = str(tmp_path / "m.dyn")
    model.save(path)
    dy2, cg2, m2 = gpu_ctx(seed=99, mb=8)
    m2.add_parameters((3, 4), "W")
    m2.add_lookup_parameters(5, 2, "E")
    m2.load(path)
    assert np.array_equal(m2.parameters[0].values.data, W_.values.data)
    assert np.array_equal(m2.lookups[0].values, E.values)


# -- the reference sink protocol (graph.py:51-66, parallel.py:30-46) ----------


class _SlotsSink:
    """A GradientSlots-style sink (reference parallel.py:30-46)."""

    def __init__(self, model):
        self.params = {id(p): np.zeros(p.size, np.float64) for p in model.parameters}
        self.lookups = {id(lp): np.zeros((lp.rows, lp.dim), np.float64) for lp in model.lookups}
        self.rows_seen = {}

    def add_param_grad(self, p, flat):
        self.params[id(p)] += np.asarray(flat).reshape(-1)

    def add_lookup_row_grad(self, lp, row, vec):
        self.lookups[id(lp)][row] += vec

    def add_lookup_rows_grad(self, lp, ids, rows):
        self.rows_seen.setdefault(id(lp), []).extend(ids)
        np.add.at(self.lookups[id(lp)], list(ids), rows)


def test_custom_sink_receives_the_default_sinks_gradients():
    """cg.sink = <sink object>: the device backward's gradients arrive through
    add_param_grad / add_lookup_rows_grad and the model's own gradients and
    touched sets stay as they were; the same graph under the default sink
    accumulates exactly those gradients into the model."""
    from paper_1701_03980_b200 import workloads as W
    from tests.helpers import pgrad

    sents = W.ptb_corpus(7, 4, vocab=500)
    dy, cg, model = gpu_ctx(seed=5, mb=64)
    task = W.RNNLM(dy, model, 500, 16, 32, 2)

    cg.renew()
    cg.backward(task.loss(cg, sents))
    ref_p = {id(p): pgrad(p) for p in model.parameters}
    ref_l = {id(lp): lp.gradient.astype(np.float64).copy() for lp in model.lookups}
    ref_t = {id(lp): sorted(lp.touched) for lp in model.lookups}
    model.zero_gradients()

    sink = _SlotsSink(model)
    cg.renew()
    cg.sink = sink
    cg.backward(task.loss(cg, sents))
    cg.sink = dc.graph.DIRECT_SINK
    for p in model.parameters:
        assert not pgrad(p).any(), f"{p.name}: model gradient written under a custom sink"
        assert np.allclose(sink.params[id(p)], ref_p[id(p)], rtol=1e-6, atol=1e-9), p.name
    for lp in model.lookups:
        assert not lp.touched and not lp.gradient.any()
        assert sorted(set(sink.rows_seen[id(lp)])) == ref_t[id(lp)]
        assert np.allclose(sink.lookups[id(lp)], ref_l[id(lp)], rtol=1e-6, atol=1e-9)


def test_loss_chain_gradients_are_exactly_one():
    """A left-deep chain of scalar adds (the bench loss, bench/tasks.py:419)
    runs as one prefix-sum unit: d loss / d loss stays the seed 1.0
    (graph.py:151) and every term and intermediate sum gets exactly 1.0.
    Regression: the element-parallel chain backward once also added into the
    final add's own slot (doubling it, and racing with the reads of it)."""
    from paper_1701_03980_b200.graph import Expression

    cg, model = make_ctx(mb=16)
    W = model.add_parameters((6, 4), "W")
    terms = []
    for k in range(40):
        x = ops.input(cg, vec([0.1 * k, -0.2, 0.3, 0.05 * k]))
        terms.append(ops.pickneglogsoftmax(ops.matmul(ops.parameter(cg, W), x), k % 6))
    loss = terms[0]
    sums = []
    for t in terms[1:]:
        loss = ops.add(loss, t)
        sums.append(loss)
    cg.backward(loss)
    assert cg.gradient(loss).data.tolist() == [1.0]
    for e in terms + sums[:-1]:
        assert cg.gradient(e).data.tolist() == [1.0], cg.nodes[e.index].kind
