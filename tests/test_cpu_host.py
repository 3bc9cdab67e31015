"""CPU-side checks: the C-ABI library loads and exports every symbol declared
in include/dyngpu.h; graph construction keeps the reference's host contract
(shape errors at construction, staleness, generations, pool accounting); and
execution without a GPU fails loudly instead of falling back to the CPU."""

import os
import re

import numpy as np
import pytest

import paper_1701_03980_b200 as dc
from paper_1701_03980_b200 import _native, ops
from paper_1701_03980_b200.errors import (
    BadShape,
    ConfigError,
    EmptyBatch,
    EmptyList,
    IndexOutOfBounds,
    LengthMismatch,
    PoolExhausted,
    ShapeError,
    StaleExpression,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def make_ctx(mb=4.0, seed=1):
    pools = dc.new_poolset(mb, mb, mb)
    return dc.ComputationGraph(pools), dc.Model(pools, seed=seed)


def vec(values, batch=1):
    return dc.from_values(dc.Shape((len(values) // batch,), batch), values)


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "dyngpu.h")).read()
    declared = sorted(set(re.findall(r"^(?:int|const char\*)\s+(dg_\w+)\(", header, re.M)))
    assert len(declared) >= 30
    lib = _native.lib()
    missing = [name for name in declared if not hasattr(lib, name)]
    assert not missing, missing
    assert set(_native.EXPORTS) <= set(declared)
    assert lib.dg_abi_version() == 1


def test_op_codes_match_header():
    header = open(os.path.join(ROOT, "include", "dyngpu.h")).read()
    for kind, code in _native.OP_CODES.items():
        assert code < 17
    assert "DG_OP_SUM_BATCHES = 16" in header
    assert _native.NODE_DTYPE.itemsize == 13 * 4


def test_generation_staleness_and_nodes():
    cg, _ = make_ctx()
    assert cg.generation == 0
    x = ops.input(cg, vec([1.0, 2.0]))
    assert len(cg.nodes) == 1
    cg.renew()
    assert cg.generation == 1 and cg.nodes == [] and cg.watermark == -1
    with pytest.raises(StaleExpression):
        ops.tanh(x)


def test_shape_errors_at_construction_without_numeric_work():
    cg, model = make_ctx()
    x = ops.input(cg, vec([1.0, 2.0, 3.0]))
    assert ops.tanh(x).shape.dims == (3,)
    A = model.add_parameters((2, 3), "A")
    with pytest.raises(ShapeError, match="matmul"):
        ops.matmul(ops.parameter(cg, A), ops.input(cg, vec([1.0] * 4)))
    with pytest.raises(ShapeError, match="affine"):
        ops.affine(ops.parameter(cg, A))
    with pytest.raises(ShapeError):
        ops.add(x, ops.input(cg, vec([1.0, 2.0])))
    with pytest.raises(ShapeError):
        ops.add(ops.input(cg, vec([1.0] * 6, 2)), ops.input(cg, vec([1.0] * 9, 3)))
    with pytest.raises(ShapeError):
        ops.pick_range(x, 2, 5)
    with pytest.raises(IndexOutOfBounds):
        ops.pickneglogsoftmax(x, 3)
    with pytest.raises(BadShape):
        ops.pickneglogsoftmax(ops.input(cg, vec([1.0] * 6, 2)), 0)
    with pytest.raises(LengthMismatch):
        ops.pickneglogsoftmax_batch(ops.input(cg, vec([1.0] * 6, 2)), [0])
    E = model.add_lookup_parameters(5, 2, "E")
    with pytest.raises(IndexOutOfBounds):
        ops.lookup(cg, E, 5)
    with pytest.raises(EmptyBatch):
        ops.lookup_batch(cg, E, [])
    with pytest.raises(EmptyList):
        ops.concatenate([])
    assert cg.watermark == -1 and cg.forward_calls == 0


def test_affine_shape_rule_broadcast():
    cg, model = make_ctx()
    W = model.add_parameters((4, 3), "W")
    b = model.add_parameters((4,), "b")
    x = ops.input(cg, vec([1.0] * 6, 2))
    y = ops.affine(ops.parameter(cg, b), ops.parameter(cg, W), x)
    assert y.shape == dc.Shape((4,), 2)


def test_parameter_init_matches_reference_rng():
    _, m = make_ctx(seed=3)
    p = m.add_parameters((4, 5), "p")
    rng = np.random.default_rng(3)
    expect = rng.uniform(-np.sqrt(6.0 / 9), np.sqrt(6.0 / 9), 20).astype(np.float32)
    assert np.array_equal(p.values.data, expect)
    lp = m.add_lookup_parameters(3, 2, "E")
    assert np.array_equal(lp.values, rng.uniform(-0.1, 0.1, (3, 2)).astype(np.float32))


def test_lstm_builder_zeroes_forget_bias_and_names():
    _, m = make_ctx()
    rnn = dc.RNNBuilder(m, 2, 3, 4, "lstm", "rnn")
    names = [p.name for p in m.parameters]
    assert names == ["rnn.l0.Wx", "rnn.l0.Wh", "rnn.l0.b", "rnn.l1.Wx", "rnn.l1.Wh", "rnn.l1.b"]
    assert np.all(rnn.params[0][2].values.data[4:8] == 0)


def test_parameter_pool_accounting_and_exhaustion():
    pools = dc.new_poolset(1, 1, 0.001)
    m = dc.Model(pools)
    m.add_parameters((10,))
    assert pools.parameters.alloc_count == 2
    assert pools.parameters.cursor == 128
    with pytest.raises(PoolExhausted):
        m.add_parameters((1000,))


def test_float64_pools_rejected():
    with pytest.raises(ConfigError):
        dc.new_poolset(1, 1, 1, dtype=np.float64)


def test_mem_flag_split():
    p = dc.poolset_from_mem_flag("3")
    assert p.forward.capacity == p.backward.capacity == p.parameters.capacity == 1 << 20


def test_execution_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cg, _ = make_ctx()
    x = ops.tanh(ops.input(cg, vec([1.0])))
    with pytest.raises(ConfigError, match="no CPU fallback"):
        cg.value(x)


def test_tree_node_validation():
    with pytest.raises(BadShape):
        dc.TreeNode(token="a", children=(dc.TreeNode.leaf("b"),))
    with pytest.raises(BadShape):
        dc.TreeNode()


def test_opdef_reference_positional_order():
    """The reference plug-in contract OpDef(name, shape, forward, backward,
    alias, flush) (pkg/src/dyncore/ops.py:33-40) constructs positionally;
    re-registering a built-in kind keeps its native kernel and encoding, and
    its Python shape rule runs at construction."""
    calls = []
    orig = ops.get_op("tanh")

    def shape(aux, in_shapes):
        calls.append(in_shapes[0])
        return in_shapes[0]

    def fwd(out, ins, aux):
        raise AssertionError("never called: the kernel is native")

    od = ops.OpDef("tanh", shape, fwd, None, None, None)
    assert od.forward is fwd and od.backward is None and od.encode is None
    try:
        reg = ops.register(od)
        assert reg.code == orig.code and reg.encode is orig.encode and reg.forward is fwd
        cg, _ = make_ctx()
        y = ops.tanh(ops.input(cg, vec([0.5, -0.5])))
        assert len(calls) == 1 and cg.nodes[y.index].shape.dims == (2,)
    finally:
        ops.REGISTRY["tanh"] = orig
        ops.FAST_KINDS["tanh"] = orig.code


def test_python_only_op_is_a_config_error():
    """No CPU execution path: a kind with only Python forward/backward raises
    the reference taxonomy's ConfigError at registration, not TypeError."""
    od = ops.OpDef("my_square", lambda aux, s: s[0], lambda out, ins, aux: None,
                   lambda i, g, iv, ov, og, aux: None)
    with pytest.raises(ConfigError):
        ops.register(od)
    assert "my_square" not in ops.REGISTRY
