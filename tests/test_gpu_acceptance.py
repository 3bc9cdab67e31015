"""Reference acceptance criteria re-run on the CUDA executor (fp32 ports of
pkg/tests/test_acceptance.py): C2 minibatch equivalence (:273-316) and C4
arena behaviour / flat memory over 10k graphs (:393-438)."""

import gc
import tracemalloc

import numpy as np
import pytest

import paper_1701_03980_b200 as dc
from paper_1701_03980_b200 import RNNBuilder, ops
from paper_1701_03980_b200.errors import PoolExhausted
from paper_1701_03980_b200.tensor import Shape, Tensor

pytestmark = pytest.mark.gpu


def make_ctx(mb=8.0, seed=1):
    pools = dc.new_poolset(mb, mb, mb)
    return dc.ComputationGraph(pools), dc.Model(pools, seed=seed)


def pairclass_scores(cg, W, b, E, i1, i2):
    """bench/tasks.py:273-282."""
    x = ops.concatenate([ops.lookup(cg, E, i1), ops.lookup(cg, E, i2)])
    return ops.softmax(ops.add(ops.matmul(ops.parameter(cg, W), x), ops.parameter(cg, b)))


def pairclass_batch_loss(cg, W, b, E, ids1, ids2, labels):
    """bench/tasks.py:285-291."""
    we, be = ops.parameter(cg, W), ops.parameter(cg, b)
    x = ops.concatenate([ops.lookup_batch(cg, E, ids1), ops.lookup_batch(cg, E, ids2)])
    return ops.sum_batches(ops.pickneglogsoftmax_batch(ops.softmax(ops.add(ops.matmul(we, x), be)), labels))


def rnnlm_sentence_nll(cg, rnn, E, W, b, ids):
    """bench/tasks.py:411-420."""
    we, be = ops.parameter(cg, W), ops.parameter(cg, b)
    state, loss = rnn.initial_state(cg), None
    for t in range(len(ids) - 1):
        state = state.add_input(ops.lookup(cg, E, ids[t]))
        step = ops.pickneglogsoftmax(ops.affine(be, we, state.output()), ids[t + 1])
        loss = step if loss is None else ops.add(loss, step)
    return loss


def rnnlm_batch_nll(cg, rnn, E, W, b, batch_ids, pad_id):
    """bench/tasks.py:423-440."""
    we, be = ops.parameter(cg, W), ops.parameter(cg, b)
    t_max = max(len(ids) for ids in batch_ids)
    state, loss = rnn.initial_state(cg), None
    for t in range(t_max - 1):
        xs = [ids[t] if t < len(ids) else pad_id for ids in batch_ids]
        labels = [ids[t + 1] if t + 1 < len(ids) else pad_id for ids in batch_ids]
        mask = np.array([1.0 if t + 1 < len(ids) else 0.0 for ids in batch_ids], dtype=np.float32)
        state = state.add_input(ops.lookup_batch(cg, E, xs))
        nll = ops.pickneglogsoftmax_batch(ops.affine(be, we, state.output()), labels)
        step = ops.sum_batches(ops.cmult(nll, ops.input(cg, Tensor(Shape((1,), len(batch_ids)), mask))))
        loss = step if loss is None else ops.add(loss, step)
    return loss


def test_c2_minibatch_equivalence():
    rng = np.random.default_rng(11)
    cg, model = make_ctx(seed=3)
    W = model.add_parameters((4, 12), "W")
    b = model.add_parameters((4,), "b")
    E = model.add_lookup_parameters(9, 6, "E")
    ex = [(int(rng.integers(0, 9)), int(rng.integers(0, 9)), int(rng.integers(0, 4))) for _ in range(16)]
    for bs in (1, 4, 16):
        batch = ex[:bs]
        cg.renew()
        batched = float(cg.value(pairclass_batch_loss(cg, W, b, E, [e[0] for e in batch], [e[1] for e in batch],
                                                      [e[2] for e in batch])).data[0])
        summed = 0.0
        for i1, i2, lab in batch:
            cg.renew()
            summed += float(cg.value(ops.pickneglogsoftmax(pairclass_scores(cg, W, b, E, i1, i2), lab)).data[0])
        assert abs(batched - summed) <= 1e-5 * max(1.0, abs(summed)), (bs, batched, summed)

    for cell, layers in (("lstm", 1), ("lstm", 2), ("gru", 1)):
        cg2, model2 = make_ctx(seed=4)
        E2 = model2.add_lookup_parameters(7, 5, "E")
        rnn = RNNBuilder(model2, layers, 5, 6, cell, "rnn")
        W2 = model2.add_parameters((7, 6), "W")
        b2 = model2.add_parameters((7,), "b")
        sents = [[int(i) for i in rng.integers(0, 7, size=int(rng.integers(2, 9)))] for _ in range(5)]
        cg2.renew()
        batched = float(cg2.value(rnnlm_batch_nll(cg2, rnn, E2, W2, b2, sents, pad_id=0)).data[0])
        summed = 0.0
        for ids in sents:
            cg2.renew()
            summed += float(cg2.value(rnnlm_sentence_nll(cg2, rnn, E2, W2, b2, ids)).data[0])
        assert abs(batched - summed) <= 1e-5 * max(1.0, abs(summed)), (cell, layers, batched, summed)


def test_c4_arena_flat_memory_over_10k_graphs():
    """Construction claims nothing from the pools; forward claims 99 slots for
    100 nodes (one parameter alias); 10,000 build/evaluate/discard cycles keep
    host memory (tracemalloc) and device memory (torch allocator, the
    executor's cudaMalloc'd caches via cudaMemGetInfo) flat; exhaustion raises
    PoolExhausted naming --mem."""
    import torch

    pools = dc.new_poolset(4, 4, 4)
    cg = dc.ComputationGraph(pools)
    model = dc.Model(pools, seed=1)
    p = model.add_parameters((8,), "p")

    def build_100_nodes():
        e = ops.parameter(cg, p)
        for _ in range(99):
            e = ops.tanh(e)
        return e

    cg.renew()
    before = (pools.forward.alloc_count, pools.backward.alloc_count, pools.parameters.alloc_count)
    tip = build_100_nodes()
    assert len(cg.nodes) == 100
    assert before == (pools.forward.alloc_count, pools.backward.alloc_count, pools.parameters.alloc_count)
    cg.value(tip)
    assert pools.forward.alloc_count == before[0] + 99

    for _ in range(200):
        cg.renew()
        cg.value(build_100_nodes())
    torch.cuda.synchronize()
    gc.collect()
    dev_free0 = torch.cuda.mem_get_info()[0]
    torch_alloc0 = torch.cuda.memory_allocated()
    tracemalloc.start()
    cg.renew()
    cg.value(build_100_nodes())
    base = tracemalloc.get_traced_memory()[0]
    for _ in range(9_800):
        cg.renew()
        cg.value(build_100_nodes())
    final = tracemalloc.get_traced_memory()[0]
    tracemalloc.stop()
    torch.cuda.synchronize()
    assert final - base < 256 * 1024, f"host memory grew by {final - base} bytes"
    assert torch.cuda.memory_allocated() == torch_alloc0
    assert dev_free0 - torch.cuda.mem_get_info()[0] < 4 * 1024 * 1024, "device memory grew"

    tiny = dc.new_poolset(0.001, 0.001, 0.5)
    cg2 = dc.ComputationGraph(tiny)
    big = ops.input(cg2, dc.from_values(dc.Shape((4096,)), np.zeros(4096)))
    with pytest.raises(PoolExhausted, match="--mem"):
        cg2.value(big)
