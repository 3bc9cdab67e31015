"""Host-only checks of the native planner (dg_schedule_stats): gated-cell
fusion, add-chain rewrite and signature batching on the BASELINE workloads.
No device memory is touched: parameters get placeholder handles and the graph
arenas are dummy addresses that the planner never dereferences."""

import ctypes

import numpy as np

import paper_1701_03980_b200 as dy
from paper_1701_03980_b200 import _native
from paper_1701_03980_b200 import workloads as W

KEYS = ["units", "groups", "cells", "chains", "cell_nodes", "max_group", "lookups", "inputs"]


def _stats(cg, model):
    lib = _native.lib()
    for x in list(model.parameters) + list(model.lookups):
        if x.handle < 0:
            h = ctypes.c_int64(-1)
            is_lp = hasattr(x, "rows")
            rows, cols = (x.rows, x.dim) if is_lp else (x.size, 1)
            _native.check(lib.dg_param_register(int(is_lp), rows, cols, 0x100, 0x200, ctypes.byref(h)))
            x.handle = h.value
    h = ctypes.c_void_p()
    _native.check(lib.dg_graph_create(0, 0x1000, 1 << 30, 0x2000, 1 << 30, 0x3000, 1 << 28, ctypes.byref(h)))
    cg._sent = 0
    cg._flush(h)
    out = np.zeros(8, np.int64)
    _native.check(lib.dg_schedule_stats(h, 0, len(cg.nodes) - 1, out.ctypes.data))
    lib.dg_graph_destroy(h)
    return dict(zip(KEYS, out.tolist()))


def _ctx():
    pools = dy.new_poolset(64, 64, 64)
    return dy.ComputationGraph(pools), dy.Model(pools, seed=1)


def test_rnnlm_cells_fused_and_loss_chain_rewritten():
    cg, m = _ctx()
    task = W.RNNLM(dy, m, 10_000, 128, 256, 2)
    batch = W.ptb_corpus(1, 64)
    task.loss(cg, batch)
    steps = max(len(s) for s in batch) - 1
    s = _stats(cg, m)
    assert s["cells"] == 2 * steps  # every LSTM layer-step is one fused cell
    assert s["cell_nodes"] == 13 * 2 * steps  # 13 nodes per LSTM cell
    assert s["chains"] == 1  # the scalar loss chain becomes one prefix sum
    # recurrence levels x (2 affines + 1 cell group) + a constant output stage:
    # the output affine / pnls / masks batch across all time steps
    assert s["groups"] <= 3 * (steps + 1) + 8
    assert s["max_group"] >= steps  # output-layer nodes of every step in one group


def test_tree_lstm_batches_by_height():
    cg, m = _ctx()
    td = W.tree_corpus(1, 1)
    task = W.TreeClassifier(dy, m, td.vocab_size)
    task.loss(cg, td.trees[0], td.labels[0])
    n_leaves = W.count_leaves(td.trees[0])
    s = _stats(cg, m)
    assert s["cells"] == 2 * n_leaves - 1  # leaves (m=0) + internal nodes (m=2)
    assert s["chains"] == 0
    # all leaf cells batch into one group; internal nodes batch per level
    assert s["max_group"] >= n_leaves
    assert s["groups"] <= 2 * n_leaves


def test_tagger_char_cells():
    cg, m = _ctx()
    tg = W.tagger_corpus(1, 50, n_types=4000)
    task = W.CharTagger(dy, m, tg)
    sent = tg.sentences[0]
    task.loss(cg, sent)
    s = _stats(cg, m)
    rare = [w for w, _ in sent if w not in tg.vocab]
    expect = 2 * len(sent) + sum(2 * len(w) for w in rare)
    assert s["cells"] == expect


def _rnn_stats(cg, model):
    lib = _native.lib()
    _stats(cg, model)  # registers placeholder parameters
    h = ctypes.c_void_p()
    _native.check(lib.dg_graph_create(0, 0x1000, 1 << 30, 0x2000, 1 << 30, 0x3000, 1 << 28, ctypes.byref(h)))
    cg._sent = 0
    cg._flush(h)
    out = np.zeros(4, np.int64)
    _native.check(lib.dg_schedule_rnn_stats(h, 0, len(cg.nodes) - 1, out.ctypes.data))
    lib.dg_graph_destroy(h)
    return dict(zip(["stacks", "chains", "steps", "ctas"], out.tolist()))


def test_rnnlm_recurrence_is_one_persistent_chain_per_layer():
    cg, m = _ctx()
    task = W.RNNLM(dy, m, 10_000, 128, 256, 2)
    batch = W.ptb_corpus(1, 64)
    task.loss(cg, batch)
    steps = max(len(s) for s in batch) - 1
    r = _rnn_stats(cg, m)
    # one persistent chain per layer (input projections are batched GEMMs
    # between them): 64 rows / 16 per CTA x 256 units / 16 per CTA = 64 CTAs each
    assert r == {"stacks": 2, "chains": 2, "steps": 2 * steps, "ctas": 128}


def test_tiny_lm_single_chain():
    cg, m = _ctx()
    task = W.RNNLM(dy, m, 1000, 64, 64, 1)
    sent = W.tiny_lm_corpus(5, 1)[0]
    task.loss(cg, [sent])
    r = _rnn_stats(cg, m)
    assert r["stacks"] == 1 and r["chains"] == 1 and r["steps"] == len(sent) - 1
    assert r["ctas"] == 4


def test_tree_has_no_chains():
    cg, m = _ctx()
    td = W.tree_corpus(1, 1)
    task = W.TreeClassifier(dy, m, td.vocab_size)
    task.loss(cg, td.trees[0], td.labels[0])
    assert _rnn_stats(cg, m)["stacks"] == 0
