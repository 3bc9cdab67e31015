"""Engine-agnostic parity cases shared by the golden generator and the tests.

Every builder takes `dy` (a dyncore-shaped namespace: the reference, the CPU
oracle, or the CUDA package), a graph and a model, and returns
(output expression, [expressions whose gradients are recorded]).  Inputs are
seeded, so all engines see identical numbers.  The scalarisation follows the
reference test helper tests/util.py:14-27 (fixed weights, catalog ops only).
"""

from __future__ import annotations

import numpy as np

from paper_1701_03980_b200 import workloads as W

WEIGHTS = np.linspace(0.3, 1.7, 97)


def _vals(seed, n, scale=1.0):
    return (np.random.default_rng(seed).standard_normal(n) * scale).astype(np.float32)


def inp(dy, cg, dims, batch, seed, scale=1.0):
    shape = dy.Shape(dims, batch)
    return dy.ops.input(cg, dy.Tensor(shape, _vals(seed, shape.size(), scale)))


def scalarize(dy, cg, e):
    shape = e.shape
    if shape.batch > 1:
        e = dy.ops.sum_batches(e)
        shape = e.shape
    if len(shape.dims) == 2:
        p = shape.dims[1]
        v = dy.ops.input(cg, dy.Tensor(dy.Shape((p,)), WEIGHTS[:p].astype(np.float32)))
        e = dy.ops.matmul(e, v)
        shape = e.shape
    n = shape.dims[0]
    u = dy.ops.input(cg, dy.Tensor(dy.Shape((1, n)), WEIGHTS[1 : n + 1].astype(np.float32)))
    return dy.ops.matmul(u, e)


def _pair(kind, ba, bb):
    def build(dy, cg, model):
        a = inp(dy, cg, (5,), ba, 1)
        b = inp(dy, cg, (5,), bb, 2)
        return getattr(dy.ops, kind)(a, b), [a, b]

    return build


def _unary(kind, scale=1.0, batch=3):
    def build(dy, cg, model):
        x = inp(dy, cg, (7,), batch, 3, scale)
        return getattr(dy.ops, kind)(x), [x]

    return build


def _scalar_mul(dy, cg, model):
    x = inp(dy, cg, (4,), 2, 4)
    return dy.ops.scalar_mul(x, -1.5), [x]


def _matmul_vec(dy, cg, model):
    A = model.add_parameters((3, 4), "A")
    x = inp(dy, cg, (4,), 3, 5)
    a = dy.ops.parameter(cg, A)
    return dy.ops.matmul(a, x), [a, x]


def _matmul_mat(dy, cg, model):
    A = model.add_parameters((3, 4), "A")
    x = inp(dy, cg, (4, 2), 1, 6)
    a = dy.ops.parameter(cg, A)
    return dy.ops.matmul(a, x), [a, x]


def _matmul_batched(dy, cg, model):
    a = inp(dy, cg, (3, 4), 2, 7)
    x = inp(dy, cg, (4, 2), 2, 8)
    return dy.ops.matmul(a, x), [a, x]


def _affine1(dy, cg, model):
    Wp = model.add_parameters((6, 4), "W")
    bp = model.add_parameters((6,), "b")
    x = inp(dy, cg, (4,), 3, 9)
    w, b = dy.ops.parameter(cg, Wp), dy.ops.parameter(cg, bp)
    return dy.ops.affine(b, w, x), [b, w, x]


def _affine2(dy, cg, model):
    W1 = model.add_parameters((6, 4), "W1")
    W2 = model.add_parameters((6, 3), "W2")
    bp = model.add_parameters((6,), "b")
    x1 = inp(dy, cg, (4,), 2, 10)
    x2 = inp(dy, cg, (3,), 1, 11)  # batch-1 operand broadcast over the batch
    w1, w2, b = dy.ops.parameter(cg, W1), dy.ops.parameter(cg, W2), dy.ops.parameter(cg, bp)
    return dy.ops.affine(b, w1, x1, w2, x2), [b, w1, x1, w2, x2]


def _affine_batched_bias(dy, cg, model):
    Wp = model.add_parameters((5, 4), "W")
    b = inp(dy, cg, (5,), 3, 12)
    x = inp(dy, cg, (4,), 1, 13)
    w = dy.ops.parameter(cg, Wp)
    return dy.ops.affine(b, w, x), [b, w, x]


def _affine_batched_w(dy, cg, model):
    w = inp(dy, cg, (5, 4), 2, 14)
    bp = model.add_parameters((5,), "b")
    x = inp(dy, cg, (4,), 2, 15)
    b = dy.ops.parameter(cg, bp)
    return dy.ops.affine(b, w, x), [b, w, x]


def _concat(dy, cg, model):
    a = inp(dy, cg, (2,), 2, 16)
    b = inp(dy, cg, (3,), 2, 17)
    c = inp(dy, cg, (4,), 2, 18)
    return dy.ops.concatenate([a, b, c]), [a, b, c]


def _pick(dy, cg, model):
    x = inp(dy, cg, (9,), 2, 19)
    return dy.ops.pick_range(x, 2, 7), [x]


def _pnls(dy, cg, model):
    x = inp(dy, cg, (11,), 1, 20, 3.0)
    return dy.ops.pickneglogsoftmax(x, 4), [x]


def _pnls_batch(dy, cg, model):
    x = inp(dy, cg, (13,), 4, 21, 3.0)
    return dy.ops.pickneglogsoftmax_batch(x, [0, 12, 5, 5]), [x]


def _sum_batches(dy, cg, model):
    x = inp(dy, cg, (6,), 4, 22)
    return dy.ops.sum_batches(x), [x]


def _lookup(dy, cg, model):
    E = model.add_lookup_parameters(10, 6, "E")
    a = dy.ops.lookup(cg, E, 3)
    b = dy.ops.lookup(cg, E, 7)
    return dy.ops.cmult(a, b), [a, b]


def _lookup_batch(dy, cg, model):
    E = model.add_lookup_parameters(10, 6, "E")
    a = dy.ops.lookup_batch(cg, E, [1, 4, 1, 9])  # repeated id accumulates
    x = inp(dy, cg, (6,), 4, 23)
    return dy.ops.cmult(a, x), [a, x]


def _chain(dy, cg, model):
    """A tiny composite: shared node used twice, add chain, tanh/logistic."""
    Wp = model.add_parameters((4, 4), "W")
    bp = model.add_parameters((4,), "b")
    x = inp(dy, cg, (4,), 2, 24)
    w, b = dy.ops.parameter(cg, Wp), dy.ops.parameter(cg, bp)
    h = dy.ops.tanh(dy.ops.affine(b, w, x))
    h2 = dy.ops.logistic(dy.ops.affine(b, w, h))
    s = dy.ops.add(dy.ops.add(h, h2), dy.ops.cmult(h, h2))
    return s, [x, h, h2]


OP_CASES = {
    "add": _pair("add", 2, 2),
    "add_bcast_a": _pair("add", 1, 3),
    "add_bcast_b": _pair("add", 3, 1),
    "cmult": _pair("cmult", 2, 2),
    "cmult_bcast_a": _pair("cmult", 1, 3),
    "cmult_bcast_b": _pair("cmult", 3, 1),
    "scalar_mul": _scalar_mul,
    "tanh": _unary("tanh", 2.0),
    "logistic": _unary("logistic", 40.0),  # exercises the +-60 clip
    "softmax": _unary("softmax", 3.0),
    "matmul_vec": _matmul_vec,
    "matmul_mat": _matmul_mat,
    "matmul_batched": _matmul_batched,
    "affine1": _affine1,
    "affine2": _affine2,
    "affine_batched_bias": _affine_batched_bias,
    "affine_batched_w": _affine_batched_w,
    "concatenate": _concat,
    "pick_range": _pick,
    "pnls": _pnls,
    "pnls_batch": _pnls_batch,
    "sum_batches": _sum_batches,
    "lookup": _lookup,
    "lookup_batch": _lookup_batch,
    "chain": _chain,
}


# ---------------------------------------------------------------------------
# workload traces (losses, per-step grads, touched rows, final params)
# ---------------------------------------------------------------------------


def call_loss(task, cg, datum):
    if isinstance(datum, tuple) and len(datum) == 2 and isinstance(datum[1], int) and not isinstance(datum[0], list):
        return task.loss(cg, datum[0], datum[1])
    return task.loss(cg, datum)


def workload_cases():
    lm_tiny = W.tiny_lm_corpus(11, 4)
    ptb = W.minibatches(W.ptb_corpus(12, 12, vocab=400), 4)
    td = W.tree_corpus(13, 3, vocab=60)
    tg = W.tagger_corpus(14, 40, n_types=400)
    return {
        # config 1 at its real size (V=1000, E=H=64, B=1), Adam sparse
        "tiny": (lambda dy, m: W.RNNLM(dy, m, 1000, 64, 64, 1), [[s] for s in lm_tiny], "adam", 3),
        # config 2 shape family at reduced width: 2 layers, MB=4, masked padding
        "ptb_mini": (lambda dy, m: W.RNNLM(dy, m, 400, 24, 32, 2), ptb, "adam", 3),
        "ptb_mini_sgd": (lambda dy, m: W.RNNLM(dy, m, 400, 24, 32, 2), ptb, "sgd", 3),
        # config 4 family: Tree-LSTM over random binary trees
        "tree_mini": (lambda dy, m: W.TreeClassifier(dy, m, 60, 5, 16, 12),
                      list(zip(td.trees, td.labels)), "adam", 3),
        # config 3 family: BiLSTM tagger with char-LSTM rare words
        "tagger_mini": (lambda dy, m: W.CharTagger(dy, m, tg, 16, 8, 8, 6, 7), tg.sentences, "adam", 3),
        # the remaining builders
        "gru_lm": (lambda dy, m: W.RNNLM(dy, m, 400, 24, 32, 2, "gru"), ptb, "adam", 3),
        "simple_lm": (lambda dy, m: W.RNNLM(dy, m, 400, 24, 32, 2, "simple"), ptb, "sgd", 3),
        "gru_lm_b1": (lambda dy, m: W.RNNLM(dy, m, 1000, 16, 24, 1, "gru"), [[s] for s in lm_tiny], "sgd", 3),
        "treernn": (lambda dy, m: W.TreeRNNClassifier(dy, m, 60, 5, 16), list(zip(td.trees, td.labels)), "adam", 3),
        "cfsm_lm": (lambda dy, m: W.CFSMLM(dy, m, 1000, 16, 24, 12), [[s] for s in lm_tiny], "adam", 3),
    }
