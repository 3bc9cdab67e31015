"""The reference frontend's scripting programs (pkg/frontend/tests/
test_programs.py:33-169: the Fig. 1 two-word classifier and the Fig. 5
recursive tree encoder) in two spellings:

* `classifier_program(dy, ...)` / `tree_program(dy, ...)`: against the
  scripting surface, i.e. the reference's `dyngraph` module itself (run
  unchanged, over the reference core to make the golden traces, or over this
  package through the `compat/dyncore` alias);
* `core_classifier_program(core, ...)` / `core_tree_program(core, ...)`: the
  same programs spelled as the core calls `dyngraph` delegates to one for one
  (`dyngraph/__init__.py`: one PoolSet from the mem flag shared by the graph
  and the model, `parameter()` per use, `E[i]` -> lookup, `*` -> matmul,
  `+` -> add, SimpleSGDTrainer -> Trainer(m, "sgd", 0.1)), so they run on the
  GPU box, where the reference frontend is not available.
"""

from __future__ import annotations

import numpy as np

EMB = 50
SEED = 5


def synthetic_pairs(seed: int, n: int, vocab: int = 30, n_classes: int = 3):
    rng = np.random.default_rng(seed)
    words = [f"w{i}" for i in range(vocab)]
    pairs = []
    for _ in range(n):
        a, b = rng.integers(0, vocab, 2)
        pairs.append((words[a], words[b], int((a + 2 * b) % n_classes)))
    return pairs, {w: i for i, w in enumerate(words)}, n_classes


# -- scripting-surface spelling ------------------------------------------------


def classifier_program(dy, pairs, vocab, n_classes, epochs=3, mem="48"):
    """Fig. 1: score = softmax(W [E[w1]; E[w2]] + b), per-example SGD."""
    dy.init(mem=mem, seed=SEED)
    model = dy.Model()
    W_p = model.add_parameters((n_classes, 2 * EMB))
    b_p = model.add_parameters(n_classes)
    E = model.add_lookup_parameters((len(vocab), EMB))
    trainer = dy.SimpleSGDTrainer(model)
    per_epoch = []
    for _ in range(epochs):
        total = 0.0
        for w1, w2, label in pairs:
            dy.renew_cg()
            W = dy.parameter(W_p)
            b = dy.parameter(b_p)
            score = dy.softmax(W * dy.concatenate([E[vocab[w1]], E[vocab[w2]]]) + b)
            loss = dy.pickneglogsoftmax(score, label)
            total += loss.value()
            loss.backward()
            trainer.update()
        per_epoch.append(total / len(pairs))
    return per_epoch


class Tree:
    def __init__(self, label, children=()):
        self.label = label
        self.children = list(children)

    def isleaf(self):
        return not self.children


VOCAB = {"<unk>": 0, "red": 1, "green": 2, "blue": 3}


def small_tree():
    return Tree(None, [Tree(None, [Tree("red"), Tree("green")]), Tree("blue")])


def tree_program(dy, hdim=12, mem="48"):
    """Fig. 5: enc(leaf) = E[w]; enc(node) = tanh(W [enc(l); enc(r)]); unary
    nodes pass through."""
    dy.init(mem=mem, seed=SEED)
    model = dy.Model()
    W_p = model.add_parameters((hdim, 2 * hdim))
    E = model.add_lookup_parameters((len(VOCAB), hdim))

    def enc(t):
        if t.isleaf():
            return E[VOCAB.get(t.label, 0)]
        if len(t.children) == 1:
            return enc(t.children[0])
        left, right = enc(t.children[0]), enc(t.children[1])
        return dy.tanh(dy.parameter(W_p) * dy.concatenate([left, right]))

    dy.renew_cg()
    return enc(small_tree()).npvalue()


# -- core-call spelling --------------------------------------------------------


def _ctx(core, mem):
    pools = core.poolset_from_mem_flag(mem)
    model = core.Model(pools, seed=SEED)
    return core.ComputationGraph(pools), model


def core_classifier_program(core, pairs, vocab, n_classes, epochs=3, mem="48", trace=None):
    ops = core.ops
    cg, model = _ctx(core, mem)
    W_p = model.add_parameters((n_classes, 2 * EMB))
    b_p = model.add_parameters(n_classes)
    E = model.add_lookup_parameters(len(vocab), EMB)
    trainer = core.Trainer(model, "sgd", 0.1)
    per_epoch = []
    for _ in range(epochs):
        total = 0.0
        for w1, w2, label in pairs:
            cg.renew()
            W = ops.parameter(cg, W_p)
            b = ops.parameter(cg, b_p)
            x = ops.concatenate([ops.lookup(cg, E, vocab[w1]), ops.lookup(cg, E, vocab[w2])])
            score = ops.softmax(ops.add(ops.matmul(W, x), b))
            loss = ops.pickneglogsoftmax(score, label)
            v = float(cg.value(loss).data[0])
            if trace is not None:
                trace.append(v)
            total += v
            cg.backward(loss)
            trainer.update()
        per_epoch.append(total / len(pairs))
    return per_epoch


def core_tree_program(core, hdim=12, mem="48", build_only=False):
    ops = core.ops
    cg, model = _ctx(core, mem)
    W_p = model.add_parameters((hdim, 2 * hdim))
    E = model.add_lookup_parameters(len(VOCAB), hdim)

    def enc(t):
        if t.isleaf():
            return ops.lookup(cg, E, VOCAB.get(t.label, 0))
        if len(t.children) == 1:
            return enc(t.children[0])
        left, right = enc(t.children[0]), enc(t.children[1])
        return ops.tanh(ops.matmul(ops.parameter(cg, W_p), ops.concatenate([left, right])))

    cg.renew()
    out = enc(small_tree())
    if build_only:
        return cg
    return np.array(cg.value(out).data, dtype=np.float64)
