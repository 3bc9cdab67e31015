"""The reference frontend's scripting programs (fetests/test_programs.py:
the Fig. 1 two-word classifier and the Fig. 5 recursive tree encoder),
written against a `Frontend` so the same script runs on the B200 backend and
on the numpy oracle."""

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


class TreeRNNBuilder:
    """Fig. 5: tanh(W [enc(left); enc(right)]), unary nodes skipped."""

    def __init__(self, dy, model, word_vocab, hdim):
        self.dy = dy
        self.W = model.add_parameters((hdim, 2 * hdim))
        self.E = model.add_lookup_parameters((len(word_vocab), hdim))
        self.w2i = word_vocab

    def encode(self, tree):
        dy = self.dy
        if tree.isleaf():
            return self.E[self.w2i.get(tree.label, 0)]
        if len(tree.children) == 1:
            return self.encode(tree.children[0])
        e1 = self.encode(tree.children[0])
        e2 = self.encode(tree.children[1])
        W = dy.parameter(self.W)
        return dy.tanh(W * dy.concatenate([e1, e2]))


VOCAB = {"<unk>": 0, "red": 1, "green": 2, "blue": 3}


def small_tree():
    return Tree(None, [Tree(None, [Tree("red"), Tree("green")]), Tree("blue")])


def tree_program(dy, hdim=12, mem="48"):
    dy.init(mem=mem, seed=SEED)
    model = dy.Model()
    builder = TreeRNNBuilder(dy, model, VOCAB, hdim)
    dy.renew_cg()
    return builder.encode(small_tree()).npvalue()
