"""Seeded synthetic workloads and the reference's per-batch graph builders.

The graph builders restate the reference bench tasks so the same node
sequence is emitted through whichever engine namespace `dy` is passed in
(this package, the CPU oracle, or the reference itself when generating
golden fixtures):

  * RNNLM per-sentence / lock-step minibatch   bench/tasks.py:411-440
  * BiLSTM tagger with char-LSTM rare words     bench/tasks.py:499-559
  * Tree-LSTM root-label loss                   bench/tasks.py:600-637

Synthetic shapes follow SURVEY.md 8(d).  Every generator is a pure function of
its seed (numpy default_rng).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BOS, EOS, UNK_ID = 1, 2, 0

# ---------------------------------------------------------------------------
# synthetic corpora
# ---------------------------------------------------------------------------


def _zipf_sampler(rng, lo, hi):
    """Zipf(s=1) over integer ids [lo, hi)."""
    ranks = np.arange(1, hi - lo + 1, dtype=np.float64)
    p = 1.0 / ranks
    p /= p.sum()
    cdf = np.cumsum(p)
    cdf[-1] = 1.0

    def draw(n):
        return lo + np.searchsorted(cdf, rng.random(n), side="right")

    return draw


def tiny_lm_corpus(seed: int, n_sent: int, vocab: int = 1000):
    """Config 1: ids 0 unk / 1 <s> / 2 </s>; lengths 8+U{0..8}; tokens U[3, vocab)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_sent):
        n = 8 + int(rng.integers(0, 9))
        toks = rng.integers(3, vocab, n)
        out.append([BOS] + [int(t) for t in toks] + [EOS])
    return out


def ptb_corpus(seed: int, n_sent: int, vocab: int = 10_000, mean_len: float = 20.1, max_len: int = 82):
    """Config 2: lengths 1+Poisson(20.1) clipped <= 82, Zipf tokens over 3..V-1."""
    rng = np.random.default_rng(seed)
    draw = _zipf_sampler(rng, 3, vocab)
    lens = np.minimum(1 + rng.poisson(mean_len, n_sent), max_len)
    return [[BOS] + [int(t) for t in draw(int(n))] + [EOS] for n in lens]


def lm_words(sentences) -> int:
    """Counting rule bench/tasks.py:460-461,473: len(ids)-1 per sentence."""
    return sum(len(s) - 1 for s in sentences)


def minibatches(items, mb: int):
    """Consecutive batching as in bench/tasks.py:474."""
    return [items[i : i + mb] for i in range(0, len(items), max(1, mb))]


@dataclass
class TaggerData:
    sentences: list  # list of list[(word, tag_id)]
    vocab: dict  # word -> id, UNK "<unk>" at 0, first-occurrence order
    chars: dict  # char -> id, UNK at 0
    n_tags: int


def tagger_corpus(seed: int, n_sent: int, n_types: int = 40_000, n_tags: int = 45,
                  alphabet: int = 80, mean_len: float = 22.9, unk_threshold: int = 5,
                  corpus_sentences: int | None = None) -> TaggerData:
    """Config 3: Zipf word types, rare words (count < 5) take the char path.

    The vocabulary (and so which words are rare) is counted over a corpus of
    `corpus_sentences` sentences (default: the n_sent returned); the WSJ-shaped
    benchmark counts it over 40k sentences (WSJ sections 02-21, ~40k
    sentences) and trains on the first n_sent of them."""
    n_all = max(n_sent, corpus_sentences or 0)
    rng = np.random.default_rng(seed)
    draw = _zipf_sampler(rng, 0, n_types)
    letters = [chr(0x21 + i) for i in range(alphabet)]
    spell_len = np.minimum(1 + rng.poisson(4.0, n_types), 20)
    spellings = ["".join(letters[c] for c in rng.integers(0, alphabet, int(n))) for n in spell_len]
    # make spellings unique deterministically (collisions would merge types)
    seen = {}
    for t, s in enumerate(spellings):
        while s in seen:
            s = s + letters[t % alphabet]
        seen[s] = t
        spellings[t] = s
    lens = 1 + rng.poisson(mean_len, n_all)
    sents = []
    for n in lens:
        types = draw(int(n))
        tags = rng.integers(0, n_tags, int(n))
        sents.append([(spellings[int(w)], int(t)) for w, t in zip(types, tags)])
    counts, order = {}, []
    for s in sents:
        for w, _ in s:
            if w not in counts:
                order.append(w)
                counts[w] = 0
            counts[w] += 1
    vocab = {"<unk>": 0}
    for w in order:
        if counts[w] >= unk_threshold:
            vocab[w] = len(vocab)
    chars = {"<unk>": 0}
    for s in sents:
        for w, _ in s:
            for ch in w:
                if ch not in chars:
                    chars[ch] = len(chars)
    return TaggerData(sents[:n_sent], vocab, chars, n_tags)


@dataclass
class TreeData:
    trees: list  # nested tuples: int leaf token | (left, right)
    labels: list
    vocab_size: int


def _split_tree(rng, n, draw):
    if n == 1:
        return int(draw(1)[0])
    left = int(rng.integers(1, n))
    return (_split_tree(rng, left, draw), _split_tree(rng, n - left, draw))


def tree_corpus(seed: int, n_trees: int, vocab: int = 18_300, n_labels: int = 5,
                mean_leaves: float = 18.2, max_leaves: int = 56) -> TreeData:
    """Config 4: leaves 1+Poisson(18.2) in [2, 56], uniform binary splits."""
    rng = np.random.default_rng(seed)
    draw = _zipf_sampler(rng, 0, vocab)
    leaves = np.clip(1 + rng.poisson(mean_leaves, n_trees), 2, max_leaves)
    trees = [_split_tree(rng, int(n), draw) for n in leaves]
    labels = [int(x) for x in rng.integers(0, n_labels, n_trees)]
    return TreeData(trees, labels, vocab)


def to_treenode(dy, t, label=None):
    if isinstance(t, int):
        return dy.TreeNode.leaf(f"w{t}", label)
    return dy.TreeNode.binary(to_treenode(dy, t[0]), to_treenode(dy, t[1]), label)


def count_leaves(t) -> int:
    return 1 if isinstance(t, int) else count_leaves(t[0]) + count_leaves(t[1])


# ---------------------------------------------------------------------------
# graph builders (engine-agnostic; `dy` is a dyncore-shaped namespace)
# ---------------------------------------------------------------------------


class RNNLM:
    """bench/tasks.py:443-452 registration order: E, rnn, W, b."""

    def __init__(self, dy, model, vocab: int, embed: int, hidden: int, layers: int, cell: str = "lstm"):
        self.dy = dy
        self.E = model.add_lookup_parameters(vocab, embed, "E")
        self.rnn = dy.RNNBuilder(model, layers, embed, hidden, cell, "rnn")
        self.W = model.add_parameters((vocab, hidden), "W")
        self.b = model.add_parameters((vocab,), "b")

    def sentence_nll(self, cg, ids):
        """bench/tasks.py:411-420."""
        ops = self.dy.ops
        we, be = ops.parameter(cg, self.W), ops.parameter(cg, self.b)
        state = self.rnn.initial_state(cg)
        loss = None
        for t in range(len(ids) - 1):
            state = state.add_input(ops.lookup(cg, self.E, ids[t]))
            step = ops.pickneglogsoftmax(ops.affine(be, we, state.output()), ids[t + 1])
            loss = step if loss is None else ops.add(loss, step)
        return loss

    def batch_nll(self, cg, batch_ids, pad_id: int = EOS):
        """bench/tasks.py:423-440: lock-step, end-padded with EOS, masked."""
        dy, ops = self.dy, self.dy.ops
        we, be = ops.parameter(cg, self.W), ops.parameter(cg, self.b)
        t_max = max(len(ids) for ids in batch_ids)
        nb = len(batch_ids)
        # the padded id matrix once per batch (the per-step columns are exactly
        # the reference's per-step list comprehensions, bench/tasks.py:432-438)
        lens = np.array([len(ids) for ids in batch_ids])
        padded = np.full((nb, t_max), pad_id, dtype=np.int64)
        for r, ids in enumerate(batch_ids):
            padded[r, : len(ids)] = ids
        cols = padded.T.tolist()
        masks = (np.arange(1, t_max)[:, None] < lens[None, :]).astype(cg.dtype)
        mask_shape = dy.Shape((1,), nb)
        rnn = self.rnn
        state = rnn.initial_state(cg)
        lookup_batch, affine, pnls_batch = ops.lookup_batch, ops.affine, ops.pickneglogsoftmax_batch
        cmult, inp, sum_batches, add, Tensor, E = ops.cmult, ops.input, ops.sum_batches, ops.add, dy.Tensor, self.E
        # LSTM steps through the native graph core (the nodes add_input makes,
        # in the same order; the layer parameters appear at the first step)
        core = getattr(cg, "_core", None)
        native = (core is not None and getattr(rnn, "cell", None) == "lstm" and type(getattr(state, "hs", None)) is list
                  and type(getattr(state, "cs", None)) is list)
        hs, cs, pex, H = (state.hs, state.cs, None, rnn.hidden_dim) if native else (None, None, None, None)
        loss = None
        for t in range(t_max - 1):
            x = lookup_batch(cg, E, cols[t])
            if native:
                if pex is None:
                    pex = rnn._graph_params(cg)
                hs, cs = core.lstm_step(pex, hs, cs, x, H)
                h = hs[-1]
            else:
                state = state.add_input(x)
                h = state.output()
            nll = pnls_batch(affine(be, we, h), cols[t + 1])
            step = sum_batches(cmult(nll, inp(cg, Tensor(mask_shape, masks[t]))))
            loss = step if loss is None else add(loss, step)
        return loss

    def loss(self, cg, batch):
        if len(batch) == 1:
            return self.sentence_nll(cg, batch[0])
        return self.batch_nll(cg, batch)


class CharTagger:
    """bench/tasks.py:499-559 (char features on): registration order E, fwd,
    bwd, W1, b1, W2, b2, CE, cfwd, cbwd, Wp, bp."""

    def __init__(self, dy, model, data: TaggerData, embed=128, hidden=50, mlp=32,
                 char_dim=20, char_hidden=50, layers=1):
        self.dy = dy
        self.vocab, self.chars = data.vocab, data.chars
        self.E = model.add_lookup_parameters(len(data.vocab), embed, "E")
        self.fwd = dy.RNNBuilder(model, layers, embed, hidden, "lstm", "fwd")
        self.bwd = dy.RNNBuilder(model, layers, embed, hidden, "lstm", "bwd")
        self.W1 = model.add_parameters((mlp, 2 * hidden), "W1")
        self.b1 = model.add_parameters((mlp,), "b1")
        self.W2 = model.add_parameters((data.n_tags, mlp), "W2")
        self.b2 = model.add_parameters((data.n_tags,), "b2")
        self.CE = model.add_lookup_parameters(len(data.chars), char_dim, "CE")
        self.cfwd = dy.RNNBuilder(model, 1, char_dim, char_hidden, "lstm", "cfwd")
        self.cbwd = dy.RNNBuilder(model, 1, char_dim, char_hidden, "lstm", "cbwd")
        self.Wp = model.add_parameters((embed, 2 * char_hidden), "Wp")
        self.bp = model.add_parameters((embed,), "bp")

    def embed_word(self, cg, word):
        ops = self.dy.ops
        if word in self.vocab:
            return ops.lookup(cg, self.E, self.vocab[word])
        chars = [ops.lookup(cg, self.CE, self.chars.get(ch, 0)) for ch in word]
        f_last = self.cfwd.initial_state(cg).transduce(chars)[-1]
        b_last = self.cbwd.initial_state(cg).transduce(list(reversed(chars)))[-1]
        return ops.affine(ops.parameter(cg, self.bp), ops.parameter(cg, self.Wp),
                          ops.concatenate([f_last, b_last]))

    def token_scores(self, cg, words):
        ops = self.dy.ops
        embs = [self.embed_word(cg, w) for w in words]
        f_outs = self.fwd.initial_state(cg).transduce(embs)
        b_outs = self.bwd.initial_state(cg).transduce(list(reversed(embs)))[::-1]
        w1e, b1e = ops.parameter(cg, self.W1), ops.parameter(cg, self.b1)
        w2e, b2e = ops.parameter(cg, self.W2), ops.parameter(cg, self.b2)
        scores = []
        for f, bk in zip(f_outs, b_outs):
            h = ops.tanh(ops.affine(b1e, w1e, ops.concatenate([f, bk])))
            scores.append(ops.affine(b2e, w2e, h))
        return scores

    def loss(self, cg, sent):
        ops = self.dy.ops
        loss = None
        for s, (_, tag) in zip(self.token_scores(cg, [w for w, _ in sent]), sent):
            step = ops.pickneglogsoftmax(s, tag)
            loss = step if loss is None else ops.add(loss, step)
        return loss


class TreeClassifier:
    """bench/tasks.py:600-637: TreeLSTM encoder then root affine + pnls."""

    def __init__(self, dy, model, vocab_size: int, n_labels: int = 5, embed=128, hidden=150):
        self.dy = dy
        w2i = {f"w{i}": i for i in range(vocab_size)}
        self.encoder = dy.TreeLSTM(model, w2i, embed, hidden, "enc")
        self.U = model.add_parameters((n_labels, hidden), "U")
        self.bu = model.add_parameters((n_labels,), "bu")

    def loss(self, cg, tree, label):
        ops = self.dy.ops
        h, _ = self.encoder.encode(cg, to_treenode(self.dy, tree))
        scores = ops.affine(ops.parameter(cg, self.bu), ops.parameter(cg, self.U), h)
        return ops.pickneglogsoftmax(scores, label)


class TreeRNNClassifier:
    """The Fig. 5 TreeRNN encoder (builders.py:183-210) under the Tree-LSTM
    task's root classifier (bench/tasks.py:600-637 shape): registration
    enc.W, enc.E, U, bu."""

    def __init__(self, dy, model, vocab_size: int, n_labels: int = 5, hidden=150):
        self.dy = dy
        self.encoder = dy.TreeRNN(model, {f"w{i}": i for i in range(vocab_size)}, hidden, "enc")
        self.U = model.add_parameters((n_labels, hidden), "U")
        self.bu = model.add_parameters((n_labels,), "bu")

    def loss(self, cg, tree, label):
        ops = self.dy.ops
        h = self.encoder.encode(cg, to_treenode(self.dy, tree))
        return ops.pickneglogsoftmax(ops.affine(ops.parameter(cg, self.bu), ops.parameter(cg, self.U), h), label)


class CFSMLM:
    """LSTM language model with a ClassFactoredSoftmax output layer
    (builders.py:282-378): per-sentence graphs, loss = sum over t of
    -log p(class) - log p(word | class).  Word w belongs to class
    (w * 7919) % n_classes (a deterministic, unbalanced map)."""

    def __init__(self, dy, model, vocab: int, embed: int, hidden: int, n_classes: int):
        self.dy = dy
        self.E = model.add_lookup_parameters(vocab, embed, "E")
        self.rnn = dy.RNNBuilder(model, 1, embed, hidden, "lstm", "rnn")
        self.out = dy.ClassFactoredSoftmax(model, hidden, {w: (w * 7919) % n_classes for w in range(vocab)}, "cfsm")

    def loss(self, cg, batch):
        ops = self.dy.ops
        ids = batch[0]
        state = self.rnn.initial_state(cg)
        loss = None
        for t in range(len(ids) - 1):
            state = state.add_input(ops.lookup(cg, self.E, ids[t]))
            step = self.out.neg_log_softmax(cg, state.output(), ids[t + 1])
            loss = step if loss is None else ops.add(loss, step)
        return loss


@dataclass
class Config:
    name: str
    params: dict = field(default_factory=dict)


CONFIGS = {
    "tiny": dict(vocab=1000, embed=64, hidden=64, layers=1, mb=1),
    "ptb16": dict(vocab=10_000, embed=128, hidden=256, layers=2, mb=16),
    "ptb64": dict(vocab=10_000, embed=128, hidden=256, layers=2, mb=64),
    "tagger": dict(embed=128, hidden=50, mlp=32, char_dim=20, char_hidden=50),
    "tree": dict(vocab=18_300, embed=128, hidden=150, labels=5),
}
