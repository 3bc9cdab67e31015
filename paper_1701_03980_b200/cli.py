"""`dyngraph <task>` benchmark runners on the B200 backend
(pkg/src/dyncore/bench/cli.py:23-95, bench/tasks.py:118-124,294-651).

    python -m paper_1701_03980_b200.cli rnnlm --train T --dev D [--epochs N ...]

Same flags, same data formats, same models (parameter names, registration
order, initialisation), same training loops and the same report lines:

    startup_secs=<time from program start to the first training instance>
    epoch=<n> loss=<mean train loss> metric=<task metric> speed=<units/s>

(loss and metric printed with 10 significant digits, speed and startup with
6).  Every forward / backward / update runs in the device executor.

Deviations: `--gen` (the reference's synthetic-corpus writer) is not part of
the backend -- generate data with the reference, or use any file in the
formats below; `--workers > 1` is served by one process per GPU
(torchrun + parallel.DataParallel), not by in-process worker threads, and is
refused here with ConfigError.

Data formats (the reference readers, bench/tasks.py:135-260):
  rnnlm      one whitespace-tokenised sentence per line
  tagger(-char)  `word<TAB>tag` lines, blank line between sentences
  treelstm   one labelled s-expression per line: `(3 (2 w) (1 w))`
  pairclass  `word1 word2 label` per line
  earlystop  `word ... label` per line, label in {-1, 1}
"""

from __future__ import annotations

import argparse
import math
import sys
import time
from collections import Counter

import numpy as np

TASKS = ("rnnlm", "tagger", "tagger-char", "treelstm", "pairclass", "earlystop")
# word embedding / recurrent / perceptron widths per task (bench/tasks.py:28-35)
DIMS = {
    "rnnlm": dict(embed=128, hidden=256),
    "tagger": dict(embed=128, hidden=50, mlp=32),
    "tagger-char": dict(embed=128, hidden=50, mlp=32, char_dim=20, char_hidden=50),
    "treelstm": dict(embed=128, hidden=128),
    "pairclass": dict(embed=50, hidden=0),
    "earlystop": dict(embed=50, hidden=0),
}
UNK, BOS, EOS = "<unk>", "<s>", "</s>"


# ---------------------------------------------------------------------------
# vocabulary (bench/vocab.py): UNK at 0, then specials, then tokens meeting
# the frequency threshold in first-occurrence order
# ---------------------------------------------------------------------------


class Vocab:
    def __init__(self, tokens, threshold):
        self.i2t = list(tokens)
        self.t2i = {t: i for i, t in enumerate(self.i2t)}
        self.threshold = threshold

    @classmethod
    def build(cls, corpus_tokens, unk_threshold=1, specials=()):
        from .errors import DataError

        counts = Counter(corpus_tokens)  # Counter keeps first-occurrence order
        if not counts:
            raise DataError("empty corpus: no tokens to build a vocabulary from")
        head = [UNK, *specials]
        kept = [t for t, n in counts.items() if n >= unk_threshold and t not in head]
        return cls(head + kept, unk_threshold)

    def id(self, token):
        return self.t2i.get(token, 0)

    def known(self, token):
        return token in self.t2i

    def __len__(self):
        return len(self.i2t)


# ---------------------------------------------------------------------------
# readers
# ---------------------------------------------------------------------------


def _lines(path):
    from .errors import FileError

    try:
        with open(path, "r", encoding="utf-8") as fh:
            return fh.read().splitlines()
    except OSError as exc:
        raise FileError(f"cannot read {path}: {exc}") from exc


def _nonempty(items, path, what):
    from .errors import DataError

    if not items:
        raise DataError(f"{path}: no {what}")
    return items


def read_token_lines(path):
    return _nonempty([ln.split() for ln in _lines(path) if ln.split()], path, "sentences")


def read_pairs(path):
    from .errors import DataError

    out = []
    for ln, line in enumerate(_lines(path), start=1):
        f = line.split()
        if not f:
            continue
        if len(f) != 3:
            raise DataError(f"{path}:{ln}: expected 'word1 word2 label'")
        try:
            out.append((f[0], f[1], int(f[2])))
        except ValueError as exc:
            raise DataError(f"{path}:{ln}: label {f[2]!r} is not an integer") from exc
    return _nonempty(out, path, "examples")


def read_tagged(path):
    from .errors import DataError

    sents, cur = [], []
    for ln, line in enumerate(_lines(path), start=1):
        if not line.strip():
            if cur:
                sents.append(cur)
            cur = []
            continue
        f = line.split("\t")
        if len(f) != 2 or not all(f):
            raise DataError(f"{path}:{ln}: expected 'word<TAB>tag', got {line!r}")
        cur.append((f[0], f[1]))
    if cur:
        sents.append(cur)
    return _nonempty(sents, path, "sentences")


def read_labeled_docs(path):
    from .errors import DataError

    docs = []
    for ln, line in enumerate(_lines(path), start=1):
        f = line.split()
        if not f:
            continue
        if len(f) < 2:
            raise DataError(f"{path}:{ln}: expected 'word... label'")
        try:
            label = int(f[-1])
        except ValueError as exc:
            raise DataError(f"{path}:{ln}: label {f[-1]!r} is not an integer") from exc
        if label not in (-1, 1):
            raise DataError(f"{path}:{ln}: label must be -1 or 1, got {label}")
        docs.append((f[:-1], label))
    return _nonempty(docs, path, "documents")


def read_trees(path):
    """Labelled s-expressions, parsed with an explicit stack."""
    from .builders import TreeNode
    from .errors import DataError

    trees = []
    for ln, line in enumerate(_lines(path), start=1):
        toks = line.replace("(", " ( ").replace(")", " ) ").split()
        if not toks:
            continue

        def fail(msg, ln=ln):
            raise DataError(f"{path}:{ln}: {msg}")

        stack = []  # open nodes: [label, token, children]
        root = None
        i = 0
        while i < len(toks):
            t = toks[i]
            if t == "(":
                if root is not None:
                    fail("trailing tokens after the tree")
                if i + 1 >= len(toks):
                    fail("missing node label")
                try:
                    stack.append([int(toks[i + 1]), None, []])
                except ValueError:
                    fail(f"node label {toks[i + 1]!r} is not an integer")
                i += 2
                continue
            if not stack:
                fail("trailing tokens after the tree" if root is not None else f"expected '(' at token {i}")
            if t == ")":
                label, token, kids = stack.pop()
                if token is not None and kids:
                    fail("node mixes a leaf token with children")
                if token is not None:
                    node = TreeNode.leaf(token, label)
                elif 1 <= len(kids) <= 2:
                    node = TreeNode(children=tuple(kids), label=label)
                else:
                    fail(f"nodes are unary or binary, got {len(kids)} children")
                if stack:
                    stack[-1][2].append(node)
                else:
                    root = node
            else:
                stack[-1][1] = t
            i += 1
        if stack:
            fail("missing ')'")
        trees.append(root)
    return _nonempty(trees, path, "trees")


def _leaves(tree):
    todo = [tree]
    while todo:
        t = todo.pop()
        if t.is_leaf():
            yield t.token
        todo.extend(reversed(t.children))


# ---------------------------------------------------------------------------
# runner plumbing (bench/tasks.py:93-130)
# ---------------------------------------------------------------------------


class Run:
    def __init__(self, cfg, out):
        import paper_1701_03980_b200 as dy

        self.dy, self.cfg, self.out = dy, cfg, out
        self.t0 = cfg.t0
        self.pools = dy.poolset_from_mem_flag(cfg.mem)
        self.cg = dy.ComputationGraph(self.pools)
        self.model = dy.Model(self.pools, seed=cfg.seed, init_zero=cfg.init_zero)
        self.report = {"startup_secs": 0.0, "epochs": [], "extra": {}}

    def trainer(self):
        if self.cfg.load:
            self.model.load(self.cfg.load)
        return self.dy.Trainer(self.model, self.cfg.trainer, self.cfg.lr, sparse=self.cfg.sparse)

    def say(self, line):
        if self.out is not None:
            print(line, file=self.out, flush=True)

    def started(self):
        self.report["startup_secs"] = time.perf_counter() - self.t0
        self.say(f"startup_secs={self.report['startup_secs']:.6g}")

    def epoch(self, n, loss, metric, speed):
        self.report["epochs"].append((n, loss, metric, speed))
        self.say(f"epoch={n} loss={loss:.10g} metric={metric:.10g} speed={speed:.6g}")

    def done(self):
        if self.cfg.save:
            self.model.save(self.cfg.save)
        return self.report

    def serial_epoch(self, items, loss_fn, trainer):
        """renew -> build -> backward -> value -> update per item (the
        reference's serial train_parallel path and the rnnlm/treelstm loops)."""
        cg, total = self.cg, 0.0
        for item in items:
            cg.renew()
            loss = loss_fn(cg, item)
            cg.backward(loss)
            total += float(cg.value(loss).data[0])
            trainer.update()
        return total

    def timed_epochs(self, items, loss_fn, trainer, units, evaluate):
        self.started()
        for n in range(1, self.cfg.epochs + 1):
            tick = time.perf_counter()
            total = self.serial_epoch(items, loss_fn, trainer)
            secs = max(time.perf_counter() - tick, 1e-9)
            metric = evaluate()
            self.epoch(n, total / self.n_train, metric, units / secs)


# ---------------------------------------------------------------------------
# tasks
# ---------------------------------------------------------------------------


def run_rnnlm(cfg, out=None):
    r = Run(cfg, out)
    ops = r.dy.ops
    train, dev = read_token_lines(cfg.train), read_token_lines(cfg.dev)
    vocab = Vocab.build((t for s in train for t in s), cfg.unk_threshold, specials=(BOS, EOS))
    m = r.model
    E = m.add_lookup_parameters(len(vocab), cfg.embed, "E")
    rnn = r.dy.RNNBuilder(m, cfg.layers, cfg.embed, cfg.hidden, "lstm", "rnn")
    W = m.add_parameters((len(vocab), cfg.hidden), "W")
    b = m.add_parameters((len(vocab),), "b")
    trainer = r.trainer()
    eos = vocab.id(EOS)

    def ids_of(toks):
        return [vocab.id(BOS), *map(vocab.id, toks), eos]

    def sentence_nll(cg, ids):
        we, be = ops.parameter(cg, W), ops.parameter(cg, b)
        state, loss = rnn.initial_state(cg), None
        for t in range(len(ids) - 1):
            state = state.add_input(ops.lookup(cg, E, ids[t]))
            term = ops.pickneglogsoftmax(ops.affine(be, we, state.output()), ids[t + 1])
            loss = term if loss is None else ops.add(loss, term)
        return loss

    def batch_nll(cg, batch):
        we, be = ops.parameter(cg, W), ops.parameter(cg, b)
        n, t_max = len(batch), max(map(len, batch))
        grid = np.full((n, t_max), eos, dtype=np.int64)
        for i, ids in enumerate(batch):
            grid[i, : len(ids)] = ids
        lens = np.array([len(ids) for ids in batch])
        state, loss = rnn.initial_state(cg), None
        for t in range(t_max - 1):
            mask = (t + 1 < lens).astype(np.float32)
            state = state.add_input(ops.lookup_batch(cg, E, grid[:, t].tolist()))
            nll = ops.pickneglogsoftmax_batch(ops.affine(be, we, state.output()), grid[:, t + 1].tolist())
            term = ops.sum_batches(ops.cmult(nll, ops.input(cg, r.dy.Tensor(r.dy.Shape((1,), n), mask))))
            loss = term if loss is None else ops.add(loss, term)
        return loss

    step = max(1, cfg.batch_size)
    batches = [[ids_of(s) for s in train[i : i + step]] for i in range(0, len(train), step)]

    def loss_fn(cg, batch):
        return sentence_nll(cg, batch[0]) if len(batch) == 1 else batch_nll(cg, batch)

    def perplexity():
        total = count = 0
        for toks in dev:
            ids = ids_of(toks)
            r.cg.renew()
            total += float(r.cg.value(sentence_nll(r.cg, ids)).data[0])
            count += len(ids) - 1
        return math.exp(total / count)

    r.n_train = len(train)
    r.timed_epochs(batches, loss_fn, trainer, sum(len(s) + 1 for s in train), perplexity)
    return r.done()


def run_tagger(cfg, out=None, char_features=None):
    if char_features is None:
        char_features = cfg.task == "tagger-char"
    r = Run(cfg, out)
    ops = r.dy.ops
    train, dev = read_tagged(cfg.train), read_tagged(cfg.dev)
    vocab = Vocab.build((w for s in train for w, _ in s), cfg.unk_threshold)
    tag2i = {}
    for s in train:
        for _, t in s:
            tag2i.setdefault(t, len(tag2i))
    m, RNN = r.model, r.dy.RNNBuilder
    E = m.add_lookup_parameters(len(vocab), cfg.embed, "E")
    fwd = RNN(m, cfg.layers, cfg.embed, cfg.hidden, "lstm", "fwd")
    bwd = RNN(m, cfg.layers, cfg.embed, cfg.hidden, "lstm", "bwd")
    W1 = m.add_parameters((cfg.mlp, 2 * cfg.hidden), "W1")
    b1 = m.add_parameters((cfg.mlp,), "b1")
    W2 = m.add_parameters((len(tag2i), cfg.mlp), "W2")
    b2 = m.add_parameters((len(tag2i),), "b2")
    if char_features:
        cvocab = Vocab.build((ch for s in train for w, _ in s for ch in w), 1)
        CE = m.add_lookup_parameters(len(cvocab), cfg.char_dim, "CE")
        cfwd = RNN(m, 1, cfg.char_dim, cfg.char_hidden, "lstm", "cfwd")
        cbwd = RNN(m, 1, cfg.char_dim, cfg.char_hidden, "lstm", "cbwd")
        Wp = m.add_parameters((cfg.embed, 2 * cfg.char_hidden), "Wp")
        bp = m.add_parameters((cfg.embed,), "bp")
    trainer = r.trainer()

    def embed(cg, word):
        if not char_features or vocab.known(word):
            return ops.lookup(cg, E, vocab.id(word))
        chars = [ops.lookup(cg, CE, cvocab.id(ch)) for ch in word]
        last_f = cfwd.initial_state(cg).transduce(chars)[-1]
        last_b = cbwd.initial_state(cg).transduce(chars[::-1])[-1]
        return ops.affine(ops.parameter(cg, bp), ops.parameter(cg, Wp), ops.concatenate([last_f, last_b]))

    def scores(cg, words):
        xs = [embed(cg, w) for w in words]
        fo = fwd.initial_state(cg).transduce(xs)
        bo = bwd.initial_state(cg).transduce(xs[::-1])[::-1]
        w1, bb1 = ops.parameter(cg, W1), ops.parameter(cg, b1)
        w2, bb2 = ops.parameter(cg, W2), ops.parameter(cg, b2)
        return [ops.affine(bb2, w2, ops.tanh(ops.affine(bb1, w1, ops.concatenate([f, k])))) for f, k in zip(fo, bo)]

    def loss_fn(cg, sent):
        loss = None
        for s, (_, tag) in zip(scores(cg, [w for w, _ in sent]), sent):
            term = ops.pickneglogsoftmax(s, tag2i[tag])
            loss = term if loss is None else ops.add(loss, term)
        return loss

    def accuracy():
        hits = total = rare_hits = rare_total = 0
        for sent in dev:
            r.cg.renew()
            for s, (word, tag) in zip(scores(r.cg, [w for w, _ in sent]), sent):
                hit = tag in tag2i and int(np.argmax(r.cg.value(s).data)) == tag2i[tag]
                hits, total = hits + hit, total + 1
                if not vocab.known(word):
                    rare_hits, rare_total = rare_hits + hit, rare_total + 1
        if rare_total:
            r.report["extra"].update(rare_accuracy=rare_hits / rare_total, rare_total=rare_total)
        return hits / total

    r.n_train = len(train)
    r.timed_epochs(train, loss_fn, trainer, sum(map(len, train)), accuracy)
    return r.done()


def run_treelstm(cfg, out=None):
    r = Run(cfg, out)
    ops = r.dy.ops
    train, dev = read_trees(cfg.train), read_trees(cfg.dev)
    vocab = Vocab.build((tok for t in train for tok in _leaves(t)), cfg.unk_threshold)
    n_labels = max(t.label for t in train) + 1
    m = r.model
    enc = r.dy.TreeLSTM(m, vocab.t2i, cfg.embed, cfg.hidden, "enc")
    U = m.add_parameters((n_labels, cfg.hidden), "U")
    bu = m.add_parameters((n_labels,), "bu")
    trainer = r.trainer()

    def root_scores(cg, tree):
        h, _ = enc.encode(cg, tree)
        return ops.affine(ops.parameter(cg, bu), ops.parameter(cg, U), h)

    def accuracy(trees):
        hits = 0
        for t in trees:
            r.cg.renew()
            hits += int(np.argmax(r.cg.value(root_scores(r.cg, t)).data)) == t.label
        return hits / len(trees)

    def dev_accuracy():
        acc = accuracy(dev)
        r.report["extra"]["train_accuracy"] = accuracy(train)
        return acc

    r.n_train = len(train)
    r.timed_epochs(train, lambda cg, t: ops.pickneglogsoftmax(root_scores(cg, t), t.label), trainer, len(train),
                   dev_accuracy)
    return r.done()


def run_pairclass(cfg, out=None):
    r = Run(cfg, out)
    ops = r.dy.ops
    train, dev = read_pairs(cfg.train), read_pairs(cfg.dev)
    vocab = Vocab.build((w for ex in train for w in ex[:2]), cfg.unk_threshold)
    n_classes = max(ex[2] for ex in train) + 1
    m = r.model
    W = m.add_parameters((n_classes, 2 * cfg.embed), "W")
    b = m.add_parameters((n_classes,), "b")
    E = m.add_lookup_parameters(len(vocab), cfg.embed, "E")
    trainer = r.trainer()

    def softmax_scores(cg, ids1, ids2):
        we, be = ops.parameter(cg, W), ops.parameter(cg, b)
        if isinstance(ids1, list):
            x = ops.concatenate([ops.lookup_batch(cg, E, ids1), ops.lookup_batch(cg, E, ids2)])
        else:
            x = ops.concatenate([ops.lookup(cg, E, ids1), ops.lookup(cg, E, ids2)])
        return ops.softmax(ops.add(ops.matmul(we, x), be))

    def loss_fn(cg, item):
        if isinstance(item, list):  # a minibatch
            s = softmax_scores(cg, [vocab.id(e[0]) for e in item], [vocab.id(e[1]) for e in item])
            return ops.sum_batches(ops.pickneglogsoftmax_batch(s, [e[2] for e in item]))
        return ops.pickneglogsoftmax(softmax_scores(cg, vocab.id(item[0]), vocab.id(item[1])), item[2])

    def accuracy():
        hits = 0
        for w1, w2, label in dev:
            r.cg.renew()
            hits += int(np.argmax(r.cg.value(softmax_scores(r.cg, vocab.id(w1), vocab.id(w2))).data)) == label
        return hits / len(dev)

    bs = cfg.batch_size
    items = train if bs <= 1 else [train[i : i + bs] for i in range(0, len(train), bs)]
    r.n_train = len(train)
    r.timed_epochs(items, loss_fn, trainer, 2 * len(train), accuracy)
    return r.done()


def run_earlystop(cfg, out=None):
    r = Run(cfg, out)
    ops = r.dy.ops
    train, dev = read_labeled_docs(cfg.train), read_labeled_docs(cfg.dev)
    vocab = Vocab.build((w for doc, _ in train for w in doc), cfg.unk_threshold)
    m = r.model
    W = m.add_parameters((1, cfg.embed), "W")
    b = m.add_parameters((1,), "b")
    E = m.add_lookup_parameters(len(vocab), cfg.embed, "E")
    trainer = r.trainer()

    def loss_fn(cg, doc):
        words, label = doc
        we, be = ops.parameter(cg, W), ops.parameter(cg, b)
        acc = None
        for w in words:
            e = ops.lookup(cg, E, vocab.id(w))
            acc = e if acc is None else ops.add(acc, e)
        return ops.logistic(ops.scalar_mul(ops.add(ops.matmul(we, acc), be), float(label)))

    def early_accuracy():
        """Incremental inference: extend the graph a word at a time, stop once
        |score| clears --threshold (bench/tasks.py:370-389)."""
        cg, hits, read = r.cg, 0, 0
        for words, label in dev:
            cg.renew()
            we = ops.parameter(cg, W)
            score = ops.parameter(cg, b)
            val = float(cg.value(score).data[0])
            for w in words:
                score = ops.add(score, ops.matmul(we, ops.lookup(cg, E, vocab.id(w))))
                read += 1
                val = float(cg.value(score).data[0])
                if abs(val) > cfg.threshold:
                    break
            hits += label * val > 0
        r.report["extra"].update(mean_words_read=read / len(dev), mean_doc_len=sum(len(d) for d, _ in dev) / len(dev))
        return hits / len(dev)

    r.n_train = len(train)
    r.timed_epochs(train, loss_fn, trainer, sum(len(d) for d, _ in train), early_accuracy)
    r.say(f"mean_words_read={r.report['extra']['mean_words_read']:.6g}")
    return r.done()


RUNNERS = {
    "rnnlm": run_rnnlm,
    "tagger": run_tagger,
    "tagger-char": run_tagger,
    "treelstm": run_treelstm,
    "pairclass": run_pairclass,
    "earlystop": run_earlystop,
}


class Config:
    """TaskConfig (bench/tasks.py:40-80): per-task default widths + flags."""

    def __init__(self, task, train, dev, **kw):
        self.task, self.train, self.dev = task, train, dev
        base = dict(embed=128, hidden=128, mlp=32, char_dim=20, char_hidden=50, layers=1, batch_size=1, epochs=5,
                    trainer="adam", lr=None, sparse=True, workers=1, mem="128", seed=1, unk_threshold=1,
                    threshold=math.inf, save=None, load=None, init_zero=False, t0=None)
        base.update(DIMS[task])
        base.update(kw)
        for k, v in base.items():
            setattr(self, k, v)
        if self.t0 is None:
            self.t0 = time.perf_counter()


def build_parser():
    p = argparse.ArgumentParser(prog="dyngraph", description="Train and evaluate the benchmark tasks on the "
                                "B200 dynamic-graph executor.")
    sub = p.add_subparsers(dest="task", required=True)
    for task in TASKS:
        s = sub.add_parser(task, help=f"run the {task} task")
        s.add_argument("--train", required=True)
        s.add_argument("--dev", required=True)
        s.add_argument("--gen", action="store_true", help="(not supported: generate data with the reference)")
        s.add_argument("--gen-sentences", type=int, default=None)
        s.add_argument("--gen-vocab", type=int, default=None)
        s.add_argument("--epochs", type=int, default=5)
        s.add_argument("--batch-size", type=int, default=1)
        s.add_argument("--trainer", choices=("sgd", "momentum", "adagrad", "adam"), default="adam")
        s.add_argument("--lr", type=float, default=None)
        s.add_argument("--sparse", choices=("on", "off"), default=None)
        s.add_argument("--workers", type=int, default=1)
        s.add_argument("--mem", default="128")
        s.add_argument("--seed", type=int, default=1)
        s.add_argument("--save", default=None)
        s.add_argument("--load", default=None)
        s.add_argument("--threshold", type=float, default=None)
        s.add_argument("--unk-threshold", type=int, default=1)
        s.add_argument("--init-zero", action="store_true")
    return p


def main(argv=None) -> int:
    t0 = time.perf_counter()
    args = build_parser().parse_args(argv)
    from .errors import ConfigError, DyncoreError

    try:
        if args.gen:
            raise ConfigError("--gen is not supported by the B200 backend; write the data files with the reference")
        if args.workers > 1:
            if args.sparse == "on":
                raise ConfigError("sparse updates are undefined across workers; use --sparse off")
            raise ConfigError("--workers > 1: run one process per GPU (torchrun) with parallel.DataParallel")
        cfg = Config(args.task, args.train, args.dev, epochs=args.epochs, batch_size=args.batch_size,
                     trainer=args.trainer, lr=args.lr, sparse=args.sparse != "off", workers=args.workers,
                     mem=args.mem, seed=args.seed, save=args.save, load=args.load,
                     threshold=math.inf if args.threshold is None else args.threshold,
                     unk_threshold=args.unk_threshold, init_zero=args.init_zero, t0=t0)
        RUNNERS[args.task](cfg, out=sys.stdout)
        return 0
    except (DyncoreError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
