"""Numpy restatement of the reference engine (TEST INFRASTRUCTURE ONLY).

Restates, for checking the CUDA backend, the behaviour of:
  * graph engine      /root/reference/pkg/src/dyncore/graph.py:69-172
  * op catalog        /root/reference/pkg/src/dyncore/ops.py:98-527
  * parameters        /root/reference/pkg/src/dyncore/params.py:55-119
  * trainers          /root/reference/pkg/src/dyncore/trainers.py:21-98
  * LSTM/GRU/simple   /root/reference/pkg/src/dyncore/builders.py:29-143
  * Tree-LSTM         /root/reference/pkg/src/dyncore/builders.py:213-274
  * DP averaging      /root/reference/pkg/src/dyncore/parallel.py:55-65,105-109

Structure differs from the reference on purpose: every node value is a 2-D
(batch, elem) float array, an op is a (shape, forward, vjp) triple where the
vjp returns an un-reduced (batch_out, n_in) contribution and the engine folds
broadcast batches, and there is no arena (pool accounting is a product concern,
pinned separately by golden counters).  Parity with the real reference is pinned
by tests/golden/*.npz (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32


class OracleError(Exception):
    pass


# ---------------------------------------------------------------------------
# shapes                                                   (tensor.py:19-47)
# ---------------------------------------------------------------------------


class Shape:
    __slots__ = ("dims", "batch")

    def __init__(self, dims, batch=1):
        self.dims = tuple(int(d) for d in dims)
        self.batch = int(batch)

    def elem_size(self):
        return math.prod(self.dims)

    def size(self):
        return self.elem_size() * self.batch

    def __eq__(self, o):
        return isinstance(o, Shape) and o.dims == self.dims and o.batch == self.batch

    def __repr__(self):
        return f"Shape({list(self.dims)}, batch={self.batch})"


class Tensor:
    """(shape, flat data) pair, layout per tensor.py:1-6."""

    __slots__ = ("shape", "data")

    def __init__(self, shape, data):
        self.shape = shape
        self.data = data

    def elems(self):
        return self.data.reshape(self.shape.batch, self.shape.elem_size())


def from_values(shape, values, dtype=np.float64):
    return Tensor(shape, np.asarray(values, dtype=dtype).reshape(-1).copy())


def new_poolset(*_args, **kw):
    """Pools are a product concern; the oracle keeps only the dtype."""
    return np.dtype(kw.get("dtype", F32))


def poolset_from_mem_flag(_flag, dtype=F32):
    """bench/cli.py --mem pools (arena.py:105-107); the oracle keeps the dtype."""
    return np.dtype(dtype)


def col_major(flat_elem, dims):
    """Element view following the layout contract (tensor.py:1-6, :65-68)."""
    return flat_elem.reshape(dims, order="F")


def _bcast(shapes):
    b = 1
    for s in shapes:
        if s.batch != 1 and b != 1 and s.batch != b:
            raise OracleError("batch mismatch")
        b = max(b, s.batch)
    return b


def _row(a, j):
    """Row j of a (batch, n) array with batch-1 replication (ops.py:60-66)."""
    return a[0] if a.shape[0] == 1 else a[j]


def _sig(x):
    # ops.py:78-83: clip +-60 before exp
    return F32(1.0) / (F32(1.0) + np.exp(-np.clip(x, -60.0, 60.0)))


# ---------------------------------------------------------------------------
# op table: kind -> (shape(aux, in_shapes), fwd(ins, aux, out_batch), vjp(i, ins, out, g, aux))
# ins/out/g are 2-D (batch, elem) float32 arrays.  vjp returns the contribution
# for input i with out's batch; the engine sums it down to a batch-1 input.
# ---------------------------------------------------------------------------

OPS = {}


def _same(aux, s):
    return Shape(s[0].dims, s[0].batch)


def _pair(aux, s):
    if s[0].dims != s[1].dims:
        raise OracleError("dims differ")
    return Shape(s[0].dims, _bcast(s))


def _expand(a, b):
    return a if a.shape[0] == b else np.broadcast_to(a, (b, a.shape[1]))


OPS["add"] = (
    _pair,
    lambda ins, aux, b: _expand(ins[0], b) + _expand(ins[1], b),
    lambda i, ins, out, g, aux: g,
)
OPS["cmult"] = (
    _pair,
    lambda ins, aux, b: _expand(ins[0], b) * _expand(ins[1], b),
    lambda i, ins, out, g, aux: g * _expand(ins[1 - i], g.shape[0]),
)
OPS["scalar_mul"] = (
    _same,
    lambda ins, aux, b: ins[0] * F32(aux),
    lambda i, ins, out, g, aux: F32(aux) * g,
)
OPS["tanh"] = (
    _same,
    lambda ins, aux, b: np.tanh(ins[0]),
    lambda i, ins, out, g, aux: (F32(1.0) - out * out) * g,
)
OPS["logistic"] = (
    _same,
    lambda ins, aux, b: _sig(ins[0]),
    lambda i, ins, out, g, aux: out * (F32(1.0) - out) * g,
)


def _softmax_rows(x):
    e = np.exp(x - x.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def _softmax_vjp(i, ins, out, g, aux):
    return out * (g - (g * out).sum(axis=1, keepdims=True))


OPS["softmax"] = (_same, lambda ins, aux, b: _softmax_rows(ins[0]), _softmax_vjp)


def _pnls_fwd(ins, aux, b):
    x = ins[0]
    labels = [aux] if isinstance(aux, int) else list(aux)
    m = x.max(axis=1)
    lse = m + np.log(np.exp(x - m[:, None]).sum(axis=1))
    return (lse - x[np.arange(len(labels)), labels])[:, None]


def _pnls_vjp(i, ins, out, g, aux):
    labels = [aux] if isinstance(aux, int) else list(aux)
    p = _softmax_rows(ins[0])
    p[np.arange(len(labels)), labels] -= F32(1.0)
    return g[:, :1] * p


OPS["pickneglogsoftmax"] = (lambda aux, s: Shape((1,)), _pnls_fwd, _pnls_vjp)
OPS["pickneglogsoftmax_batch"] = (lambda aux, s: Shape((1,), s[0].batch), _pnls_fwd, _pnls_vjp)
OPS["sum_batches"] = (
    lambda aux, s: Shape(s[0].dims, 1),
    lambda ins, aux, b: ins[0].sum(axis=0, keepdims=True),
    None,  # special-cased: replicate upstream across the batch
)


def _pick_fwd(ins, aux, b):
    lo, hi = aux
    return ins[0][:, lo:hi].copy()


def _pick_vjp(i, ins, out, g, aux):
    lo, hi = aux
    full = np.zeros((g.shape[0], ins[0].shape[1]), dtype=g.dtype)
    full[:, lo:hi] = g
    return full


OPS["pick_range"] = (lambda aux, s: Shape((aux[1] - aux[0],), s[0].batch), _pick_fwd, _pick_vjp)


def _concat_vjp(i, ins, out, g, aux):
    off = sum(x.shape[1] for x in ins[:i])
    return g[:, off : off + ins[i].shape[1]]


OPS["concatenate"] = (
    lambda aux, s: Shape((sum(x.dims[0] for x in s),), s[0].batch),
    lambda ins, aux, b: np.concatenate(ins, axis=1),
    _concat_vjp,
)


def _affine_shape(aux, s):
    return Shape(s[0].dims, _bcast(s))


def _affine_fwd(ins, aux, b):
    out = np.array(_expand(ins[0], b), dtype=ins[0].dtype)
    m = out.shape[1]
    for k in range(1, len(ins), 2):
        w, x = ins[k], ins[k + 1]
        n = x.shape[1]
        if w.shape[0] == 1:
            out += _expand(x, b) @ col_major(w[0], (m, n)).T
        else:
            for j in range(b):
                out[j] += col_major(w[j], (m, n)) @ _row(x, j)
    return out


def _affine_vjp(i, ins, out, g, aux):
    # ops.py:335-357 restated as a vjp: bias -> g; W -> g^T x (per batch row);
    # x -> g W.  W contributions are returned per batch row of g so the
    # engine's batch fold produces the sum over rows.
    if i == 0:
        return g
    k = ((i - 1) // 2) * 2 + 1
    w, x = ins[k], ins[k + 1]
    m, n = g.shape[1], x.shape[1]
    if i == k:
        if w.shape[0] == 1:
            xb = _expand(x, g.shape[0])
            if x.shape[0] == g.shape[0]:
                gw = g.T @ xb  # (m, n)
            else:
                gw = np.outer(g.sum(axis=0), x[0])
            return np.asarray(gw, dtype=g.dtype).reshape(1, m * n, order="F")
        rows = [np.outer(g[j], _row(x, j)).reshape(-1, order="F") for j in range(g.shape[0])]
        return np.stack(rows)
    if w.shape[0] == 1:
        if x.shape[0] == 1 and g.shape[0] > 1:
            return (g @ col_major(w[0], (m, n))).sum(axis=0, keepdims=True)
        return g @ col_major(w[0], (m, n))
    rows = [col_major(w[j], (m, n)).T @ g[j] for j in range(g.shape[0])]
    return np.stack(rows)


OPS["affine"] = (_affine_shape, _affine_fwd, _affine_vjp)


def _matmul_shape(aux, s):
    a, x = s
    m, n = a.dims
    dims = (m,) if len(x.dims) == 1 else (m, x.dims[1])
    return Shape(dims, _bcast(s))


def _matmul_fwd(ins, aux, b):
    a, x = ins
    a_dims, x_dims = aux
    m, n = a_dims
    rows = []
    for j in range(b):
        am = col_major(_row(a, j), (m, n))
        xm = col_major(_row(x, j), x_dims)
        rows.append((am @ xm).reshape(-1, order="F"))
    return np.stack(rows).astype(a.dtype)


def _matmul_vjp(i, ins, out, g, aux):
    a, x = ins
    (m, n), x_dims = aux
    p = 1 if len(x_dims) == 1 else x_dims[1]
    rows = []
    for j in range(g.shape[0]):
        am = col_major(_row(a, j), (m, n))
        xm = col_major(_row(x, j), x_dims).reshape(n, p, order="F")
        gm = col_major(g[j], (m, p))
        r = gm @ xm.T if i == 0 else am.T @ gm
        rows.append(r.reshape(-1, order="F"))
    return np.stack(rows).astype(g.dtype)


OPS["matmul"] = (_matmul_shape, _matmul_fwd, _matmul_vjp)

LEAVES = ("input", "parameter", "lookup", "lookup_batch")


# ---------------------------------------------------------------------------
# persistent state                                        (params.py:55-119)
# ---------------------------------------------------------------------------


class Parameter:
    def __init__(self, name, dims, values):
        self.name = name
        self.dims = tuple(dims)
        self.values = values  # flat, column-major element order
        self.gradient = np.zeros_like(values)


class LookupParameter:
    def __init__(self, name, rows, dim, values):
        self.name = name
        self.rows = rows
        self.dim = dim
        self.values = values  # (rows, dim) row-major
        self.gradient = np.zeros_like(values)
        self.touched = set()


class Model:
    def __init__(self, pools=None, seed=0, init_zero=False, dtype=F32):
        dtype = pools if isinstance(pools, np.dtype) else dtype
        self.rng = np.random.default_rng(seed)
        self.init_zero = init_zero
        self.dtype = np.dtype(dtype)
        self.parameters = []
        self.lookups = []

    def _name(self, name, prefix):
        return name if name is not None else f"{prefix}{len(self.parameters) + len(self.lookups)}"

    def add_parameters(self, dims, name=None):
        dims = (dims,) if isinstance(dims, int) else tuple(dims)
        size = math.prod(dims)
        vals = np.zeros(size, dtype=self.dtype)
        if not self.init_zero:
            # Glorot uniform, vectors use fan_in 1 (params.py:90-95)
            fan_in = dims[1] if len(dims) > 1 else 1
            bound = np.sqrt(6.0 / (fan_in + dims[0]))
            vals[:] = self.rng.uniform(-bound, bound, size)
        p = Parameter(self._name(name, "p"), dims, vals)
        self.parameters.append(p)
        return p

    def add_lookup_parameters(self, rows, dim, name=None):
        vals = np.zeros((rows, dim), dtype=self.dtype)
        if not self.init_zero:
            vals[:] = self.rng.uniform(-0.1, 0.1, (rows, dim))  # params.py:106-107
        lp = LookupParameter(self._name(name, "lp"), rows, dim, vals)
        self.lookups.append(lp)
        return lp

    def zero_gradients(self):
        for p in self.parameters:
            p.gradient[:] = 0
        for lp in self.lookups:
            lp.gradient[:] = 0
            lp.touched.clear()


# ---------------------------------------------------------------------------
# graph                                                      (graph.py:69-172)
# ---------------------------------------------------------------------------


class Expr:
    __slots__ = ("g", "i", "gen")

    def __init__(self, g, i, gen):
        self.g, self.i, self.gen = g, i, gen

    @property
    def shape(self):
        return self.g.shapes[self.i]


class ComputationGraph:
    def __init__(self, pools=None, dtype=F32):
        self.dtype = pools if isinstance(pools, np.dtype) else np.dtype(dtype)
        self.generation = 0
        self.forward_calls = 0
        self.sink = None  # None -> model storage; else a Slots object
        self._clear()

    def _clear(self):
        self.kinds, self.inputs, self.shapes, self.auxs = [], [], [], []
        self.vals, self.grads = [], []
        self.watermark = -1

    def renew(self):
        self._clear()
        self.generation += 1

    def _check(self, e):
        if e.g is not self or e.gen != self.generation:
            raise OracleError("stale expression")

    def add(self, kind, inputs=(), aux=None):
        for e in inputs:
            self._check(e)
        in_idx = tuple(e.i for e in inputs)
        in_shapes = [self.shapes[i] for i in in_idx]
        if kind == "input":
            shape = Shape(aux.shape.dims, aux.shape.batch)
        elif kind == "parameter":
            shape = Shape(aux.dims)
        elif kind == "lookup":
            shape = Shape((aux[0].dim,))
        elif kind == "lookup_batch":
            shape = Shape((aux[0].dim,), len(aux[1]))
        else:
            if kind == "matmul":
                aux = (in_shapes[0].dims, in_shapes[1].dims)
            shape = OPS[kind][0](aux, in_shapes)
        self.kinds.append(kind)
        self.inputs.append(in_idx)
        self.shapes.append(shape)
        self.auxs.append(aux)
        self.vals.append(None)
        self.grads.append(None)
        return Expr(self, len(self.kinds) - 1, self.generation)

    def _forward(self, upto):
        for i in range(self.watermark + 1, upto + 1):
            kind, aux, s = self.kinds[i], self.auxs[i], self.shapes[i]
            if kind == "input":
                v = np.asarray(aux.data, dtype=self.dtype).reshape(s.batch, s.elem_size()).copy()
            elif kind == "parameter":
                v = aux.values.reshape(1, -1)  # alias (ops.py:117)
            elif kind == "lookup":
                v = aux[0].values[aux[1]][None, :].copy()
            elif kind == "lookup_batch":
                v = aux[0].values[list(aux[1])].copy()
            else:
                ins = [self.vals[j] for j in self.inputs[i]]
                v = np.ascontiguousarray(OPS[kind][1](ins, aux, s.batch), dtype=self.dtype)
            self.vals[i] = v
            self.forward_calls += 1
        self.watermark = max(self.watermark, upto)

    def forward_to(self, e):
        self._check(e)
        self._forward(e.i)

    def value(self, e):
        """Flat copy in layout order (graph.py:132-135)."""
        self._check(e)
        self._forward(e.i)
        return Tensor(self.shapes[e.i], self.vals[e.i].reshape(-1).copy())

    def backward(self, e):
        self._check(e)
        s = self.shapes[e.i]
        if s.elem_size() != 1 or s.batch != 1:
            raise OracleError("non-scalar loss")
        self._forward(e.i)
        n = e.i + 1
        # all nodes <= loss get a fresh zero slot and are swept (graph.py:146-164)
        grads = [np.zeros((self.shapes[i].batch, self.shapes[i].elem_size()), dtype=self.dtype) for i in range(n)]
        grads[e.i][0, 0] += 1.0
        for i in range(e.i, -1, -1):
            kind, aux, g = self.kinds[i], self.auxs[i], grads[i]
            if kind in LEAVES:
                self._flush(kind, aux, g)
                continue
            ins = [self.vals[j] for j in self.inputs[i]]
            for k, j in enumerate(self.inputs[i]):
                if kind == "sum_batches":
                    grads[j] += g
                    continue
                c = OPS[kind][2](k, ins, self.vals[i], g, aux)
                if grads[j].shape[0] == c.shape[0]:
                    grads[j] += c
                else:
                    grads[j] += c.sum(axis=0, keepdims=True)
        self.grads = grads + [None] * (len(self.kinds) - n)

    def _flush(self, kind, aux, g):
        sink = self.sink
        if kind == "parameter":
            if sink is None:
                aux.gradient += g.reshape(-1)
            else:
                sink.params[id(aux)] += g.reshape(-1)
        elif kind == "lookup":
            lp, row = aux
            if sink is None:
                lp.gradient[row] += g[0]
                lp.touched.add(row)
            else:
                sink.lookups[id(lp)][row] += g[0]
        elif kind == "lookup_batch":
            lp, ids = aux
            target = lp.gradient if sink is None else sink.lookups[id(lp)]
            np.add.at(target, list(ids), g)  # repeated ids accumulate
            if sink is None:
                lp.touched.update(ids)

    def gradient(self, e):
        self._check(e)
        return Tensor(self.shapes[e.i], self.grads[e.i].reshape(-1).copy())


# ---------------------------------------------------------------------------
# expression surface                                        (ops.py:535-611)
# ---------------------------------------------------------------------------


class ops:  # noqa: N801 - namespace mirroring the reference module
    @staticmethod
    def input(g, t):
        return g.add("input", (), t)

    @staticmethod
    def parameter(g, p):
        return g.add("parameter", (), p)

    @staticmethod
    def lookup(g, lp, idx):
        return g.add("lookup", (), (lp, int(idx)))

    @staticmethod
    def lookup_batch(g, lp, ids):
        return g.add("lookup_batch", (), (lp, tuple(int(i) for i in ids)))

    @staticmethod
    def add(a, b):
        return a.g.add("add", (a, b))

    @staticmethod
    def cmult(a, b):
        return a.g.add("cmult", (a, b))

    @staticmethod
    def scalar_mul(a, c):
        return a.g.add("scalar_mul", (a,), float(c))

    @staticmethod
    def tanh(a):
        return a.g.add("tanh", (a,))

    @staticmethod
    def logistic(a):
        return a.g.add("logistic", (a,))

    @staticmethod
    def softmax(a):
        return a.g.add("softmax", (a,))

    @staticmethod
    def matmul(a, x):
        return a.g.add("matmul", (a, x))

    @staticmethod
    def affine(*xs):
        return xs[0].g.add("affine", xs)

    @staticmethod
    def concatenate(parts):
        parts = tuple(parts)
        return parts[0].g.add("concatenate", parts)

    @staticmethod
    def pick_range(a, lo, hi):
        return a.g.add("pick_range", (a,), (int(lo), int(hi)))

    @staticmethod
    def pickneglogsoftmax(a, label):
        return a.g.add("pickneglogsoftmax", (a,), int(label))

    @staticmethod
    def pickneglogsoftmax_batch(a, labels):
        return a.g.add("pickneglogsoftmax_batch", (a,), tuple(int(x) for x in labels))

    @staticmethod
    def sum_batches(a):
        return a.g.add("sum_batches", (a,))


# ---------------------------------------------------------------------------
# trainers                                                (trainers.py:21-98)
# ---------------------------------------------------------------------------

DEFAULT_LR = {"sgd": 0.1, "momentum": 0.01, "adagrad": 0.1, "adam": 0.001}


class Trainer:
    def __init__(self, model, rule="sgd", lr=None, momentum=0.9, adagrad_eps=1e-20,
                 beta1=0.9, beta2=0.999, adam_eps=1e-8, sparse=True):
        self.model, self.rule = model, rule
        self.lr = DEFAULT_LR[rule] if lr is None else float(lr)
        self.momentum, self.adagrad_eps = momentum, adagrad_eps
        self.beta1, self.beta2, self.adam_eps = beta1, beta2, adam_eps
        self.sparse = sparse
        self.t = 0
        self.state = {}

    def _slot(self, key, like, name):
        d = self.state.setdefault(name, {})
        if key not in d:
            d[key] = np.zeros_like(like)
        return d[key]

    def _rule(self, th, g, key, rows):
        lr = self.lr
        sel = slice(None) if rows is None else rows
        if self.rule == "sgd":
            th[sel] = th[sel] - lr * g[sel]
        elif self.rule == "momentum":
            v = self._slot(key, th, "vel")
            v[sel] = self.momentum * v[sel] - lr * g[sel]
            th[sel] = th[sel] + v[sel]
        elif self.rule == "adagrad":
            sq = self._slot(key, th, "sq")
            sq[sel] = sq[sel] + g[sel] * g[sel]
            th[sel] = th[sel] - lr * g[sel] / (np.sqrt(sq[sel]) + self.adagrad_eps)
        else:
            m1, m2 = self._slot(key, th, "m1"), self._slot(key, th, "m2")
            m1[sel] = self.beta1 * m1[sel] + (1.0 - self.beta1) * g[sel]
            m2[sel] = self.beta2 * m2[sel] + (1.0 - self.beta2) * (g[sel] * g[sel])
            mhat = m1[sel] / (1.0 - self.beta1 ** self.t)
            vhat = m2[sel] / (1.0 - self.beta2 ** self.t)
            th[sel] = th[sel] - lr * mhat / (np.sqrt(vhat) + self.adam_eps)

    def update(self):
        if self.rule == "adam":
            self.t += 1
        for p in self.model.parameters:
            self._rule(p.values, p.gradient, id(p), None)
        for lp in self.model.lookups:
            if not self.sparse:
                self._rule(lp.values, lp.gradient, id(lp), None)
            elif lp.touched:
                self._rule(lp.values, lp.gradient, id(lp), np.array(sorted(lp.touched)))
        self.model.zero_gradients()


# ---------------------------------------------------------------------------
# data-parallel averaging                                 (parallel.py:30-109)
# ---------------------------------------------------------------------------


class Slots:
    def __init__(self, model):
        self.params = {id(p): np.zeros_like(p.values) for p in model.parameters}
        self.lookups = {id(lp): np.zeros_like(lp.values) for lp in model.lookups}


def dp_step(model, trainer, graphs_and_losses_fn, n_ranks):
    """Deterministic DP restatement: each rank shard backprops
    into its own slot set, slots are averaged over the R participants, loaded
    into the model, touched = union of shard lookups, then one update."""
    slots, touched, losses = [], {}, []
    for r in range(n_ranks):
        g, loss = graphs_and_losses_fn(r)
        s = Slots(model)
        g.sink = s
        g.backward(loss)
        losses.append(float(g.value(loss).data[0]))
        slots.append(s)
        for i in range(loss.i + 1):
            if g.kinds[i] in ("lookup", "lookup_batch"):
                lp = g.auxs[i][0]
                ids = [g.auxs[i][1]] if g.kinds[i] == "lookup" else list(g.auxs[i][1])
                touched.setdefault(id(lp), set()).update(ids)
    n = float(len(slots))
    for p in model.parameters:
        p.gradient[:] = sum(s.params[id(p)] for s in slots) / n
    for lp in model.lookups:
        lp.gradient[:] = sum(s.lookups[id(lp)] for s in slots) / n
        lp.touched = set(touched.get(id(lp), set()))
    trainer.update()
    return losses


# ---------------------------------------------------------------------------
# builders                                                (builders.py:29-274)
# ---------------------------------------------------------------------------

GATES = {"simple": 1, "lstm": 4, "gru": 3}


class RNNBuilder:
    def __init__(self, model, layers, input_dim, hidden_dim, cell="lstm", name=None):
        prefix = name if name is not None else f"{cell}{len(model.parameters) + len(model.lookups)}"
        self.cell, self.layers, self.hid = cell, layers, hidden_dim
        rows = GATES[cell] * hidden_dim
        self.params = []
        for layer in range(layers):
            ind = input_dim if layer == 0 else hidden_dim
            wx = model.add_parameters((rows, ind), f"{prefix}.l{layer}.Wx")
            wh = model.add_parameters((rows, hidden_dim), f"{prefix}.l{layer}.Wh")
            b = model.add_parameters((rows,), f"{prefix}.l{layer}.b")
            if cell == "lstm":
                b.values[hidden_dim : 2 * hidden_dim] = 0.0
            self.params.append((wx, wh, b))
        self._cache = {}

    def _pe(self, g):
        c = self._cache.get(id(g))
        if c is None or c[0] != g.generation:
            c = (g.generation, [tuple(ops.parameter(g, p) for p in lp) for lp in self.params])
            self._cache[id(g)] = c
        return c[1]

    def initial_state(self, g):
        zero = Tensor(Shape((self.hid,)), np.zeros(self.hid, dtype=g.dtype))
        hs = [ops.input(g, zero) for _ in range(self.layers)]
        cs = [ops.input(g, zero) for _ in range(self.layers)] if self.cell == "lstm" else None
        return RNNState(self, g, hs, cs)

    def step(self, st, x):
        g, H = st.g, self.hid
        pe = self._pe(g)
        hs, cs, inp = [], [], x
        for layer in range(self.layers):
            wx, wh, b = pe[layer]
            h = st.hs[layer]
            if self.cell == "simple":
                nh = ops.tanh(ops.affine(b, wx, inp, wh, h))
            elif self.cell == "lstm":
                gates = ops.affine(b, wx, inp, wh, h)
                i_g = ops.logistic(ops.pick_range(gates, 0, H))
                f_g = ops.logistic(ops.pick_range(gates, H, 2 * H))
                o_g = ops.logistic(ops.pick_range(gates, 2 * H, 3 * H))
                g_g = ops.tanh(ops.pick_range(gates, 3 * H, 4 * H))
                nc = ops.add(ops.cmult(f_g, st.cs[layer]), ops.cmult(i_g, g_g))
                nh = ops.cmult(o_g, ops.tanh(nc))
                cs.append(nc)
            else:
                zr = ops.affine(b, wx, inp, wh, h)
                z = ops.logistic(ops.pick_range(zr, 0, H))
                r = ops.logistic(ops.pick_range(zr, H, 2 * H))
                cx = ops.pick_range(ops.affine(b, wx, inp), 2 * H, 3 * H)
                ch = ops.pick_range(ops.matmul(wh, ops.cmult(r, h)), 2 * H, 3 * H)
                cand = ops.tanh(ops.add(cx, ch))
                ones = Tensor(Shape((H,)), np.ones(H, dtype=g.dtype))
                keep = ops.add(ops.input(g, ones), ops.scalar_mul(z, -1.0))
                nh = ops.add(ops.cmult(keep, h), ops.cmult(z, cand))
            hs.append(nh)
            inp = nh
        return RNNState(self, g, hs, cs if self.cell == "lstm" else None)


class RNNState:
    def __init__(self, b, g, hs, cs):
        self.b, self.g, self.hs, self.cs = b, g, hs, cs

    def add_input(self, x):
        return self.b.step(self, x)

    def output(self):
        return self.hs[-1]

    def transduce(self, xs):
        outs, st = [], self
        for x in xs:
            st = st.add_input(x)
            outs.append(st.output())
        return outs


class TreeLSTM:
    """Gate order i, f1, f2, o, g (builders.py:213-274)."""

    def __init__(self, model, word_vocab, input_dim, hidden_dim, name=None):
        name = name if name is not None else f"treelstm{len(model.parameters) + len(model.lookups)}"
        self.w2i = dict(word_vocab)
        vocab_size = len(self.w2i)
        rows = 5 * hidden_dim
        self.hid = hidden_dim
        self.Wx = model.add_parameters((rows, input_dim), f"{name}.Wx")
        self.U1 = model.add_parameters((rows, hidden_dim), f"{name}.U1")
        self.U2 = model.add_parameters((rows, hidden_dim), f"{name}.U2")
        self.b = model.add_parameters((rows,), f"{name}.b")
        self.b.values[hidden_dim : 3 * hidden_dim] = 0.0
        self.E = model.add_lookup_parameters(max(1, vocab_size), input_dim, f"{name}.E")
        self._cache = {}

    def _pe(self, g):
        c = self._cache.get(id(g))
        if c is None or c[0] != g.generation:
            c = (g.generation, tuple(ops.parameter(g, p) for p in (self.Wx, self.U1, self.U2, self.b)))
            self._cache[id(g)] = c
        return c[1]

    def _compose(self, gates, terms):
        H = self.hid
        i_g = ops.logistic(ops.pick_range(gates, 0, H))
        o_g = ops.logistic(ops.pick_range(gates, 3 * H, 4 * H))
        g_g = ops.tanh(ops.pick_range(gates, 4 * H, 5 * H))
        c = ops.cmult(i_g, g_g)
        for t in terms:
            c = ops.add(c, t)
        return ops.cmult(o_g, ops.tanh(c)), c

    def encode(self, g, tree):
        wx, u1, u2, b = self._pe(g)
        H = self.hid
        if tree.token is not None:
            x = ops.lookup(g, self.E, self.w2i.get(tree.token, 0))
            return self._compose(ops.affine(b, wx, x), [])
        if len(tree.children) == 1:
            return self.encode(g, tree.children[0])
        h1, c1 = self.encode(g, tree.children[0])
        h2, c2 = self.encode(g, tree.children[1])
        gates = ops.affine(b, u1, h1, u2, h2)
        f1 = ops.logistic(ops.pick_range(gates, H, 2 * H))
        f2 = ops.logistic(ops.pick_range(gates, 2 * H, 3 * H))
        return self._compose(gates, [ops.cmult(f1, c1), ops.cmult(f2, c2)])


class TreeNode:
    """leaf(token) | unary(child) | binary(left, right) (builders.py:146-180)."""

    __slots__ = ("token", "children", "label")

    def __init__(self, token=None, children=(), label=None):
        self.token, self.children, self.label = token, tuple(children), label

    @staticmethod
    def leaf(token, label=None):
        return TreeNode(token=token, label=label)

    @staticmethod
    def unary(child, label=None):
        return TreeNode(children=(child,), label=label)

    @staticmethod
    def binary(left, right, label=None):
        return TreeNode(children=(left, right), label=label)

    def is_leaf(self):
        return self.token is not None


class TreeRNN:
    """builders.py:183-210: leaf -> E row, unary -> child, binary ->
    tanh(W [h_l; h_r]); parameters W then E; one W node per graph."""

    def __init__(self, model, word_vocab, hidden_dim, name=None):
        name = name if name is not None else f"treernn{len(model.parameters) + len(model.lookups)}"
        self.w2i = dict(word_vocab)
        self.W = model.add_parameters((hidden_dim, 2 * hidden_dim), f"{name}.W")
        self.E = model.add_lookup_parameters(max(1, len(self.w2i)), hidden_dim, f"{name}.E")
        self._cache = {}

    def encode(self, g, tree):
        if tree.token is not None:
            return ops.lookup(g, self.E, self.w2i.get(tree.token, 0))
        if len(tree.children) == 1:
            return self.encode(g, tree.children[0])
        a = self.encode(g, tree.children[0])
        b = self.encode(g, tree.children[1])
        c = self._cache.get(id(g))
        if c is None or c[0] != g.generation:
            c = (g.generation, ops.parameter(g, self.W))
            self._cache[id(g)] = c
        return ops.tanh(ops.matmul(c[1], ops.concatenate([a, b])))


class ClassFactoredSoftmax:
    """builders.py:282-378: classes renumbered densely in sorted raw-id order,
    words slotted in map order; parameters Wc, bc, Ww[0..C), bw[0..C); the
    class and word score affines are built once per (generation, h.index);
    -log p(w) = pnls(class scores, c) + pnls(word scores of c, slot)."""

    def __init__(self, model, hidden_dim, word_to_class, name=None):
        name = name if name is not None else f"cfsm{len(model.parameters) + len(model.lookups)}"
        dense = {raw: i for i, raw in enumerate(sorted(set(word_to_class.values())))}
        self.members = [[] for _ in dense]
        self.slot = {}
        for w, raw in word_to_class.items():
            c = dense[raw]
            self.slot[w] = (c, len(self.members[c]))
            self.members[c].append(w)
        C = len(dense)
        self.Wc = model.add_parameters((C, hidden_dim), f"{name}.Wc")
        self.bc = model.add_parameters((C,), f"{name}.bc")
        self.Ww = [model.add_parameters((len(m), hidden_dim), f"{name}.Ww{c}") for c, m in enumerate(self.members)]
        self.bw = [model.add_parameters((len(m),), f"{name}.bw{c}") for c, m in enumerate(self.members)]
        self._cache = {}

    def _scores(self, g, h):
        key = (g.generation, h.i)
        c = self._cache.get(id(g))
        if c is None or c[0] != key:
            cs = ops.affine(ops.parameter(g, self.bc), ops.parameter(g, self.Wc), h)
            ws = [ops.affine(ops.parameter(g, self.bw[k]), ops.parameter(g, self.Ww[k]), h)
                  for k in range(len(self.members))]
            c = (key, (cs, ws))
            self._cache[id(g)] = c
        return c[1]

    def neg_log_softmax(self, g, h, word):
        c, k = self.slot[word]
        cs, ws = self._scores(g, h)
        return ops.add(ops.pickneglogsoftmax(cs, c), ops.pickneglogsoftmax(ws[c], k))

