"""Scripting frontend (the reference's `dyngraph`, pkg/frontend/src/dyngraph/
__init__.py) over this backend.

One implicit global graph renewed per example with `renew_cg()`; expressions
overload `+` and `*` (matrix product / scalar scaling), lookup tables support
bracket indexing.  Every call delegates to exactly one core operation, so
the scripts of the reference (its Fig. 1 two-word classifier and Fig. 5 tree
encoder transliterations, fetests/test_programs.py) run unchanged on the B200
executor: `import paper_1701_03980_b200.dyngraph as dy`.

`Frontend(core)` binds the same surface to any engine with the reference's
core API (this package, or the numpy oracle for parity checks); the module
level names are a Frontend bound to this package.
"""

from __future__ import annotations

import numpy as np


class Frontend:
    """The scripting surface bound to one core engine (module-like object)."""

    def __init__(self, core):
        self.core = core
        self.ops = core.ops
        self._ctx = {"mem": "64", "seed": 0, "pools": None, "cg": None}
        fe = self

        class Expression:
            """Thin handle over a core expression; staleness checks stay in the core."""

            __slots__ = ("inner",)

            def __init__(self, inner):
                self.inner = inner

            def value(self):
                t = fe._cg().value(self.inner)
                if t.shape.size() == 1:
                    return float(t.data[0])
                return t.data.copy()

            def npvalue(self) -> np.ndarray:
                t = fe._cg().value(self.inner)
                if len(t.shape.dims) > 1:
                    return np.array(t.elem(0)) if t.shape.batch == 1 else t.data.copy()
                return t.data.copy()

            def forward(self) -> None:
                fe._cg().forward_to(self.inner)

            def backward(self) -> None:
                fe._cg().backward(self.inner)

            def __add__(self, other):
                if isinstance(other, Expression):
                    return Expression(fe.ops.add(self.inner, other.inner))
                if other == 0:  # sum() starts from 0
                    return self
                return NotImplemented

            __radd__ = __add__

            def __mul__(self, other):
                if isinstance(other, Expression):
                    return Expression(fe.ops.matmul(self.inner, other.inner))
                return Expression(fe.ops.scalar_mul(self.inner, float(other)))

            def __rmul__(self, other):
                return Expression(fe.ops.scalar_mul(self.inner, float(other)))

        class Parameters:
            """Persistent parameter; parameter() turns it into an expression."""

            __slots__ = ("core",)

            def __init__(self, core_param):
                self.core = core_param

        class LookupParameters:
            """Embedding table; indexing emits a lookup into the live graph."""

            __slots__ = ("core",)

            def __init__(self, core_table):
                self.core = core_table

            def __getitem__(self, index: int):
                return Expression(fe.ops.lookup(fe._cg(), self.core, int(index)))

        class Model:
            def __init__(self):
                self.core = fe.core.Model(fe._pools(), seed=fe._ctx["seed"])

            def add_parameters(self, dims):
                return Parameters(self.core.add_parameters(dims))

            def add_lookup_parameters(self, dims):
                rows, dim = dims
                return LookupParameters(self.core.add_lookup_parameters(rows, dim))

        class _Trainer:
            def __init__(self, m, rule, lr=None, **kw):
                self.core = fe.core.Trainer(m.core, rule, lr, **kw)

            def update(self) -> None:
                self.core.update()

        class SimpleSGDTrainer(_Trainer):
            def __init__(self, m, learning_rate: float = 0.1):
                super().__init__(m, "sgd", learning_rate)

        class MomentumSGDTrainer(_Trainer):
            def __init__(self, m, learning_rate: float = 0.01, mom: float = 0.9):
                super().__init__(m, "momentum", learning_rate, momentum=mom)

        class AdagradTrainer(_Trainer):
            def __init__(self, m, learning_rate: float = 0.1, eps: float = 1e-20):
                super().__init__(m, "adagrad", learning_rate, adagrad_eps=eps)

        class AdamTrainer(_Trainer):
            def __init__(self, m, alpha: float = 0.001, beta_1: float = 0.9, beta_2: float = 0.999,
                         eps: float = 1e-8):
                super().__init__(m, "adam", alpha, beta1=beta_1, beta2=beta_2, adam_eps=eps)

        self.Expression = Expression
        self.Parameters = Parameters
        self.LookupParameters = LookupParameters
        self.Model = Model
        self.model = Model  # both spellings appear in scripts
        self.SimpleSGDTrainer = SimpleSGDTrainer
        self.MomentumSGDTrainer = MomentumSGDTrainer
        self.AdagradTrainer = AdagradTrainer
        self.AdamTrainer = AdamTrainer
        self.inputVector = self.vectorInput

    # -- global context ----------------------------------------------------

    def init(self, mem: str = "64", seed: int = 0) -> None:
        """Pool sizes (the reference --mem flag) and model seed; resets the context."""
        self._ctx.update(mem=str(mem), seed=int(seed), pools=None, cg=None)

    def _pools(self):
        if self._ctx["pools"] is None:
            make = getattr(self.core, "poolset_from_mem_flag", None)
            self._ctx["pools"] = make(self._ctx["mem"]) if make else self.core.new_poolset()
        return self._ctx["pools"]

    def _cg(self):
        if self._ctx["cg"] is None:
            self._ctx["cg"] = self.core.ComputationGraph(self._pools())
        return self._ctx["cg"]

    def renew_cg(self) -> None:
        self._cg().renew()

    # -- expression surface --------------------------------------------------

    def parameter(self, p):
        return self.Expression(self.ops.parameter(self._cg(), p.core))

    def lookup(self, lp, index: int):
        return lp[index]

    def vectorInput(self, values):  # noqa: N802 - scripting-surface name
        arr = np.asarray(values, dtype=np.float64).reshape(-1)
        t = self.core.from_values(self.core.Shape((arr.shape[0],)), arr)
        return self.Expression(self.ops.input(self._cg(), t))

    def concatenate(self, parts):
        return self.Expression(self.ops.concatenate([p.inner for p in parts]))

    def softmax(self, e):
        return self.Expression(self.ops.softmax(e.inner))

    def tanh(self, e):
        return self.Expression(self.ops.tanh(e.inner))

    def logistic(self, e):
        return self.Expression(self.ops.logistic(e.inner))

    def pickneglogsoftmax(self, e, label: int):
        return self.Expression(self.ops.pickneglogsoftmax(e.inner, int(label)))


def _bind_module():
    import sys

    from . import __name__ as pkg_name

    fe = Frontend(sys.modules[pkg_name])
    names = ["init", "renew_cg", "parameter", "lookup", "vectorInput", "inputVector", "concatenate", "softmax",
             "tanh", "logistic", "pickneglogsoftmax", "Expression", "Parameters", "LookupParameters", "Model",
             "model", "SimpleSGDTrainer", "MomentumSGDTrainer", "AdagradTrainer", "AdamTrainer"]
    mod = sys.modules[__name__]
    for n in names:
        setattr(mod, n, getattr(fe, n))
    mod._FRONTEND = fe
    return names


__all__ = ["Frontend"] + _bind_module()
