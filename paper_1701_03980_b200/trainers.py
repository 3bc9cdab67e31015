"""Online update rules of the drop-in API (pkg/src/dyncore/trainers.py:21-98),
executed by the native trainer: one multi-tensor launch applies the dense rule
to every dense parameter (and to every lookup row when sparse is off), one
launch per lookup table applies it to the sorted touched rows; gradients are
zeroed in the same pass and touched sets cleared (Model.zero_gradients)."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from . import device as _dev
from .errors import BadShape
from .params import Model, materialize_pending

RULES = ("sgd", "momentum", "adagrad", "adam")
DEFAULT_LR = {"sgd": 0.1, "momentum": 0.01, "adagrad": 0.1, "adam": 0.001}
_SLOTS = {"sgd": (), "momentum": ("vel",), "adagrad": ("sq",), "adam": ("m1", "m2")}


class _SlotView:
    """dict-like view `trainer.m1[id(p)]` -> host copy of the device state."""

    def __init__(self, trainer, which: int):
        self._t = trainer
        self._w = which

    def __getitem__(self, key):
        x = self._t._by_id[key]
        dev = self._t._state[x.handle][self._w]
        arr = dev.cpu().numpy()
        return arr.reshape(x.rows, x.dim) if hasattr(x, "rows") else arr

    def __contains__(self, key):
        return key in self._t._by_id

    def keys(self):
        return self._t._by_id.keys()


class Trainer:
    def __init__(self, model: Model, rule: str = "sgd", lr: float | None = None, momentum: float = 0.9,
                 adagrad_eps: float = 1e-20, beta1: float = 0.9, beta2: float = 0.999, adam_eps: float = 1e-8,
                 sparse: bool = True):
        if rule not in RULES:
            raise BadShape(f"unknown trainer rule {rule!r}; pick one of {RULES}")
        self.model = model
        self.rule = rule
        self.lr = DEFAULT_LR[rule] if lr is None else float(lr)
        self.momentum = momentum
        self.adagrad_eps = adagrad_eps
        self.beta1 = beta1
        self.beta2 = beta2
        self.adam_eps = adam_eps
        self.sparse = sparse
        self._h = None
        self._t_host = 0
        self._state = {}  # handle -> (slot0 tensor | None, slot1 tensor | None)
        self._by_id = {}
        for i, name in enumerate(_SLOTS[rule]):
            setattr(self, name, _SlotView(self, i))

    @property
    def t(self) -> int:
        if self._h is None:
            return self._t_host
        v = ctypes.c_int64(0)
        _native.check(_native.lib().dg_trainer_step_count(self._h, ctypes.byref(v)))
        return int(v.value)

    @t.setter
    def t(self, value: int) -> None:
        self._t_host = int(value)
        if self._h is not None:
            _native.check(_native.lib().dg_trainer_set_step(self._h, int(value)))

    def set_sparse(self, flag: bool) -> None:
        self.sparse = flag

    def _native(self):
        lib = _native.lib()
        if self._h is None:
            h = ctypes.c_void_p()
            # (1 - beta) and eps are applied in fp32 like the reference's
            # float32 arrays combined with python floats (trainers.py:77-83)
            _native.check(lib.dg_trainer_create(RULES.index(self.rule), self.lr, self.momentum, self.adagrad_eps,
                                                self.beta1, self.beta2, self.adam_eps, int(self.sparse),
                                                ctypes.byref(h)))
            self._h = h
            _native.check(lib.dg_trainer_set_step(h, self._t_host))
        _native.check(lib.dg_trainer_set(self._h, self.lr, int(self.sparse)))
        n_slots = len(_SLOTS[self.rule])
        for x in list(self.model.parameters) + list(self.model.lookups):
            if x.handle in self._state:
                continue
            n = x.rows * x.dim if hasattr(x, "rows") else x.size
            s = tuple(_dev.zeros_f32(n) if k < n_slots else None for k in range(2))
            self._state[x.handle] = s
            self._by_id[id(x)] = x
            _native.check(lib.dg_trainer_attach(self._h, x.handle, _native.ptr(s[0]) if s[0] is not None else None,
                                                _native.ptr(s[1]) if s[1] is not None else None))
        return self._h

    def update(self) -> None:
        materialize_pending()
        h = self._native()
        _native.check(_native.lib().dg_trainer_update(h, _dev.stream_ptr()))
        # the native pass zeroes dense grads and touched rows; a table whose
        # gradient the host wrote directly may hold other rows: zero it whole
        # (Model.zero_gradients semantics, params.py:114-119)
        for lp in self.model.lookups:
            if lp._gm.host_written:
                lp._gm.dev.zero_()
                lp._gm.host_written = False
        _dev.bump_epoch()

    def __del__(self):
        try:
            if self._h is not None:
                _native.lib().dg_trainer_destroy(self._h)
        except Exception:  # noqa: BLE001
            pass
