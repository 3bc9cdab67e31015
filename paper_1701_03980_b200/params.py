"""Persistent trainable state of the drop-in API (pkg/src/dyncore/params.py).

Initialisation is the reference's: Glorot-uniform from default_rng(seed) in
registration order, lookup tables U(+-0.1) (params.py:63,90-107), computed on
the host.  Storage lives on the device: on first execution a Model lays its
dense parameters out in ONE flat value buffer and ONE flat gradient buffer
(a single NCCL all-reduce covers every dense gradient) and each lookup table
in its own (rows x dim) buffers; every tensor is registered with the native
executor by handle.

The reference exposes storage as live numpy views; here `.values.data`,
`.gradient.data`, `LookupParameter.values/.gradient` return host mirrors that
are downloaded lazily when the device is newer and re-uploaded before the next
device use after any host access (SURVEY 8(b) coherence contract).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native
from . import device as _dev
from .arena import PoolSet
from .errors import BadShape, DuplicateName, FileError, FormatError, RosterMismatch
from .tensor import Shape, Tensor

MAGIC = b"DYN1"
FORMAT_VERSION = 1
_PENDING_MODELS: set = set()


def materialize_pending() -> None:
    """Lay out device storage for models that gained parameters, then upload
    every host-dirtied mirror.  Called before any device operation."""
    if _PENDING_MODELS:
        for m in list(_PENDING_MODELS):
            m._materialize()
        _PENDING_MODELS.clear()
    _dev.flush_dirty()


class _Mirror:
    """Host mirror of one device tensor (values or gradient of a parameter)."""

    __slots__ = ("host", "dev", "epoch", "host_written", "__weakref__")

    def __init__(self, host: np.ndarray):
        self.host = host
        self.dev = None  # flat torch float32 tensor view
        self.epoch = -1  # device epoch the host copy reflects; -1 = host is the truth
        self.host_written = False  # host access since the last full device zeroing

    def pull(self) -> np.ndarray:
        if self.dev is not None and self.epoch >= 0 and self.epoch < _dev.EPOCH[0]:
            self.host.reshape(-1)[:] = self.dev.cpu().numpy()
            self.epoch = _dev.EPOCH[0]
        return self.host

    def touch_host(self) -> None:
        """Host may write: upload before the next device use."""
        if self.dev is not None:
            _dev.DIRTY.add(self)
        self.epoch = -1
        self.host_written = True

    def _upload(self) -> None:
        if self.dev is not None:
            t = _dev.torch()
            self.dev.copy_(t.from_numpy(np.ascontiguousarray(self.host.reshape(-1), dtype=np.float32)))
            self.epoch = _dev.EPOCH[0]

    def host_view(self) -> np.ndarray:
        self.pull()
        self.touch_host()
        return self.host


class _MirrorTensor(Tensor):
    """Tensor whose `.data` is a coherent host mirror of device storage."""

    __slots__ = ("_m",)

    def __init__(self, shape: Shape, mirror: _Mirror):
        object.__setattr__(self, "shape", shape)
        self._m = mirror

    @property
    def data(self):  # noqa: D401 - mirrors Tensor.data
        return self._m.host_view()

    @data.setter
    def data(self, value):
        self._m.host_view().reshape(-1)[:] = np.asarray(value).reshape(-1)

    def copy(self) -> Tensor:
        return Tensor(self.shape, np.array(self._m.pull().reshape(-1), dtype=np.float32))


class Parameter:
    __slots__ = ("name", "shape", "values", "gradient", "_vm", "_gm", "handle", "model", "_off")

    def __init__(self, name: str, shape: Shape, host_values: np.ndarray, model):
        self.name = name
        self.shape = shape
        self._vm = _Mirror(host_values)
        self._gm = _Mirror(np.zeros_like(host_values))
        self.values = _MirrorTensor(shape, self._vm)
        self.gradient = _MirrorTensor(shape, self._gm)
        self.handle = -1
        self.model = model
        self._off = 0

    def set_value(self, values) -> None:
        flat = np.asarray(values).reshape(-1)
        self._vm.host_view()[:] = flat

    @property
    def size(self) -> int:
        return self.shape.size()


class LookupParameter:
    """Embedding table, rows contiguous (params.py:41-52)."""

    __slots__ = ("name", "rows", "dim", "_vm", "_gm", "handle", "model", "_touched_host")

    def __init__(self, name: str, rows: int, dim: int, host_values: np.ndarray, model):
        self.name = name
        self.rows = rows
        self.dim = dim
        self._vm = _Mirror(host_values)
        self._gm = _Mirror(np.zeros_like(host_values))
        self.handle = -1
        self.model = model
        self._touched_host: set = set()

    @property
    def values(self) -> np.ndarray:
        return self._vm.host_view()

    @values.setter
    def values(self, v) -> None:
        self._vm.host_view()[:] = np.asarray(v).reshape(self.rows, self.dim)

    @property
    def gradient(self) -> np.ndarray:
        return self._gm.host_view()

    @gradient.setter
    def gradient(self, v) -> None:
        self._gm.host_view()[:] = np.asarray(v).reshape(self.rows, self.dim)

    @property
    def touched(self) -> set:
        if self.handle < 0:
            return set(self._touched_host)
        lib = _native.lib()
        n = ctypes.c_int64(0)
        _native.check(lib.dg_touched_count(self.handle, ctypes.byref(n)))
        ids = np.zeros(max(1, n.value), dtype=np.int64)
        _native.check(lib.dg_touched_get(self.handle, ids.ctypes.data, n.value))
        return set(int(i) for i in ids[: n.value])

    @touched.setter
    def touched(self, ids) -> None:
        ids = np.array(sorted(int(i) for i in ids), dtype=np.int64)
        if self.handle < 0:
            self._touched_host = set(int(i) for i in ids)
            return
        lib = _native.lib()
        _native.check(lib.dg_touched_clear(self.handle))
        if ids.size:
            _native.check(lib.dg_touched_add(self.handle, ids.ctypes.data, ids.size))


class Model:
    """Ordered parameter collection (params.py:55-119)."""

    def __init__(self, pools: PoolSet, seed: int = 0, init_zero: bool = False):
        self.pools = pools
        self.dtype = pools.dtype
        self.seed = seed
        self.init_zero = init_zero
        self.rng = np.random.default_rng(seed)
        self.parameters: list[Parameter] = []
        self.lookups: list[LookupParameter] = []
        self._names: set[str] = set()
        self._dense_vals = None
        self._dense_grads = None
        self._materialized = 0  # number of params laid out on the device

    # -- registration ------------------------------------------------------

    def _claim_name(self, name, prefix):
        if name is None:
            name = f"{prefix}{len(self.parameters) + len(self.lookups)}"
        if name in self._names:
            raise DuplicateName(f"parameter name {name!r} already registered")
        self._names.add(name)
        return name

    def _charge(self, count: int) -> None:
        # reference accounting: values then gradient from the parameters pool
        nbytes = count * 4
        self.pools.parameters.allocate(nbytes)
        self.pools.parameters.allocate(nbytes)

    def add_parameters(self, dims, name: str | None = None) -> Parameter:
        if isinstance(dims, int):
            dims = (dims,)
        shape = Shape(dims)
        name = self._claim_name(name, "p")
        self._charge(shape.size())
        vals = np.zeros(shape.size(), dtype=np.float32)
        if not self.init_zero:
            fan_out = dims[0]
            fan_in = dims[1] if len(dims) > 1 else 1
            bound = np.sqrt(6.0 / (fan_in + fan_out))
            vals[:] = self.rng.uniform(-bound, bound, shape.size())
        p = Parameter(name, shape, vals, self)
        self.parameters.append(p)
        _PENDING_MODELS.add(self)
        return p

    def add_lookup_parameters(self, rows: int, dim: int, name: str | None = None) -> LookupParameter:
        if rows < 1 or dim < 1:
            raise BadShape(f"lookup table needs rows ≥ 1 and dim ≥ 1, got {rows}×{dim}")
        name = self._claim_name(name, "lp")
        self._charge(rows * dim)
        vals = np.zeros((rows, dim), dtype=np.float32)
        if not self.init_zero:
            vals[:] = self.rng.uniform(-0.1, 0.1, (rows, dim))
        lp = LookupParameter(name, rows, dim, vals, self)
        self.lookups.append(lp)
        _PENDING_MODELS.add(self)
        return lp

    # -- device layout -----------------------------------------------------

    def _all(self):
        return list(self.parameters) + list(self.lookups)

    def _materialize(self) -> None:
        """(Re)lay out device storage: dense values/grads in two flat buffers
        (64-byte aligned slices), one buffer pair per lookup table."""
        lib = _native.lib()
        t = _dev.require_cuda()
        for x in self._all():  # keep device-side state when re-laying out
            x._vm.pull()
            x._gm.pull()
        total = 0
        for p in self.parameters:
            p._off = total
            total += (p.size + 15) & ~15
        self._dense_vals = _dev.zeros_f32(total)
        self._dense_grads = _dev.zeros_f32(total)
        for p in self.parameters:
            p._vm.dev = self._dense_vals[p._off : p._off + p.size]
            p._gm.dev = self._dense_grads[p._off : p._off + p.size]
        for lp in self.lookups:
            lp._vm.dev = _dev.zeros_f32(lp.rows * lp.dim)
            lp._gm.dev = _dev.zeros_f32(lp.rows * lp.dim)
        for x in self._all():
            rows, cols = (x.rows, x.dim) if isinstance(x, LookupParameter) else (x.size, 1)
            kind = 1 if isinstance(x, LookupParameter) else 0
            if x.handle < 0:
                h = ctypes.c_int64(-1)
                _native.check(lib.dg_param_register(kind, rows, cols, _native.ptr(x._vm.dev), _native.ptr(x._gm.dev),
                                                    ctypes.byref(h)))
                x.handle = h.value
                if kind == 1 and x._touched_host:
                    ids = np.array(sorted(x._touched_host), dtype=np.int64)
                    _native.check(lib.dg_touched_add(x.handle, ids.ctypes.data, ids.size))
                    x._touched_host = set()
            else:
                _native.check(lib.dg_param_rebind(x.handle, _native.ptr(x._vm.dev), _native.ptr(x._gm.dev)))
            x._vm._upload()
            x._gm._upload()
            _dev.DIRTY.discard(x._vm)
            _dev.DIRTY.discard(x._gm)
        self._materialized = len(self._all())
        del t

    def dense_gradient_buffer(self):
        """Flat device tensor holding every dense gradient (for all-reduce)."""
        materialize_pending()
        return self._dense_grads

    # -- gradients ---------------------------------------------------------

    def zero_gradients(self) -> None:
        """params.py:114-119: zero every gradient and clear touched sets."""
        if self._dense_grads is not None:
            materialize_pending()
            self._dense_grads.zero_()
            for lp in self.lookups:
                lp._gm.dev.zero_()
                _native.check(_native.lib().dg_touched_clear(lp.handle))
            _dev.bump_epoch()
        else:
            for x in self._all():
                x._gm.host[...] = 0
            for lp in self.lookups:
                lp._touched_host = set()

    # -- persistence (DYN1, params.py:128-189) -------------------------------

    def _roster(self):
        roster = {p.name: (0, p.shape.dims) for p in self.parameters}
        roster.update({lp.name: (1, (lp.rows, lp.dim)) for lp in self.lookups})
        return roster

    def _entries(self):
        """(kind, name, dims, flat host values) in roster order."""
        for p in self.parameters:
            yield 0, p.name, tuple(p.shape.dims), p._vm.pull().reshape(-1)
        for lp in self.lookups:
            yield 1, lp.name, (lp.rows, lp.dim), lp._vm.pull().reshape(-1)

    def save(self, path: str) -> None:
        """DYN1 (params.py:128-143): magic, <u32 version, u32 count>, then per
        entry <u8 kind, u16 name length> name <u8 rank> <u32 dims...> and the
        little-endian f32 values.  Values are read back from the device."""
        entries = list(self._entries())
        blob = bytearray(MAGIC) + struct.pack("<II", FORMAT_VERSION, len(entries))
        for kind, name, dims, flat in entries:
            raw = name.encode("utf-8")
            blob += struct.pack(f"<BH{len(raw)}sB{len(dims)}I", kind, len(raw), raw, len(dims), *dims)
            blob += np.asarray(flat, dtype="<f4").tobytes()
        try:
            with open(path, "wb") as fh:
                fh.write(blob)
        except OSError as exc:
            raise FileError(f"cannot write {path}: {exc}") from exc

    def load(self, path: str) -> None:
        """params.py:145-189: the file's roster (names, kinds, shapes) must equal
        this model's; values land in the host mirrors and reach the device
        before the next device use."""
        try:
            with open(path, "rb") as fh:
                blob = fh.read()
        except OSError as exc:
            raise FileError(f"cannot read {path}: {exc}") from exc
        seen = dict(_dyn1_records(blob, path))
        got = {name: (kind, dims) for name, (kind, dims, _) in seen.items()}
        roster = self._roster()
        if roster != got:
            missing = sorted(set(roster) ^ set(got))
            raise RosterMismatch(
                f"{path}: parameter roster differs from this model"
                + (f" (by {missing})" if missing else " (kind or shape changed)")
            )
        for x in self._all():
            x._vm.host_view().reshape(-1)[:] = seen[x.name][2]


def _dyn1_records(blob: bytes, path: str):
    """Yield (name, (kind, dims, values)) for every entry of a DYN1 blob."""
    if blob[:4] != MAGIC:
        raise FormatError(f"{path}: bad magic {blob[:4]!r}")
    try:
        version, count = struct.unpack_from("<II", blob, 4)
        if version != FORMAT_VERSION:
            raise FormatError(f"{path}: unsupported format version {version}")
        at = 12
        for _ in range(count):
            kind, nlen = struct.unpack_from("<BH", blob, at)
            name = blob[at + 3 : at + 3 + nlen].decode("utf-8")
            at += 3 + nlen
            rank = blob[at]
            dims = struct.unpack_from(f"<{rank}I", blob, at + 1)
            at += 1 + 4 * rank
            size = int(np.prod(dims))
            values = np.frombuffer(blob, dtype="<f4", count=size, offset=at)
            at += 4 * size
            yield name, (kind, tuple(dims), values)
    except (struct.error, IndexError, ValueError) as exc:
        raise FormatError(f"{path}: truncated or corrupt file") from exc
