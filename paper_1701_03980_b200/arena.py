"""Memory pools of the drop-in API (pkg/src/dyncore/arena.py:14-110) backed by
device arenas.

The forward and backward pools are device bump arenas owned by the native
graph executor: it charges exactly the reference's 64-byte-rounded sizes per
node, so `alloc_count`, `cursor`, `remaining` and PoolExhausted behave as in
the reference (arena.py:48-56), while the physical placement inside the arena
is chosen by the batching planner.  The parameters pool keeps the reference
accounting on the host; parameter storage itself is laid out per Model on the
device (params.py).  Device memory is allocated on first execution, so graphs
can be constructed (and construction errors raised) without a GPU.
"""

from __future__ import annotations

import numpy as np

from . import device as _dev
from .errors import AllocationFailed, ConfigError, PoolExhausted

ALIGNMENT = 64
MIB = 1 << 20


class Pool:
    """Accounting view of one pool."""

    __slots__ = ("name", "capacity", "_cursor", "_alloc_count", "_owner")

    def __init__(self, name: str, capacity: int):
        if capacity <= 0:
            raise AllocationFailed(f"pool '{name}' requires positive capacity, got {capacity}")
        self.name = name
        self.capacity = int(capacity)
        self._cursor = 0
        self._alloc_count = 0
        self._owner = None  # native graph (forward/backward pools)

    def _counters(self):
        if self._owner is not None:
            c = self._owner._counters()
            return (c[3], c[1]) if self.name == "forward" else (c[4], c[2])
        return self._cursor, self._alloc_count

    @property
    def cursor(self) -> int:
        return int(self._counters()[0])

    @property
    def alloc_count(self) -> int:
        return int(self._counters()[1])

    @property
    def remaining(self) -> int:
        return self.capacity - self.cursor

    def allocate(self, nbytes: int) -> tuple[int, int]:
        """Host-side bump (parameters pool; arena.py:48-56 rounding rule)."""
        if self._owner is not None:
            raise ConfigError(f"pool '{self.name}' is managed by the device executor")
        rounded = (nbytes + ALIGNMENT - 1) & ~(ALIGNMENT - 1)
        offset = self._cursor
        if rounded > self.capacity - offset:
            raise PoolExhausted(self.name, nbytes, self.capacity - offset)
        self._cursor = offset + rounded
        self._alloc_count += 1
        return offset, nbytes

    def reset(self, zero_used: bool = False) -> None:
        if self._owner is None:
            self._cursor = 0


class PoolSet:
    """forward/backward/parameters pools plus the element type (float32 only)."""

    __slots__ = ("forward", "backward", "parameters", "dtype", "work_bytes", "_buffers", "_bound")

    def __init__(self, forward_mb: float, backward_mb: float, param_mb: float, dtype=np.float32,
                 work_mb: float | None = None):
        for label, mb in (("forward", forward_mb), ("backward", backward_mb), ("parameters", param_mb)):
            if mb <= 0:
                raise AllocationFailed(f"pool '{label}' size must be > 0 MiB, got {mb}")
        if np.dtype(dtype) != np.float32:
            raise ConfigError("the B200 executor computes in float32; PoolSet dtype must be float32")
        self.forward = Pool("forward", int(forward_mb * MIB))
        self.backward = Pool("backward", int(backward_mb * MIB))
        self.parameters = Pool("parameters", int(param_mb * MIB))
        self.dtype = np.dtype(np.float32)
        # plan tables + split-K / reduction scratch (half each)
        self.work_bytes = int((work_mb if work_mb is not None else 256) * MIB)
        self._buffers = None
        self._bound = None

    def device_buffers(self):
        """Allocate (once) the device arenas through PyTorch."""
        if self._buffers is None:
            self._buffers = (
                _dev.empty_bytes(self.forward.capacity),
                _dev.empty_bytes(self.backward.capacity),
                _dev.empty_bytes(self.work_bytes),
            )
        return self._buffers

    def bind(self, graph) -> None:
        if self._bound is not None and self._bound is not graph:
            raise ConfigError("a PoolSet backs exactly one ComputationGraph")
        self._bound = graph
        self.forward._owner = graph
        self.backward._owner = graph

    def reset_transient(self) -> None:
        if self._bound is not None:
            self._bound._native_renew()


def new_poolset(forward_mb: float, backward_mb: float, param_mb: float, dtype=np.float32) -> PoolSet:
    return PoolSet(forward_mb, backward_mb, param_mb, dtype=dtype)


def poolset_from_mem_flag(flag: str, dtype=np.float32) -> PoolSet:
    """`--mem` value: total MiB (split in thirds) or `fwd,bwd,param` (arena.py:99-110)."""
    try:
        sizes = [float(p) for p in str(flag).split(",")]
    except ValueError as exc:
        raise AllocationFailed(f"bad --mem value {flag!r}") from exc
    if len(sizes) == 1:
        sizes = [sizes[0] / 3.0] * 3
    if len(sizes) != 3:
        raise AllocationFailed(f"--mem takes one total or three sizes, got {flag!r}")
    return PoolSet(*sizes, dtype=dtype)
