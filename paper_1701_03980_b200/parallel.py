"""Synchronous data parallelism over minibatches.

Replaces the reference's in-process Hogwild worker pool
(pkg/src/dyncore/parallel.py:132-242) with synchronous replicas while keeping
its averaging semantics: the gradient applied by the single update per round
is the arithmetic mean over the participating contexts (average_slots,
parallel.py:55-65, loaded into the model by _load_average_into_model,
:105-109).

One `DataParallel.sync()` per step, after backward and before update:

  * dense gradients: every dense parameter's gradient lives in ONE flat device
    buffer per Model (params.py), so the exchange is a single all-reduce
    (NCCL ReduceOp.AVG on NVLink; sum then divide elsewhere);
  * lookup tables with sparse updates: the touched-row ids are host data, so
    they travel over the host channel (one gather of every table's ids, no
    device synchronisation); each rank packs its touched rows of every table
    into ONE flat device buffer (dg_lookup_pack), a single device all-gather
    moves the rows, and every rank merges them with the same deterministic
    sorted segmented sum divided by the participant count (dg_lookup_merge),
    so replicas stay bit-identical; touched := union of the ranks' sets.  The
    reference forbids sparse + workers (parallel.py:118-119); SURVEY 8(c).1
    defines the union semantics the oracle restates (oracle.engine.dp_step);
  * lookup tables with sparse off: all-reduce of the table gradient.

The exchange is written against two small interfaces so the same `sync` code
runs everywhere:

  * a Communicator: `ProcessGroupComm` (torch.distributed: NCCL device
    collectives plus a gloo group for the host ids; or gloo alone for CPU
    tests) or `ThreadComm` (R replicas as threads of one process, e.g. R
    model replicas on one GPU — the multi-replica GPU parity test);
  * a gradient store: `DeviceGradStore` (the product: Model storage in HBM
    through libdyngpu) or a test store over oracle models (tests/).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native
from . import device as _dev
from .errors import CallbackError, ConfigError


def _dist():
    import torch.distributed as dist

    return dist


def merge_plan(ids_per_rank):
    """Host logic of the sparse merge: concatenated ids in rank order and the
    sorted unique ids with segment offsets (the order dg_lookup_merge uses:
    a stable sort, so a segment lists its ranks' rows in rank order)."""
    ids = np.concatenate([np.asarray(x, dtype=np.int64) for x in ids_per_rank]) if ids_per_rank else np.zeros(0, np.int64)
    order = np.argsort(ids, kind="stable")
    uniq, starts = np.unique(ids[order], return_index=True)
    seg = np.append(starts, len(ids)).astype(np.int64)
    return ids, order, uniq, seg


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------


class Communicator:
    """What DataParallel.sync needs from a group of R replicas."""

    world = 1
    rank = 0

    def all_reduce_mean(self, t, divisor: float | None = None) -> None:
        """In place: t = (sum over ranks of t) / divisor (default R)."""
        raise NotImplementedError

    def all_gather(self, t):
        """Equal-shaped tensors of every rank stacked as [R, *t.shape]."""
        raise NotImplementedError

    def all_gather_host(self, a: np.ndarray) -> list:
        """Variable-length int64 host arrays of every rank, in rank order."""
        raise NotImplementedError


class ProcessGroupComm(Communicator):
    """torch.distributed, one process per rank.  Device collectives run on the
    group's backend (NCCL over NVLink on the GPU box); the host ids go over
    a gloo group (the group itself when it is gloo), so no device tensor has
    to be read back to size the row exchange."""

    def __init__(self, group=None):
        dist = _dist()
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = str(dist.get_backend(group)).lower()
        if self.backend == "gloo":
            self.host_group = group
        else:  # collective: every rank constructs its DataParallel in the same order
            ranks = None if group is None else dist.get_process_group_ranks(group)
            self.host_group = dist.new_group(ranks=ranks, backend="gloo")

    def all_reduce_mean(self, t, divisor=None):
        dist = self.dist
        if self.backend == "nccl" and (divisor is None or divisor == self.world):
            dist.all_reduce(t, op=dist.ReduceOp.AVG, group=self.group)
            return
        dist.all_reduce(t, group=self.group)
        t.div_(float(divisor if divisor is not None else self.world))

    def all_gather(self, t):
        dist = self.dist
        out = t.new_empty((self.world,) + tuple(t.shape))
        if self.backend == "nccl":
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        else:
            dist.all_gather(list(out.unbind(0)), t.contiguous(), group=self.group)
        return out

    def all_gather_host(self, a):
        import torch

        dist = self.dist
        a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64))
        n = torch.tensor([a.numel()], dtype=torch.int64)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(counts, n, group=self.host_group)
        counts = [int(c[0]) for c in counts]
        cap = max(1, max(counts))
        pad = torch.zeros(cap, dtype=torch.int64)
        pad[: a.numel()] = a
        outs = [torch.zeros(cap, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.host_group)
        return [outs[r][: counts[r]].numpy() for r in range(self.world)]


class _ThreadShared:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.result = None


class ThreadComm(Communicator):
    """R replicas as threads of one process (one CUDA stream: every device op
    is enqueued in barrier order, so stream order is the collective order).
    Reductions run in rank order, exactly the reference's
    `sum(slots) / n` (parallel.py:60-64)."""

    def __init__(self, shared: _ThreadShared, rank: int):
        self.shared = shared
        self.world = shared.world
        self.rank = rank

    @classmethod
    def group(cls, world: int) -> list:
        sh = _ThreadShared(world)
        return [cls(sh, r) for r in range(world)]

    def _exchange(self, obj):
        sh = self.shared
        sh.slots[self.rank] = obj
        sh.barrier.wait()
        got = list(sh.slots)
        sh.barrier.wait()
        return got

    def all_reduce_mean(self, t, divisor=None):
        parts = self._exchange(t)
        if self.rank == 0:
            acc = parts[0].clone()
            for x in parts[1:]:
                acc += x
            acc /= float(divisor if divisor is not None else self.world)
            self.shared.result = acc
        self.shared.barrier.wait()
        t.copy_(self.shared.result)
        self.shared.barrier.wait()

    def all_gather(self, t):
        import torch

        return torch.stack([x.contiguous() for x in self._exchange(t)])

    def all_gather_host(self, a):
        return [np.asarray(x, dtype=np.int64).copy() for x in self._exchange(np.asarray(a, dtype=np.int64))]


def default_comm(group=None) -> Communicator:
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return Communicator()
    return ProcessGroupComm(group)


# ---------------------------------------------------------------------------
# gradient stores
# ---------------------------------------------------------------------------


class DeviceGradStore:
    """The product store: a Model's gradients in HBM, touched sets in
    libdyngpu.  All calls are asynchronous on the current stream."""

    def __init__(self, model):
        self.model = model
        self._ids = {}

    def begin(self):
        _dev.flush_dirty()  # host-written gradients reach the device first

    def end(self):
        _dev.bump_epoch()  # host mirrors of gradients are stale now

    def dense(self):
        return self.model.dense_gradient_buffer()

    def lookups(self):
        return list(self.model.lookups)

    def table_grad(self, lp):
        return lp._gm.dev

    def touched(self, lp) -> np.ndarray:
        lib = _native.lib()
        n = ctypes.c_int64(0)
        _native.check(lib.dg_touched_count(lp.handle, ctypes.byref(n)))
        out = np.zeros(max(1, n.value), dtype=np.int64)
        if n.value:
            _native.check(lib.dg_touched_get(lp.handle, out.ctypes.data, n.value))
        return out[: n.value]

    def alloc(self, n_floats: int):
        t = _dev.torch()
        return t.zeros(max(1, int(n_floats)), dtype=t.float32, device=_dev.device())

    def pack(self, lp, ids: np.ndarray, out) -> None:
        t = _dev.torch()
        buf = self._ids.get(lp.handle)
        if buf is None or buf.numel() < len(ids):
            buf = t.zeros(max(64, 2 * len(ids)), dtype=t.int64, device=_dev.device())
            self._ids[lp.handle] = buf
        got = ctypes.c_int64(0)
        _native.check(_native.lib().dg_lookup_pack(lp.handle, _native.ptr(buf), _native.ptr(out), len(ids),
                                                   ctypes.byref(got), _dev.stream_ptr()))
        if got.value != len(ids):
            raise ConfigError("touched set changed during the exchange")

    def merge(self, lp, counts, ids: np.ndarray, rank_rows: list, divisor: float) -> None:
        R = len(counts)
        c_counts = np.ascontiguousarray(counts, dtype=np.int64)
        c_ids = np.ascontiguousarray(ids, dtype=np.int64)
        ptrs = (ctypes.c_void_p * R)(*[_native.ptr(x) for x in rank_rows])
        _native.check(_native.lib().dg_lookup_merge(lp.handle, R, c_counts.ctypes.data, c_ids.ctypes.data, ptrs,
                                                    float(divisor), _dev.stream_ptr()))


# ---------------------------------------------------------------------------
# the exchange
# ---------------------------------------------------------------------------


class DataParallel:
    """Gradient exchange for one Model across R replicas."""

    def __init__(self, model, sparse: bool = True, group=None, comm: Communicator | None = None, store=None):
        self.model = model
        self.sparse = sparse
        self.comm = comm if comm is not None else default_comm(group)
        self.store = store if store is not None else DeviceGradStore(model)

    @property
    def world(self) -> int:
        return self.comm.world

    def sync(self, participants: int | None = None) -> None:
        """Average gradients over the participating replicas (call after
        backward, before update).  `participants` (default R) is the
        average_slots divisor; a non-participating replica contributes zero
        gradients and an empty touched set."""
        comm, st = self.comm, self.store
        R = comm.world
        if R == 1:
            return
        div = float(participants if participants is not None else R)
        st.begin()
        dense = st.dense()
        if dense is not None and dense.numel():
            comm.all_reduce_mean(dense, div)
        lps = st.lookups()
        if not self.sparse:
            for lp in lps:
                comm.all_reduce_mean(st.table_grad(lp), div)
            st.end()
            return
        if not lps:
            st.end()
            return
        mine = [st.touched(lp) for lp in lps]
        # one host exchange of every table's ids: [n_0, .., n_{T-1}, ids_0.., ids_1.., ...]
        head = np.array([len(m) for m in mine], dtype=np.int64)
        got = comm.all_gather_host(np.concatenate([head] + mine))
        T = len(lps)
        counts = np.zeros((R, T), dtype=np.int64)
        ids = [[None] * T for _ in range(R)]
        for r, a in enumerate(got):
            counts[r] = a[:T]
            off = T
            for t in range(T):
                ids[r][t] = a[off : off + counts[r, t]]
                off += counts[r, t]
        caps = counts.max(axis=0)
        dims = [lp.dim for lp in lps]
        offs = np.concatenate([[0], np.cumsum(caps * np.array(dims, dtype=np.int64))])
        if offs[-1] == 0:
            st.end()
            return
        buf = st.alloc(int(offs[-1]))
        for t, lp in enumerate(lps):
            if len(mine[t]):
                st.pack(lp, mine[t], buf[offs[t] : offs[t] + len(mine[t]) * dims[t]])
        gathered = comm.all_gather(buf)  # [R, total]
        for t, lp in enumerate(lps):
            if counts[:, t].sum() == 0:
                continue
            flat_ids = np.concatenate([ids[r][t] for r in range(R)])
            rows = [gathered[r, offs[t] : offs[t + 1]] for r in range(R)]
            st.merge(lp, counts[:, t], flat_ids, rows, div)
        st.end()


def train_parallel(plan, model, trainer, data: list, epochs: int, comm: Communicator | None = None) -> list[float]:
    """Reference-compatible entry (parallel.py:112-129) over R replicas: rank
    r takes data[r], data[r+R], ...; each round averages the participating
    ranks' gradients (the average_slots divisor counts participants only,
    parallel.py:55-65) and applies one update on every rank, so replicas stay
    in lockstep.  Returns the aggregate loss per epoch (summed over ranks)."""
    if plan.workers < 1:
        raise ConfigError(f"workers must be >= 1, got {plan.workers}")
    dp = DataParallel(model, sparse=trainer.sparse, comm=comm)
    R, rank = dp.comm.world, dp.comm.rank
    cg = plan._parent(model)
    out = []
    for _ in range(epochs):
        total = 0.0
        rounds = (len(data) + R - 1) // R
        for k in range(rounds):
            idx = k * R + rank
            parts = min(R, len(data) - k * R)
            if idx < len(data):
                try:
                    cg.renew()
                    loss = plan.loss_fn(cg, model, data[idx])
                    cg.backward(loss)
                    total += float(cg.value(loss).data[0])
                except Exception as exc:
                    raise CallbackError(idx, exc) from exc
            dp.sync(participants=parts)
            trainer.update()
        if R > 1:
            totals = dp.comm.all_gather_host(np.array([total], dtype=np.float64).view(np.int64))
            total = float(sum(np.asarray(x).view(np.float64)[0] for x in totals))
        out.append(total)
    return out


class ParallelPlan:
    """Worker count plus the per-datum loss builder (parallel.py:68-102)."""

    def __init__(self, workers: int, loss_fn, parent_cg=None, forward_mb: float = 256.0, backward_mb: float = 256.0):
        self.workers = workers
        self.loss_fn = loss_fn
        self.parent_cg = parent_cg
        self.forward_mb = forward_mb
        self.backward_mb = backward_mb

    def _parent(self, model):
        if self.parent_cg is None:
            from .arena import new_poolset
            from .graph import ComputationGraph

            self.parent_cg = ComputationGraph(new_poolset(self.forward_mb, self.backward_mb, 1))
        return self.parent_cg
