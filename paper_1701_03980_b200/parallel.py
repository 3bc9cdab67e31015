"""Synchronous data parallelism over minibatches, one process per GPU.

Replaces the reference's in-process Hogwild worker pool
(pkg/src/dyncore/parallel.py:132-242) with NCCL ranks while keeping its
averaging semantics: the gradient applied by the single update per round is
the arithmetic mean over the participating contexts (average_slots,
parallel.py:55-65, loaded into the model by _load_average_into_model,
:105-109).

  * dense gradients: every dense parameter's gradient lives in ONE flat device
    buffer per Model (params.py), so the exchange is a single all-reduce;
  * lookup tables (sparse updates on): each rank packs its sorted touched rows
    (ids, rows), counts are all-gathered, ids/rows all-gathered padded to the
    max count, and every rank merges them with the same deterministic sorted
    segmented sum scaled by 1/R (dg_lookup_merge), so replicas stay
    bit-identical; touched := union of the ranks' touched sets.  (The
    reference forbids sparse + workers, parallel.py:118-119; SURVEY 8(c).1
    defines the union semantics the oracle restates.)
  * lookup tables with sparse off: dense all-reduce of the table gradient.

The process group may be NCCL (GPU) or gloo (CPU tests of the host logic).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from . import device as _dev
from .errors import CallbackError, ConfigError


def _dist():
    import torch.distributed as dist

    return dist


def merge_plan(ids_per_rank):
    """Host logic of the sparse merge: concatenated ids in rank order and the
    sorted unique ids with segment offsets (the order dg_lookup_merge uses).
    Pure numpy; exercised by the gloo CPU tests."""
    ids = np.concatenate([np.asarray(x, dtype=np.int64) for x in ids_per_rank]) if ids_per_rank else np.zeros(0, np.int64)
    order = np.argsort(ids, kind="stable")
    uniq, starts = np.unique(ids[order], return_index=True)
    seg = np.append(starts, len(ids)).astype(np.int64)
    return ids, order, uniq, seg


def exchange_rows(dist, group, world: int, n_local: int, dim: int, pack, device):
    """Variable-length (ids, rows) all-gather without all-gatherv: counts
    first, then ids/rows padded to the max count.  `pack(ids, rows, cap)`
    fills this rank's sorted touched rows.  Returns (ids in rank order as a
    numpy array, the matching rows as one contiguous tensor)."""
    import torch as t

    cnt = t.tensor([n_local], dtype=t.int64, device=device)
    counts = [t.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(1, max(counts))
    ids = t.zeros(cap, dtype=t.int64, device=device)
    rows = t.zeros((cap, dim), dtype=t.float32, device=device)
    pack(ids, rows, cap)
    all_ids = [t.zeros(cap, dtype=t.int64, device=device) for _ in range(world)]
    all_rows = [t.zeros((cap, dim), dtype=t.float32, device=device) for _ in range(world)]
    dist.all_gather(all_ids, ids, group=group)
    dist.all_gather(all_rows, rows, group=group)
    flat_ids = t.cat([all_ids[r][: counts[r]] for r in range(world)]).cpu().numpy().astype(np.int64)
    flat_rows = t.cat([all_rows[r][: counts[r]] for r in range(world)]).contiguous()
    return flat_ids, flat_rows


class DataParallel:
    """Gradient exchange for one Model across the default process group."""

    def __init__(self, model, sparse: bool = True, group=None):
        self.model = model
        self.sparse = sparse
        self.group = group
        dist = _dist()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self._pack = {}

    def _buffers(self, lp, cap):
        t = _dev.torch()
        buf = self._pack.get(lp.handle)
        if buf is None or buf[0].shape[0] < cap:
            ids = t.zeros(cap, dtype=t.int64, device=_dev.device())
            rows = t.zeros((cap, lp.dim), dtype=t.float32, device=_dev.device())
            buf = (ids, rows)
            self._pack[lp.handle] = buf
        return buf

    def sync(self) -> None:
        """Average gradients over ranks (call after backward, before update)."""
        if self.world == 1:
            return
        dist = _dist()
        t = _dev.torch()
        R = self.world
        dense = self.model.dense_gradient_buffer()
        if dense is not None and dense.numel():
            dist.all_reduce(dense, group=self.group)
            dense.mul_(1.0 / R)
        lib = _native.lib()
        stream = _dev.stream_ptr()
        for lp in self.model.lookups:
            if not self.sparse:
                g = lp._gm.dev
                dist.all_reduce(g, group=self.group)
                g.mul_(1.0 / R)
                continue
            n = ctypes.c_int64(0)
            _native.check(lib.dg_touched_count(lp.handle, ctypes.byref(n)))

            def pack(ids, rows, cap, lp=lp):
                got = ctypes.c_int64(0)
                _native.check(lib.dg_lookup_pack(lp.handle, _native.ptr(ids), _native.ptr(rows), cap,
                                                 ctypes.byref(got), stream))

            flat_ids, flat_rows = exchange_rows(dist, self.group, R, n.value, lp.dim, pack, _dev.device())
            if flat_ids.size:
                _native.check(lib.dg_lookup_merge(lp.handle, flat_ids.ctypes.data, _native.ptr(flat_rows),
                                                  flat_ids.size, 1.0 / R, stream))
        _dev.bump_epoch()


def train_parallel(plan, model, trainer, data: list, epochs: int) -> list[float]:
    """Reference-compatible entry (parallel.py:112-129) on NCCL ranks: rank r
    takes data[r], data[r+R], ...; each round averages the participating
    ranks' gradients and applies one update on every rank (replicas stay in
    lockstep).  Returns the aggregate loss per epoch (summed over ranks)."""
    dist = _dist()
    R = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if plan.workers < 1:
        raise ConfigError(f"workers must be >= 1, got {plan.workers}")
    cg = plan._parent(model)
    dp = DataParallel(model, sparse=trainer.sparse)
    t = _dev.torch()
    out = []
    for _ in range(epochs):
        total = 0.0
        rounds = (len(data) + R - 1) // R
        for k in range(rounds):
            idx = k * R + rank
            part = 1.0 if idx < len(data) else 0.0
            if part:
                try:
                    cg.renew()
                    loss = plan.loss_fn(cg, model, data[idx])
                    cg.backward(loss)
                    total += float(cg.value(loss).data[0])
                except Exception as exc:
                    raise CallbackError(idx, exc) from exc
            if R > 1:
                # the divisor is the number of participants (parallel.py:60-64)
                n_part = t.tensor([part], dtype=t.float32, device=_dev.device())
                dist.all_reduce(n_part)
                parts = float(n_part.item())
                dp.world = R
                dp.sync()
                if parts != R:
                    scale = R / parts
                    model.dense_gradient_buffer().mul_(scale)
                    for lp in model.lookups:
                        lp._gm.dev.mul_(scale)
            trainer.update()
        if R > 1:
            tot = t.tensor([total], dtype=t.float64, device=_dev.device())
            dist.all_reduce(tot)
            total = float(tot.item())
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
