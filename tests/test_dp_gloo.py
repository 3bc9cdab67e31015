"""World-size-2 (gloo, CPU) test of the data-parallel exchange protocol.

The GPU path (parallel.DataParallel) all-reduces the flat dense gradient and
exchanges sparse lookup rows with `exchange_rows` (counts all-gather, padded
ids/rows all-gather, rank-order concatenation) before a deterministic sorted
segmented merge.  Here the same protocol runs over gloo on CPU tensors with
oracle-computed per-rank gradients and a numpy merge, and must reproduce the
oracle's deterministic DP restatement (oracle.engine.dp_step: average over R
participants, touched = union), with bit-identical replicas on both ranks.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import engine as orc
from paper_1701_03980_b200 import workloads as W
from paper_1701_03980_b200.parallel import exchange_rows, merge_plan

R = 2
VOCAB, E, H = 120, 8, 12


def _shards():
    sents = W.ptb_corpus(31, 8, vocab=VOCAB)
    return W.minibatches(sents, 4)  # rank r takes batch r


def _make(seed=1):
    pools = orc.new_poolset()
    cg, m = orc.ComputationGraph(pools), orc.Model(pools, seed=seed)
    return cg, m, W.RNNLM(orc, m, VOCAB, E, H, 2)


def _numpy_merge(grad, ids, rows, scale):
    """The merge dg_lookup_merge performs, restated for the CPU check."""
    _, order, uniq, seg = merge_plan([ids])
    grad[uniq] = 0
    for u, rid in enumerate(uniq):
        acc = np.zeros(grad.shape[1], dtype=np.float32)
        for k in range(seg[u], seg[u + 1]):
            acc += rows[order[k]]
        grad[rid] += np.float32(scale) * acc


def _worker(rank, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=R)
    cg, m, task = _make()
    tr = orc.Trainer(m, "adam")
    batch = _shards()[rank]
    cg.renew()
    loss = task.loss(cg, batch)
    cg.backward(loss)
    # dense: one flat all-reduce (average over R participants)
    flat = torch.from_numpy(np.concatenate([p.gradient for p in m.parameters]))
    dist.all_reduce(flat)
    flat /= R
    off = 0
    for p in m.parameters:
        p.gradient[:] = flat[off : off + p.gradient.size].numpy()
        off += p.gradient.size
    # sparse rows
    for lp in m.lookups:
        mine = np.array(sorted(lp.touched), dtype=np.int64)

        def pack(ids, rows, cap, mine=mine, lp=lp):
            ids[: len(mine)] = torch.from_numpy(mine)
            rows[: len(mine)] = torch.from_numpy(lp.gradient[mine])

        ids, rows = exchange_rows(dist, None, R, len(mine), lp.dim, pack, torch.device("cpu"))
        _numpy_merge(lp.gradient, ids, rows.numpy(), 1.0 / R)
        lp.touched = set(int(i) for i in ids)
    tr.update()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             **{p.name: p.values for p in m.parameters}, **{lp.name: lp.values for lp in m.lookups})
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_merge_plan_is_sorted_stable():
    ids, order, uniq, seg = merge_plan([[5, 1, 5], [1, 9]])
    assert list(uniq) == [1, 5, 9]
    assert list(seg) == [0, 2, 4, 5]
    # rank order preserved inside a segment (stable): id 1 from rank 0 first
    assert list(order[:2]) == [1, 3]


def test_dp_exchange_matches_oracle_restatement(tmp_path):
    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=R, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    for k in r0.files:
        assert np.array_equal(r0[k], r1[k]), f"replicas diverged on {k}"
    # serial oracle DP restatement on the same shards
    cgs = [_make() for _ in range(R)]
    _, m, task = _make()
    tr = orc.Trainer(m, "adam")
    shards = _shards()

    def graph_for(r):
        g = orc.ComputationGraph(orc.new_poolset())
        return g, task.loss(g, shards[r])

    orc.dp_step(m, tr, graph_for, R)
    for p in m.parameters:
        np.testing.assert_allclose(r0[p.name], p.values, rtol=1e-5, atol=1e-7)
    for lp in m.lookups:
        np.testing.assert_allclose(r0[lp.name], lp.values, rtol=1e-5, atol=1e-7)
    del cgs
