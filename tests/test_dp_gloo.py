"""CPU tests of the data-parallel exchange: the product `DataParallel.sync`
(paper_1701_03980_b200/parallel.py) runs unchanged over

  * a world-size-2 gloo process group (`ProcessGroupComm`, mp.spawn), and
  * in-process replicas (`ThreadComm`, 3 threads: a non-power-of-two R),

with an oracle-backed gradient store standing in for HBM (the device store is
covered by tests/test_gpu_dp.py on the GPU).  Results must reproduce the
oracle's deterministic DP restatement (oracle.engine.dp_step: average over
the R participants, touched = union; reference parallel.py:55-65,105-109),
with bit-identical replicas.
"""

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import engine as orc
from paper_1701_03980_b200 import workloads as W
from paper_1701_03980_b200.parallel import DataParallel, ProcessGroupComm, ThreadComm, merge_plan

VOCAB, E, H = 120, 8, 12


class OracleGradStore:
    """DataParallel's store interface over an oracle Model (numpy arrays)."""

    def __init__(self, model):
        self.m = model
        self._dense = None

    def begin(self):
        self._dense = torch.from_numpy(np.concatenate([p.gradient.ravel() for p in self.m.parameters]))

    def end(self):
        off = 0
        for p in self.m.parameters:
            n = p.gradient.size
            p.gradient.ravel()[:] = self._dense[off : off + n].numpy()
            off += n

    def dense(self):
        return self._dense

    def lookups(self):
        return list(self.m.lookups)

    def table_grad(self, lp):
        return torch.from_numpy(lp.gradient)

    def touched(self, lp):
        return np.array(sorted(lp.touched), dtype=np.int64)

    def alloc(self, n):
        return torch.zeros(max(1, int(n)), dtype=torch.float32)

    def pack(self, lp, ids, out):
        out.view(-1, lp.dim)[:] = torch.from_numpy(lp.gradient[ids])

    def merge(self, lp, counts, ids, rank_rows, divisor):
        """What dg_lookup_merge computes: rows of the union = (sum in rank
        order) / divisor; the union joins the touched set."""
        rows = np.concatenate([rank_rows[r].numpy().reshape(-1, lp.dim)[: counts[r]] for r in range(len(counts))])
        _, order, uniq, seg = merge_plan([ids])
        for u, rid in enumerate(uniq):
            acc = np.zeros(lp.dim, dtype=np.float32)
            for k in range(seg[u], seg[u + 1]):
                acc += rows[order[k]]
            lp.gradient[rid] = acc / np.float32(divisor)
        lp.touched = set(lp.touched) | set(int(i) for i in uniq)


def _shards(n):
    sents = W.ptb_corpus(31, 4 * n, vocab=VOCAB)
    return W.minibatches(sents, 4)  # rank r takes batch r


def _make(seed=1):
    pools = orc.new_poolset()
    cg, m = orc.ComputationGraph(pools), orc.Model(pools, seed=seed)
    return cg, m, W.RNNLM(orc, m, VOCAB, E, H, 2)


def _replica_step(rank, R, comm, sparse, rule="adam"):
    cg, m, task = _make()
    tr = orc.Trainer(m, rule)
    tr.sparse = sparse
    cg.renew()
    loss = task.loss(cg, _shards(R)[rank])
    cg.backward(loss)
    DataParallel(m, sparse=sparse, comm=comm, store=OracleGradStore(m)).sync()
    tr.update()
    return {**{p.name: p.values.copy() for p in m.parameters}, **{lp.name: lp.values.copy() for lp in m.lookups}}


def _oracle(R, sparse, rule="adam"):
    _, m, task = _make()
    tr = orc.Trainer(m, rule)
    tr.sparse = sparse
    shards = _shards(R)

    def graph_for(r):
        g = orc.ComputationGraph(orc.new_poolset())
        return g, task.loss(g, shards[r])

    orc.dp_step(m, tr, graph_for, R)
    return {**{p.name: p.values for p in m.parameters}, **{lp.name: lp.values for lp in m.lookups}}


def _worker(rank, port, outdir, sparse):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    out = _replica_step(rank, 2, ProcessGroupComm(), sparse)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
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


@pytest.mark.parametrize("sparse", [True, False])
def test_sync_over_gloo_matches_oracle_dp(tmp_path, sparse):
    mp.spawn(_worker, args=(_free_port(), str(tmp_path), sparse), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    ref = _oracle(2, sparse)
    for k in r0.files:
        assert np.array_equal(r0[k], r1[k]), f"replicas diverged on {k}"
        # R=2: the gloo sum of two addends then /2 is the reference's sum/2
        np.testing.assert_array_equal(r0[k], ref[k], err_msg=k)


@pytest.mark.parametrize("sparse", [True, False])
def test_sync_over_threads_is_bit_exact(sparse):
    R = 3
    comms = ThreadComm.group(R)
    outs = [None] * R
    errs = []

    def run(r):
        try:
            outs[r] = _replica_step(r, R, comms[r], sparse)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            comms[r].shared.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    ref = _oracle(R, sparse)
    for k in ref:
        for r in range(R):
            # rank-order sums divided by R: exactly the reference's average_slots
            np.testing.assert_array_equal(outs[r][k], ref[k], err_msg=f"{k} rank {r}")


def test_sync_touched_is_union():
    R = 2
    comms = ThreadComm.group(R)
    touched = [None] * R

    def run(r):
        cg, m, task = _make()
        cg.renew()
        cg.backward(task.loss(cg, _shards(R)[r]))
        mine = set(m.lookups[0].touched)
        DataParallel(m, sparse=True, comm=comms[r], store=OracleGradStore(m)).sync()
        touched[r] = (mine, set(m.lookups[0].touched))

    th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    union = touched[0][0] | touched[1][0]
    assert touched[0][0] != touched[1][0]
    assert touched[0][1] == union and touched[1][1] == union
