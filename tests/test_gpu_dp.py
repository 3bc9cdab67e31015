"""Data parallelism on the device (reference parallel.py:55-65,
105-109): R model replicas in one process on one GPU, one thread each, the
product `DataParallel.sync` (DeviceGradStore: dg_lookup_pack /
dg_lookup_merge, the flat dense buffer) over `ThreadComm`, against the
oracle's deterministic DP restatement (oracle.engine.dp_step).

Bar: touched sets equal the union bit-exactly at every step, replicas stay
bit-identical, parameters match the oracle within rtol 1e-4 after 3 SGD steps.
"""

import threading

import numpy as np
import pytest

from oracle import engine as orc
from paper_1701_03980_b200 import workloads as W
from paper_1701_03980_b200.parallel import DataParallel, ParallelPlan, ThreadComm, train_parallel
from tests.helpers import parity, pvals

pytestmark = pytest.mark.gpu

VOCAB, E, H, L, MB = 2000, 32, 64, 2, 8


def _run_threads(R, fn):
    comms = ThreadComm.group(R)
    outs, errs = [None] * R, []

    def run(r):
        try:
            outs[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs.append(e)
            comms[r].shared.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return outs


def _batches(R, steps):
    sents = W.ptb_corpus(5, MB * R * steps, vocab=VOCAB)
    return W.minibatches(sents, MB)


@pytest.mark.parametrize("R,sparse,rule", [(2, True, "sgd"), (3, True, "sgd"), (2, False, "sgd"), (2, True, "adam")])
def test_replicas_match_oracle_dp(R, sparse, rule):
    import paper_1701_03980_b200 as dy
    from paper_1701_03980_b200.params import materialize_pending

    steps = 3
    batches = _batches(R, steps)
    reps = []
    for _ in range(R):
        pools = dy.new_poolset(128, 128, 64)
        cg, m = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
        task = W.RNNLM(dy, m, VOCAB, E, H, L)
        tr = dy.Trainer(m, rule, sparse=sparse)
        reps.append((cg, m, task, tr))
    materialize_pending()  # register every replica's storage before the threads start

    def replica(r, comm):
        cg, m, task, tr = reps[r]
        dp = DataParallel(m, sparse=sparse, comm=comm)
        touched, losses = [], []
        for s in range(steps):
            cg.renew()
            loss = task.loss(cg, batches[s * R + r])
            cg.backward(loss)
            losses.append(float(cg.value(loss).data[0]))
            dp.sync()
            touched.append(sorted(m.lookups[0].touched))
            tr.update()
        return touched, losses

    outs = _run_threads(R, replica)

    # oracle restatement on the same shards
    pools = orc.new_poolset()
    om = orc.Model(pools, seed=1)
    otask = W.RNNLM(orc, om, VOCAB, E, H, L)
    otr = orc.Trainer(om, rule, sparse=sparse)
    for s in range(steps):
        def graph_for(r, s=s):
            g = orc.ComputationGraph(orc.new_poolset())
            return g, otask.loss(g, batches[s * R + r])

        # the union the oracle uses, recomputed to compare with the device's
        union = set()
        for r in range(R):
            g, loss = graph_for(r)
            for i in range(loss.i + 1):
                if g.kinds[i] == "lookup_batch":
                    union.update(int(x) for x in g.auxs[i][1])
        olosses = orc.dp_step(om, otr, graph_for, R)
        for r in range(R):
            if sparse:
                assert outs[r][0][s] == sorted(union), f"step {s} rank {r}: touched != union"
            parity(outs[r][1][s], olosses[r], what=f"loss step {s} rank {r}")
    band = 2 * otr.lr * steps if rule == "adam" else 0.0
    for name in [p.name for p in om.parameters] + [lp.name for lp in om.lookups]:
        vals = [pvals(next(x for x in reps[r][1]._all() if x.name == name)) for r in range(R)]
        for r in range(1, R):
            assert np.array_equal(vals[0], vals[r]), f"replica {r} diverged on {name}"
        ref = next(x for x in list(om.parameters) + list(om.lookups) if x.name == name)
        parity(vals[0], np.asarray(ref.values, dtype=np.float64).reshape(-1), band=band, what=name)


def test_train_parallel_threads_uneven_rounds():
    """train_parallel over ThreadComm: 5 data items on 2 replicas -> the last
    round has one participant (average_slots divides by participants)."""
    import paper_1701_03980_b200 as dy
    from paper_1701_03980_b200.params import materialize_pending

    R = 2
    batches = _batches(R, 3)[:5]
    reps = []
    for _ in range(R):
        pools = dy.new_poolset(128, 128, 64)
        m = dy.Model(pools, seed=3)
        task = W.RNNLM(dy, m, VOCAB, E, H, L)
        reps.append((m, task, dy.Trainer(m, "sgd")))
    materialize_pending()

    def replica(r, comm):
        m, task, tr = reps[r]
        plan = ParallelPlan(R, lambda cg, model, datum, task=task: task.loss(cg, datum), forward_mb=128,
                            backward_mb=128)
        return train_parallel(plan, m, tr, batches, 1, comm=comm)

    outs = _run_threads(R, replica)
    assert outs[0] == outs[1]
    # oracle: rounds of dp_step over the participants of each round
    om = orc.Model(orc.new_poolset(), seed=3)
    otask = W.RNNLM(orc, om, VOCAB, E, H, L)
    otr = orc.Trainer(om, "sgd")
    total = 0.0
    for k in range(3):
        idx = [k * R + r for r in range(R) if k * R + r < len(batches)]

        def graph_for(j, idx=idx):
            g = orc.ComputationGraph(orc.new_poolset())
            return g, otask.loss(g, batches[idx[j]])

        total += sum(orc.dp_step(om, otr, graph_for, len(idx)))
    parity(outs[0][0], total, what="epoch loss")
    for p in om.parameters:
        got = pvals(next(x for x in reps[0][0].parameters if x.name == p.name))
        parity(got, np.asarray(p.values, dtype=np.float64).reshape(-1), what=p.name)
