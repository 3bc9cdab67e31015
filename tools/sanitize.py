"""Small workloads through every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): persistent cluster recurrences (fwd/bwd),
TMA tcgen05 GEMMs, grouped SIMT GEMMs, pnls, gathers / scatters, cells,
trainer updates.  Run under gpurun, e.g.
    compute-sanitizer --tool racecheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1701_03980_b200 as dy  # noqa: E402
from paper_1701_03980_b200 import workloads as W  # noqa: E402


def run(task_fn, data, steps=2, rule="adam"):
    pools = dy.new_poolset(512, 512, 64)
    cg, m = dy.ComputationGraph(pools), dy.Model(pools, seed=1)
    task = task_fn(m)
    tr = dy.Trainer(m, rule)
    for s in range(steps):
        cg.renew()
        d = data[s]
        loss = task.loss(cg, *d) if isinstance(d, tuple) else task.loss(cg, d)
        cg.backward(loss)
        v = float(cg.value(loss).data[0])
        tr.update()
    torch.cuda.synchronize()
    return v


# PTB-shaped, reduced width: cluster recurrence (MB 16 -> BS 16), TMA GEMMs (V 2048)
ptb = W.minibatches(W.ptb_corpus(3, 32, vocab=2048, mean_len=8.0), 16)
print("ptb", run(lambda m: W.RNNLM(dy, m, 2048, 64, 128, 2), ptb))
tiny = W.tiny_lm_corpus(4, 2)
print("tiny", run(lambda m: W.RNNLM(dy, m, 1000, 64, 64, 1), [[s] for s in tiny]))
td = W.tree_corpus(5, 2, vocab=200)
print("tree", run(lambda m: W.TreeClassifier(dy, m, 200, 5, 32, 48), list(zip(td.trees, td.labels))))
tg = W.tagger_corpus(6, 2, n_types=500)
print("tagger", run(lambda m: W.CharTagger(dy, m, tg, 32, 16, 16, 8, 16), tg.sentences))
gru = W.minibatches(W.ptb_corpus(7, 8, vocab=300, mean_len=6.0), 4)
print("gru", run(lambda m: W.RNNLM(dy, m, 300, 16, 32, 1, "gru"), gru, rule="sgd"))
print("sanitize workloads done")
