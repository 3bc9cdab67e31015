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
    vals = []
    for s in range(steps):
        cg.renew()
        d = data[s]
        loss = task.loss(cg, *d) if isinstance(d, tuple) else task.loss(cg, d)
        cg.backward(loss)
        if os.environ.get("DG_SAN_EARLY") and s == 0:
            import numpy as np
            from paper_1701_03980_b200.graph import Expression
            for i in range(len(cg.nodes) - 1, len(cg.nodes) - 6, -1):
                gi = np.asarray(cg.gradient(Expression(cg, i, cg.generation)).data, dtype=np.float64)
                print("  early", i, cg.nodes[i].kind, repr(float(np.abs(gi).sum())))
            p0 = m.parameters[0]
            print("  early p0", p0.name, repr(float(np.abs(np.asarray(p0.values.data, dtype=np.float64)).sum())))
        vals.append(repr(float(cg.value(loss).data[0])))
        if os.environ.get("DG_SAN_NODES") and s == 0:
            import numpy as np
            from paper_1701_03980_b200.graph import Expression
            for i, node in enumerate(cg.nodes):
                gi = np.asarray(cg.gradient(Expression(cg, i, cg.generation)).data, dtype=np.float64)
                vi = np.asarray(cg.value(Expression(cg, i, cg.generation)).data, dtype=np.float64)
                print("  node", i, node.kind, repr(float(np.abs(gi).sum())), repr(float(np.abs(vi).sum())))
        if os.environ.get("DG_SAN_DUMP") and s == 0:
            import numpy as np
            for x in list(m.parameters) + list(m.lookups):
                g = x.gradient
                g = np.asarray(g if isinstance(g, np.ndarray) else g.data, dtype=np.float64)
                print("  grad0", x.name, repr(float(g.sum())), repr(float(np.abs(g).sum())))
        tr.update()
        if os.environ.get("DG_SAN_NODES") and s == 0:
            import numpy as np
            from paper_1701_03980_b200.graph import Expression
            for i, node in enumerate(cg.nodes):
                gi = np.asarray(cg.gradient(Expression(cg, i, cg.generation)).data, dtype=np.float64)
                vi = np.asarray(cg.value(Expression(cg, i, cg.generation)).data, dtype=np.float64)
                print("  node", i, node.kind, repr(float(np.abs(gi).sum())), repr(float(np.abs(vi).sum())))
        if os.environ.get("DG_SAN_DUMP") and s == 0:
            import numpy as np
            for x in list(m.parameters) + list(m.lookups):
                v = x.values
                v = np.asarray(v if isinstance(v, np.ndarray) else v.data, dtype=np.float64)
                print("  val1", x.name, repr(float(v.sum())))
    torch.cuda.synchronize()
    return " ".join(vals)


ONLY = sys.argv[1:]


def want(name):
    return not ONLY or name in ONLY


# PTB-shaped, reduced width: cluster recurrence (MB 16 -> BS 16), TMA GEMMs (V 2048)
ptb = W.minibatches(W.ptb_corpus(3, 32, vocab=2048, mean_len=8.0), 16)
if want("ptb"):
    print("ptb", run(lambda m: W.RNNLM(dy, m, 2048, 64, 128, 2), ptb))
tiny = W.tiny_lm_corpus(4, 2)
if want("tiny"):
    print("tiny", run(lambda m: W.RNNLM(dy, m, 1000, 64, 64, 1), [[s] for s in tiny]))
td = W.tree_corpus(5, 2, vocab=200)
if want("tree"):
    print("tree", run(lambda m: W.TreeClassifier(dy, m, 200, 5, 32, 48), list(zip(td.trees, td.labels))))
tg = W.tagger_corpus(6, 2, n_types=500)
if want("tagger"):
    print("tagger", run(lambda m: W.CharTagger(dy, m, tg, 32, 16, 16, 8, 16), tg.sentences))
gru = W.minibatches(W.ptb_corpus(7, 8, vocab=300, mean_len=6.0), 4)
if want("gru"):
    print("gru", run(lambda m: W.RNNLM(dy, m, 300, 16, 32, 1, "gru"), gru, rule="sgd"))
# headline-shaped output layer (V 10k, H 256, MB 64): the persistent logits
# GEMM with TMA stores, the split dW units and both backward overlap windows
big = W.minibatches(W.ptb_corpus(8, 64, vocab=10000, mean_len=16.0), 64)
if want("ptb_big"):
    print("ptb_big", run(lambda m: W.RNNLM(dy, m, 10000, 128, 256, 2), big, steps=1))
print("sanitize workloads done")
