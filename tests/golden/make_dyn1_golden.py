"""DYN1 interop fixtures from the REAL reference (build container only):

    python tests/golden/make_dyn1_golden.py

* ref_init.dyn  — a model (seed 11) saved by the reference's Model.save right
  after registration (pkg/src/dyncore/params.py:128-143);
* ref_trained.dyn — the same model after 3 SGD steps of a tiny RNNLM on the
  reference (so its values are not reproducible from the RNG alone).
The GPU tests load both on the device and compare byte-for-byte / value-for-
value, and check the device writer produces ref_init.dyn's exact bytes.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")

import dyncore as ref  # noqa: E402

from paper_1701_03980_b200 import workloads as W  # noqa: E402


def build(mod, model):
    """Roster of the interop model: an RNNLM (E, rnn.*, W, b) + a CFSM head."""
    task = W.RNNLM(mod, model, 50, 6, 8, 1)
    mod.ClassFactoredSoftmax(model, 8, {i: i % 3 for i in range(50)}, "cf")
    return task


def main():
    assert ref.__file__.startswith("/root/reference/")
    pools = ref.new_poolset(64, 64, 64)
    model = ref.Model(pools, seed=11)
    task = build(ref, model)
    model.save(os.path.join(HERE, "ref_init.dyn"))
    cg = ref.ComputationGraph(pools)
    tr = ref.Trainer(model, "sgd")
    for sent in W.tiny_lm_corpus(21, 3, vocab=50):
        cg.renew()
        cg.backward(task.loss(cg, [sent]))
        tr.update()
    model.save(os.path.join(HERE, "ref_trained.dyn"))
    for f in ("ref_init.dyn", "ref_trained.dyn"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
