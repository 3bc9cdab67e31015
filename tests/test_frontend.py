"""The scripting frontend (pkg/frontend/src/dyngraph) on the B200 backend.

* The reference's `dyngraph` module runs UNCHANGED over this package through
  the `compat/dyncore` alias: it builds the same node tables as the core-call
  spelling of the same programs (CPU; needs /root/reference, skipped where it
  is absent).
* Golden traces (tests/golden/frontend.npz, made by
  tests/golden/make_frontend_golden.py from the reference frontend on the
  reference core): the core-call spelling reproduces them on the oracle (CPU)
  and on the device (GPU): Fig. 1 per-epoch losses within the north-star rtol
  1e-4 (the reference's own CLI-vs-script bar is 1e-6 between two runs of the
  same numpy engine, fetests/test_programs.py:82; the measured device error is
  printed), the Fig. 5 encoding within 1e-6.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests import frontend_programs as P
from tests.helpers import parity

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_FE = "/root/reference/pkg/frontend/src"
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "frontend.npz"))
PAIRS = P.synthetic_pairs(3, 60)


def _node_table(cg):
    return [[n.kind, list(n.inputs), list(n.shape.dims), n.shape.batch] for n in cg.nodes]


_REF_SCRIPT = r"""
import json, sys
sys.path.insert(0, ROOT)
import dyncore, dyngraph as dy
from tests import frontend_programs as P
assert dyncore.__name__ == "paper_1701_03980_b200", dyncore.__name__
pairs, vocab, nc = P.synthetic_pairs(3, 60)
dy.init(mem="48", seed=P.SEED)
model = dy.Model()
W_p = model.add_parameters((nc, 2 * P.EMB)); b_p = model.add_parameters(nc)
E = model.add_lookup_parameters((len(vocab), P.EMB))
w1, w2, label = pairs[0]
dy.renew_cg()
W = dy.parameter(W_p); b = dy.parameter(b_p)
score = dy.softmax(W * dy.concatenate([E[vocab[w1]], E[vocab[w2]]]) + b)
loss = dy.pickneglogsoftmax(score, label)
cg = dy._cg()
table = [[n.kind, list(n.inputs), list(n.shape.dims), n.shape.batch] for n in cg.nodes]
print(json.dumps({"classifier": table, "values": [float(x) for x in model.core.parameters[0].values.data[:4]]}))
"""


@pytest.mark.skipif(not os.path.isdir(REF_FE), reason="reference frontend not present (GPU box)")
def test_reference_frontend_runs_unchanged_over_the_package():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "compat"), REF_FE]))
    out = subprocess.run([sys.executable, "-c", f"ROOT={ROOT!r}\n" + _REF_SCRIPT], capture_output=True,
                         text=True, env=env, cwd="/tmp")
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout)

    import paper_1701_03980_b200 as dy

    pairs, vocab, nc = PAIRS
    cg, model = P._ctx(dy, "48")
    W_p = model.add_parameters((nc, 2 * P.EMB))
    b_p = model.add_parameters(nc)
    E = model.add_lookup_parameters(len(vocab), P.EMB)
    w1, w2, label = pairs[0]
    cg.renew()
    W, b = dy.ops.parameter(cg, W_p), dy.ops.parameter(cg, b_p)
    x = dy.ops.concatenate([dy.ops.lookup(cg, E, vocab[w1]), dy.ops.lookup(cg, E, vocab[w2])])
    dy.ops.pickneglogsoftmax(dy.ops.softmax(dy.ops.add(dy.ops.matmul(W, x), b)), label)
    assert got["classifier"] == _node_table(cg)
    assert np.array_equal(np.float32(got["values"]), W_p.values.data[:4])


def test_core_spelling_reproduces_reference_frontend_on_oracle():
    from oracle import engine as orc

    parity(P.core_classifier_program(orc, *PAIRS), GOLD["classifier/per_epoch"], atol_frac=0,
           rtol=1e-6, what="Fig. 1 per-epoch losses (oracle)")
    assert np.allclose(P.core_tree_program(orc), GOLD["tree/encoding"], rtol=0, atol=1e-7)


def test_tree_program_graph_shape():
    import paper_1701_03980_b200 as dy

    cg = P.core_tree_program(dy, build_only=True)
    kinds = [n.kind for n in cg.nodes]
    assert kinds.count("tanh") == 2 and kinds.count("lookup") == 3 and kinds.count("parameter") == 2


@pytest.mark.gpu
def test_classifier_program_matches_reference_frontend():
    import paper_1701_03980_b200 as dy

    got = np.array(P.core_classifier_program(dy, *PAIRS))
    want = GOLD["classifier/per_epoch"]
    print("Fig. 1 per-epoch max rel err vs reference frontend:", float(np.max(np.abs(got - want) / np.abs(want))))
    parity(got, want, what="Fig. 1 per-epoch losses (device)")


@pytest.mark.gpu
def test_tree_encoder_program_matches_reference_frontend():
    import paper_1701_03980_b200 as dy

    got = P.core_tree_program(dy)
    assert np.allclose(got, GOLD["tree/encoding"], rtol=0, atol=1e-6), (got, GOLD["tree/encoding"])


@pytest.mark.gpu
def test_prediction_surface():
    import paper_1701_03980_b200 as dy

    pairs, vocab, nc = P.synthetic_pairs(4, 20)
    cg, model = P._ctx(dy, "48")
    W_p = model.add_parameters((nc, 2 * P.EMB))
    b_p = model.add_parameters(nc)
    E = model.add_lookup_parameters(len(vocab), P.EMB)
    for w1, w2, label in pairs:
        cg.renew()
        x = dy.ops.concatenate([dy.ops.lookup(cg, E, vocab[w1]), dy.ops.lookup(cg, E, vocab[w2])])
        score = dy.ops.softmax(dy.ops.add(dy.ops.matmul(dy.ops.parameter(cg, W_p), x), dy.ops.parameter(cg, b_p)))
        v = cg.value(score).data
        assert v.shape == (nc,) and abs(float(v.sum()) - 1.0) < 1e-5
