"""The scripting frontend (dyngraph surface, pkg/frontend/src/dyngraph) on
the B200 backend: the reference's frontend programs produce the same losses
and encodings as on the numpy oracle (GPU), and the surface itself behaves
like the reference's on the oracle engine (CPU)."""

import numpy as np
import pytest

from tests import frontend_programs as P
from tests.helpers import parity


def _oracle_fe():
    from oracle import engine as orc
    from paper_1701_03980_b200.dyngraph import Frontend

    return Frontend(orc)


def test_frontend_surface_on_oracle():
    import paper_1701_03980_b200.dyngraph as dyg

    for name in ("init", "renew_cg", "parameter", "lookup", "vectorInput", "inputVector", "concatenate",
                 "softmax", "tanh", "logistic", "pickneglogsoftmax", "Model", "model", "SimpleSGDTrainer",
                 "MomentumSGDTrainer", "AdagradTrainer", "AdamTrainer", "Expression"):
        assert hasattr(dyg, name), name
    fe = _oracle_fe()
    pairs, vocab, nc = P.synthetic_pairs(1, 12)
    losses = P.classifier_program(fe, pairs, vocab, nc, epochs=2)
    assert len(losses) == 2 and all(np.isfinite(losses))
    v = P.tree_program(fe)
    assert v.shape == (12,)
    fe.init()
    fe.renew_cg()
    e = fe.vectorInput([1.0, 2.0, 3.0])
    assert np.allclose((2 * e).npvalue(), [2.0, 4.0, 6.0])
    assert sum([e, e]).npvalue().tolist() == [2.0, 4.0, 6.0]


@pytest.mark.gpu
def test_classifier_program_matches_oracle():
    import paper_1701_03980_b200.dyngraph as dyg

    pairs, vocab, nc = P.synthetic_pairs(3, 60)
    got = P.classifier_program(dyg, pairs, vocab, nc)
    want = P.classifier_program(_oracle_fe(), pairs, vocab, nc)
    parity(got, want, what="per-epoch losses")


@pytest.mark.gpu
def test_tree_encoder_program_matches_oracle():
    import paper_1701_03980_b200.dyngraph as dyg

    got = P.tree_program(dyg)
    want = P.tree_program(_oracle_fe())
    assert np.allclose(got, want, atol=1e-6), (got, want)


@pytest.mark.gpu
def test_prediction_surface():
    import paper_1701_03980_b200.dyngraph as dyg

    pairs, vocab, nc = P.synthetic_pairs(4, 20)
    dyg.init(seed=1)
    model = dyg.Model()
    W_p = model.add_parameters((nc, 2 * P.EMB))
    b_p = model.add_parameters(nc)
    E = model.add_lookup_parameters((len(vocab), P.EMB))
    for w1, w2, label in pairs:
        dyg.renew_cg()
        score = dyg.softmax(dyg.parameter(W_p) * dyg.concatenate([E[vocab[w1]], E[vocab[w2]]]) + dyg.parameter(b_p))
        v = score.npvalue()
        assert v.shape == (nc,) and abs(float(v.sum()) - 1.0) < 1e-5
