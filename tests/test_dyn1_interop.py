"""DYN1 persistence interop with the REAL reference (SURVEY 8(f)3,
pkg/src/dyncore/params.py:128-189): fixtures written by the reference's
Model.save (tests/golden/make_dyn1_golden.py) are read by this package, and
this package's files are byte-identical to the reference's for the same
model.  The reader below is an independent restatement of the format used as
the checker."""

import os
import struct

import numpy as np
import pytest

from paper_1701_03980_b200 import workloads as W
from tests.helpers import parity

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INIT = os.path.join(GOLD, "ref_init.dyn")
TRAINED = os.path.join(GOLD, "ref_trained.dyn")


def read_dyn1(path):
    blob = open(path, "rb").read()
    assert blob[:4] == b"DYN1"
    version, count = struct.unpack_from("<II", blob, 4)
    assert version == 1
    pos, out = 12, {}
    for _ in range(count):
        kind, nlen = struct.unpack_from("<BH", blob, pos)
        name = blob[pos + 3 : pos + 3 + nlen].decode()
        pos += 3 + nlen
        rank = blob[pos]
        dims = struct.unpack_from(f"<{rank}I", blob, pos + 1)
        pos += 1 + 4 * rank
        n = int(np.prod(dims))
        out[name] = (kind, dims, np.frombuffer(blob, "<f4", n, pos).copy())
        pos += 4 * n
    assert pos == len(blob)
    return out


def build(dy, seed=11, pools=None):
    pools = pools or dy.new_poolset(64, 64, 64)
    model = dy.Model(pools, seed=seed)
    task = W.RNNLM(dy, model, 50, 6, 8, 1)
    dy.ClassFactoredSoftmax(model, 8, {i: i % 3 for i in range(50)}, "cf")
    return pools, model, task


def test_host_writer_matches_reference_bytes(tmp_path):
    import paper_1701_03980_b200 as dy

    _, model, _ = build(dy)
    out = tmp_path / "m.dyn"
    model.save(str(out))
    assert out.read_bytes() == open(INIT, "rb").read()


@pytest.mark.gpu
def test_device_writer_matches_reference_bytes(tmp_path):
    """Values materialised on the device and read back by save()."""
    import paper_1701_03980_b200 as dy

    pools, model, task = build(dy)
    cg = dy.ComputationGraph(pools)
    cg.value(task.loss(cg, [W.tiny_lm_corpus(21, 1, vocab=50)[0]]))  # device storage now live
    out = tmp_path / "m.dyn"
    model.save(str(out))
    assert out.read_bytes() == open(INIT, "rb").read()


@pytest.mark.gpu
def test_reference_file_loads_on_device_and_trains_like_the_reference(tmp_path):
    """Load ref_init.dyn into a differently seeded device model, train the
    reference's 3 SGD steps on the device, save, and compare with the
    reference's own ref_trained.dyn (rtol 1e-4); then resume from the
    reference's trained file and check the device sees its exact values."""
    import paper_1701_03980_b200 as dy

    pools, model, task = build(dy, seed=99)
    model.load(INIT)
    init = read_dyn1(INIT)
    for p in model.parameters:
        assert np.array_equal(p.values.data.reshape(-1), init[p.name][2])
    cg = dy.ComputationGraph(pools)
    tr = dy.Trainer(model, "sgd")
    for sent in W.tiny_lm_corpus(21, 3, vocab=50):
        cg.renew()
        cg.backward(task.loss(cg, [sent]))
        tr.update()
    out = tmp_path / "trained.dyn"
    model.save(str(out))
    got, want = read_dyn1(str(out)), read_dyn1(TRAINED)
    assert [(k, v[0], v[1]) for k, v in got.items()] == [(k, v[0], v[1]) for k, v in want.items()]
    for name in want:
        parity(got[name][2], want[name][2], what=f"trained {name}")

    pools2, resumed, task2 = build(dy, seed=5)
    resumed.load(TRAINED)
    cg2 = dy.ComputationGraph(pools2)
    cg2.value(task2.loss(cg2, [W.tiny_lm_corpus(22, 1, vocab=50)[0]]))  # force device use
    for x in list(resumed.parameters) + list(resumed.lookups):
        vals = x.values.data if hasattr(x.values, "data") else x.values
        assert np.array_equal(np.asarray(vals).reshape(-1), want[x.name][2]), x.name
