"""Golden traces of the reference's scripting frontend (run in the build
container, where /root/reference exists):

    python tests/golden/make_frontend_golden.py

Runs the reference `dyngraph` module UNCHANGED over the reference core
(pkg/frontend/src/dyngraph + pkg/src/dyncore) on the Fig. 1 classifier and
the Fig. 5 tree-encoder programs of tests/frontend_programs.py and writes
tests/golden/frontend.npz (per-epoch losses, the tree encoding).  The GPU
test replays the same programs on the device and compares.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
for p in ("/root/reference/pkg/frontend/src", "/root/reference/pkg/src"):
    if p not in sys.path:
        sys.path.insert(0, p)

import dyncore  # noqa: E402
import dyngraph  # noqa: E402

from tests import frontend_programs as P  # noqa: E402

CLASSIFIER_DATA = (3, 60)  # synthetic_pairs(seed, n)


def main():
    assert dyncore.__file__.startswith("/root/reference/"), dyncore.__file__
    pairs, vocab, nc = P.synthetic_pairs(*CLASSIFIER_DATA)
    out = {
        "classifier/per_epoch": np.array(P.classifier_program(dyngraph, pairs, vocab, nc), dtype=np.float64),
        "tree/encoding": np.array(P.tree_program(dyngraph), dtype=np.float64),
    }
    np.savez(os.path.join(HERE, "frontend.npz"), **out)
    print({k: v.tolist() for k, v in out.items()})


if __name__ == "__main__":
    main()
