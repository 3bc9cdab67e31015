"""CPU oracle for the ComputationGraph forward/backward/update hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this; only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline leg
(`--impl reference` and the `cpu_baseline` object) may use it, and only as the
checker / the timed CPU reference.  It is a numpy restatement of the reference
algorithm (arXiv 1701.03980 desk-scale `dyncore`, /root/reference/pkg/src/dyncore)
written from its behaviour, not copied from it.

Parity of the oracle itself is pinned by golden vectors generated from the real
reference in the build container (tests/golden/make_golden.py, committed
fixtures under tests/golden/, checked by tests/test_oracle_golden.py).
"""

from . import engine  # noqa: F401
