"""Shared test helpers: backend contexts and the parity comparator.

Comparator (SURVEY 7 "the parity metric itself needs an atol floor"):
    |gpu - ref| <= rtol * |ref| + atol_frac * max|ref|
with rtol = 1e-4 and atol_frac = 1e-6 for losses, gradients and SGD parameters
(the north-star bar "within rtol 1e-4 in fp32").  N-step Adam parameters are
additionally allowed a band of 2 * lr * steps: Adam's m/sqrt(v) turns
last-bit gradient differences into +-lr steps (SURVEY 7 measured the oracle
failing rtol against ITSELF in fp32 vs fp64); the Adam kernel itself is
checked exactly on injected gradients (test_gpu_semantics.py).
"""

from __future__ import annotations

import numpy as np

RTOL = 1e-4
ATOL_FRAC = 1e-6


def parity(got, ref, rtol=RTOL, atol_frac=ATOL_FRAC, band=0.0, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    scale = float(np.abs(ref).max(initial=0.0))
    tol = rtol * np.abs(ref) + np.maximum(atol_frac * scale, band)
    err = np.abs(got - ref)
    bad = err > tol
    assert not bad.any(), (
        f"{what}: {int(bad.sum())}/{bad.size} over tol; worst err {err.max():.3e} "
        f"(ref scale {scale:.3e})"
    )


def gpu_ctx(seed=1, mb=256.0):
    import paper_1701_03980_b200 as dy

    pools = dy.new_poolset(mb, mb, mb)
    return dy, dy.ComputationGraph(pools), dy.Model(pools, seed=seed)


def oracle_ctx(seed=1, dtype=np.float32):
    from oracle import engine as orc

    pools = orc.new_poolset(dtype=dtype)
    return orc, orc.ComputationGraph(pools), orc.Model(pools, seed=seed)


def pvals(x):
    """Host values of a parameter of either backend."""
    v = x.values
    return np.array(v if isinstance(v, np.ndarray) else v.data, dtype=np.float64).reshape(-1)


def pgrad(x):
    g = x.gradient
    return np.array(g if isinstance(g, np.ndarray) else g.data, dtype=np.float64).reshape(-1)
