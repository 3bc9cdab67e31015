"""Every kernel path the executor can take produces the same results: the
full-size PTB parity test (tests/test_gpu_parity.py) re-run in a subprocess
with each fast path switched off, so the fallbacks stay parity-green too.

  DG_RNN_CLUSTER=0  persistent LSTM kernels exchanging through L2 + global
                    arrival counters instead of cluster distributed smem
  DG_RNN=0          no persistent recurrence: level-batched GEMM + fused cells
  DG_TMA=0          cp.async tcgen05 GEMM instead of the TMA warp-specialised one
  DG_TMA_CONV=0     TMA GEMM reading pre-split residual copies instead of forming
                    them in shared memory
  DG_TC=0           SIMT GEMMs only
  DG_SCHED_CACHE=0  schedules rebuilt for every graph
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "rnn_no_cluster": {"DG_RNN_CLUSTER": "0"},
    "rnn_off": {"DG_RNN": "0"},
    "tma_off": {"DG_TMA": "0"},
    "tma_presplit": {"DG_TMA_CONV": "0"},
    "tma_a_in_smem": {"DG_TMA_AT": "0"},
    "tma_ungrouped": {"DG_TMA_GROUP": "0"},
    "pdl_off": {"DG_PDL": "0"},
    "tma_lite_off": {"DG_TMA_LITE": "0"},
    "tensor_cores_off": {"DG_TC": "0"},
    "schedule_cache_off": {"DG_SCHED_CACHE": "0"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_ptb_parity_on_every_kernel_path(variant):
    env = dict(os.environ, **VARIANTS[variant])
    tests = ["tests/test_gpu_parity.py::test_ptb_mb16_full_size_vs_oracle",
             "tests/test_gpu_parity.py::test_char_tagger_full_size_vs_oracle"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
