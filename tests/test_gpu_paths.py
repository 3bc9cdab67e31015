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
  DG_PLAN_CACHE=0   launch plans rebuilt for every graph (no plan cache)
  DG_CUDA_GRAPH=1   cached plans replayed as CUDA graphs (default: launch by launch)
  DG_AFFCELL=0      gate affine and gated cell of a small level as a grouped
                    GEMM + cell kernel instead of one fused launch
  DG_TREE_PERSIST=0 one fused launch per tree level instead of one
                    cooperative launch for every level
  DG_TMA_GSPLIT=0, DG_TMA_PERS=0, DG_TMA_TSTORE=0, DG_TMA_PERS_SPLIT=0
                    split-K only through clusters / no persistent kernel /
                    its epilogue with thread stores and in-kernel split
                    reduction / persistent kernel for unsplit problems only
  DG_EARLY_DW=0     the output layer's dW after the backward recurrences instead
                    of overlapped with the first one (run on the MB64 test)

(the fused affine + cell path is exercised by the Tree-LSTM test added to
the list below)
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
    "plan_cache_off": {"DG_PLAN_CACHE": "0"},
    "cuda_graph_on": {"DG_CUDA_GRAPH": "1"},
    "affine_cell_unfused": {"DG_AFFCELL": "0"},
    "tree_levels_per_launch": {"DG_TREE_PERSIST": "0"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_ptb_parity_on_every_kernel_path(variant):
    env = dict(os.environ, **VARIANTS[variant])
    tests = ["tests/test_gpu_parity.py::test_ptb_mb16_full_size_vs_oracle",
             "tests/test_gpu_parity.py::test_char_tagger_full_size_vs_oracle",
             "tests/test_gpu_parity.py::test_tree_lstm_full_size_vs_oracle"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# output-layer GEMM paths that only the MB64 shapes reach (workspace split-K
# for the K = 10^4 dX, the persistent logits kernel and its TMA stores)
GEMM_VARIANTS = {
    "tma_cluster_split_only": {"DG_TMA_GSPLIT": "0"},
    "tma_pers_off": {"DG_TMA_PERS": "0"},
    "tma_pers_thread_stores": {"DG_TMA_TSTORE": "0"},
    "tma_pers_unsplit_only": {"DG_TMA_PERS_SPLIT": "0"},
    "dw_after_recurrences": {"DG_EARLY_DW": "0"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(GEMM_VARIANTS))
def test_ptb_mb64_parity_on_every_gemm_path(variant):
    env = dict(os.environ, **GEMM_VARIANTS[variant])
    tests = ["tests/test_gpu_parity.py::test_ptb_mb64_full_size_vs_oracle_sgd"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


_REPLAY = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_1701_03980_b200 as dy
from paper_1701_03980_b200 import workloads as W
# equal padded length -> equal structure: the plan of step 0 serves steps 1..
# (each batch: one 22-token sentence + 7 shorter ones, so masks differ)
corpus = W.ptb_corpus(9, 4000, vocab=500)
longs = [s for s in corpus if len(s) == 22][:6]
shorts = [s for s in corpus if 2 <= len(s) < 22][:42]
batches = [[longs[k]] + shorts[7 * k: 7 * k + 7] for k in range(6)]
pools = dy.new_poolset(256, 256, 64)
cg, m = dy.ComputationGraph(pools), dy.Model(pools, seed=2)
task = W.RNNLM(dy, m, 500, 32, 64, 2)
tr = dy.Trainer(m, "adam")
losses = []
for b in batches:
    cg.renew()
    loss = task.loss(cg, b)
    cg.backward(loss)
    losses.append(float(cg.value(loss).data[0]))
    tr.update()
h = hashlib.sha256()
for x in list(m.parameters) + list(m.lookups):
    v = x.values
    h.update(np.ascontiguousarray(v if isinstance(v, np.ndarray) else v.data, dtype=np.float32).tobytes())
st = cg.plan_stats()
print(json.dumps({"losses": losses, "params": h.hexdigest(), "hits": int(st[5]), "replays": int(st[6])}))
"""


@pytest.mark.gpu
def test_plan_cache_and_cuda_graph_replay_are_bitwise_identical():
    """Six minibatches of one structure (same padded length, different ids,
    labels and masks): the cached plans (patched data, CUDA-graph replay)
    give bit-identical losses and parameters to planning every graph."""
    outs = {}
    for name, env in {"cached": {"DG_CUDA_GRAPH": "1"}, "uncached": {"DG_PLAN_CACHE": "0"},
                      "no_graph": {}}.items():
        r = subprocess.run([sys.executable, "-c", f"ROOT={ROOT!r}\n" + _REPLAY], cwd=ROOT, capture_output=True,
                           text=True, timeout=600, env=dict(os.environ, **env))
        assert r.returncode == 0, r.stderr[-3000:]
        outs[name] = __import__("json").loads(r.stdout.strip().splitlines()[-1])
    assert outs["cached"]["hits"] >= 10 and outs["cached"]["replays"] >= 6, outs["cached"]
    assert outs["uncached"]["hits"] == 0 and outs["no_graph"]["replays"] == 0
    for name in ("uncached", "no_graph"):
        assert outs[name]["losses"] == outs["cached"]["losses"], name
        assert outs[name]["params"] == outs["cached"]["params"], name
