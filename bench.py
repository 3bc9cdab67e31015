#!/usr/bin/env python
"""Benchmark: train words/sec of the PTB-shaped 2-layer LSTM RNNLM (BASELINE
configs[1]: H=256, V=10k, E=128, lock-step minibatch 64, Adam lr 1e-3,
sparse lookup updates) on the B200 executor, one rank per GPU.

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config ptb64|ptb16|tiny|tree|tagger]

One step = one minibatch: renew -> build the graph through the reference API
(host) -> backward (native batched forward+backward) -> value(loss) ->
trainer.update (native), i.e. the reference runner's inner loop
(bench/tasks.py:480-488).  Words are counted as len(ids)-1 per sentence
(bench/tasks.py:460-461,473).

Reported numbers (rank 0 prints one JSON line):
  value  device throughput: the K minibatch graphs are constructed and handed
         to the executor (dg_graph_append) before the timed region; the timed
         region (CUDA events per step, max over ranks) is planning + every
         kernel of forward, backward, gradient exchange and update; L2 is
         flushed between steps (outside the per-step windows).
  e2e    the full public-API loop with host graph construction, the executor's
         H2D of each step's node tables/inputs and the D2H of the loss.
  roofline  the op class with the largest measured device time, timed live with
         CUDA events around its launches inside the value region.
  cpu_baseline  the oracle (numpy restatement of the reference, same graph,
         same seeds) on this host's cores, bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "ptb64": dict(kind="rnnlm", vocab=10_000, embed=128, hidden=256, layers=2, mb=64),
    "ptb16": dict(kind="rnnlm", vocab=10_000, embed=128, hidden=256, layers=2, mb=16),
    "tiny": dict(kind="rnnlm", vocab=1000, embed=64, hidden=64, layers=1, mb=1),
    "tree": dict(kind="tree", vocab=18_300, embed=128, hidden=150, labels=5, mb=1),
    "tagger": dict(kind="tagger", mb=1),
}
METRIC = "train words/sec (RNNLM, BiLSTM tagger), sents/sec (Tree-LSTM); 1/8 B200"


_WL = None


def workloads():
    """paper_1701_03980_b200/workloads.py loaded by path: pure numpy corpus
    generators + graph builders generic over the engine namespace, so the
    reference arm never imports the product package (or maps its .so)."""
    global _WL
    if _WL is None:
        import importlib.util

        spec = importlib.util.spec_from_file_location(
            "dg_bench_workloads", os.path.join(ROOT, "paper_1701_03980_b200", "workloads.py"))
        _WL = importlib.util.module_from_spec(spec)
        sys.modules[spec.name] = _WL
        spec.loader.exec_module(_WL)
    return _WL


def bench_config(name, cfg, world):
    """The `config` object of the JSON line (identical for both arms)."""
    return {"workload": name, **cfg, "global_batch": cfg["mb"] * world, "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write)"}


def make_task(dy, model, cfg, tagger_data=None):
    W = workloads()

    if cfg["kind"] == "rnnlm":
        return W.RNNLM(dy, model, cfg["vocab"], cfg["embed"], cfg["hidden"], cfg["layers"])
    if cfg["kind"] == "tree":
        return W.TreeClassifier(dy, model, cfg["vocab"], cfg["labels"], cfg["embed"], cfg["hidden"])
    return W.CharTagger(dy, model, tagger_data)


def make_data(cfg, n_steps, rank, world, seed=1):
    """Per-rank minibatches: rank r takes batches r, r+R, ... of one corpus."""
    W = workloads()

    total = n_steps * world
    if cfg["kind"] == "rnnlm":
        if cfg["vocab"] == 1000:
            sents = W.tiny_lm_corpus(seed, total * cfg["mb"])
        else:
            sents = W.ptb_corpus(seed, total * cfg["mb"], vocab=cfg["vocab"])
        batches = W.minibatches(sents, cfg["mb"])
        mine = batches[rank::world][:n_steps]
        return mine, [W.lm_words(b) for b in mine], None
    if cfg["kind"] == "tree":
        td = W.tree_corpus(seed, total)
        items = list(zip(td.trees, td.labels))[rank::world][:n_steps]
        return items, [1] * len(items), None
    # WSJ-shaped: vocabulary (rare words -> char path) counted over 40k sentences
    tg = W.tagger_corpus(seed, max(total, 200), corpus_sentences=40_000)
    items = tg.sentences[rank::world][:n_steps]
    return items, [len(s) for s in items], tg


def unit_of(cfg):
    return "sents/sec" if cfg["kind"] == "tree" else "words/sec"


def call_loss(task, cg, datum):
    if isinstance(datum, tuple):
        return task.loss(cg, datum[0], datum[1])
    return task.loss(cg, datum)


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------


class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 9:
                    self.samples.append(parts)
            except Exception:  # noqa: BLE001 - sampling is best effort
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU arm: the oracle (numpy restatement of the reference), bounded sample
# ---------------------------------------------------------------------------


def cpu_threads(n):
    """Cap the BLAS pool of the oracle (numpy/OpenBLAS) at n threads."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=n)


def cpu_throughput(cfg, budget_s: float, seed=1, threads=None):
    if threads is not None:
        with cpu_threads(threads):
            return cpu_throughput(cfg, budget_s, seed)
    from oracle import engine as orc

    data, units, tg = make_data(cfg, 64, 0, 1, seed)
    pools = orc.new_poolset()
    cg, model = orc.ComputationGraph(pools), orc.Model(pools, seed=seed)
    task = make_task(orc, model, cfg, tg)
    tr = orc.Trainer(model, "adam")
    done_units, t0, steps = 0, time.perf_counter(), 0
    while steps < len(data):
        cg.renew()
        loss = call_loss(task, cg, data[steps])
        cg.backward(loss)
        float(cg.value(loss).data[0])
        tr.update()
        done_units += units[steps]
        steps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return done_units / dt, steps, done_units, dt


def cpu_baseline(cfg, name, budget_s):
    """The oracle on this host at the box's full thread count (the reported
    value) and at one BLAS thread (both are reported)."""
    nproc = os.cpu_count() or 1
    v, s, u, dt = cpu_throughput(cfg, budget_s, threads=nproc)
    v1, s1, u1, dt1 = cpu_throughput(cfg, max(1.0, budget_s / 3), threads=1)
    return {"value": v, "unit": unit_of(cfg), "cores": nproc, "kind": "port",
            "sample": f"{s} graphs ({u} units) of the {name} workload through the numpy oracle in {dt:.1f} s, "
                      f"BLAS threads={nproc}",
            "single_thread": {"value": v1, "cores": 1,
                              "sample": f"{s1} graphs ({u1} units) in {dt1:.1f} s, BLAS threads=1"}}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    nproc = os.cpu_count() or 1
    steps, units, dt = 0, 0, 0.0
    with cpu_threads(nproc):
        # warmup + K timed steps, each a bounded sample (~budget/K seconds)
        cpu_throughput(cfg, min(5.0, 1.0 * args.warmup))
        for _ in range(args.steps):
            v, s, u, d = cpu_throughput(cfg, args.ref_budget / max(1, args.steps))
            steps += s
            units += u
            dt += d
    value = units / dt
    line = {
        "metric": METRIC, "value": value, "unit": unit_of(cfg), "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(1, steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.config, cfg, world), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": unit_of(cfg), "cores": nproc, "kind": "port",
                         "sample": f"{steps} minibatches ({units} units) of the {args.config} workload through the "
                                   f"numpy oracle (the reference algorithm restated), {dt:.1f} s, "
                                   f"BLAS threads={nproc}"},
        "e2e": {"value": value, "unit": unit_of(cfg), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def _traffic():
    """Measured DRAM bytes per launch by op class (tools/summarize_profiles.py
    writes profiles/traffic.json from one ncu --set full capture each)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        return {k: v["dram_bytes"] for k, v in t["classes"].items()}, t["source"]
    except (OSError, KeyError, ValueError):
        return {}, None


def _roofline(name, d, peaks):
    """achieved = algorithmic FLOPs (or bytes) per launch / mean launch time;
    traffic = the ncu-measured DRAM bytes per launch of the same kernel."""
    traffic, source = _traffic()
    r = _roofline_core(name, d, peaks)
    if r is not None:
        r["traffic"] = traffic.get(name)
        if r["traffic"] is not None:
            r["traffic_source"] = source
            r["algorithmic_bytes_per_launch"] = d["bytes"] / max(1, d["launches"])
    return r


def _roofline_core(name, d, peaks):
    avg_ms = d["ms"] / max(1, d["launches"])
    if avg_ms <= 0:
        return None
    if d["flops"] > 0:
        achieved = d["flops"] / max(1, d["launches"]) / (avg_ms * 1e-3) / 1e12
        peak = peaks.get("bf16_tflops", 1590.0)
        r = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
             "traffic": None, "kernel": name,
             "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if "bf16_tflops" in peaks
             else "fallback 1.59 PFLOP/s bf16 (B200_PROFILING.md)",
             # fp32 parity: tensor-core classes issue 3 TF32 MMAs per product
             # (dense TF32 = 1/2 of bf16); the recurrence runs on the FP32 pipe
             "tf32x3_issued_frac": 3 * achieved / (peak / 2),
             "fp32_simt_frac": achieved / (148 * 128 * 2 * 1.965e-3)}
    else:
        achieved = d["bytes"] / max(1, d["launches"]) / (avg_ms * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
             "traffic": None, "kernel": name,
             "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
             else "fallback 6.65 TB/s (B200_PROFILING.md)"}
    r["ms_per_launch"] = avg_ms
    return r


def measure(dy, cfg, K, Wm, world, rank, local, profile, seed=1):
    """One configuration: e2e through the public API, device-timed value over
    pre-built graphs, optional per-class profile pass."""
    import torch
    import torch.distributed as dist

    from paper_1701_03980_b200.parallel import DataParallel

    data, units, tg = make_data(cfg, K + Wm + K, rank, world, seed)
    mb_pool = 1024 if cfg["kind"] == "rnnlm" and cfg["mb"] >= 16 else 128
    pools = dy.new_poolset(mb_pool, mb_pool, 64)
    cg = dy.ComputationGraph(pools)
    model = dy.Model(pools, seed=1)
    task = make_task(dy, model, cfg, tg)
    trainer = dy.Trainer(model, "adam")
    dp = DataParallel(model, sparse=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def maxr(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sumr(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return float(t.item())

    def api_step(g, datum):
        g.renew()
        loss = call_loss(task, g, datum)
        g.backward(loss)
        lv = float(g.value(loss).data[0])
        dp.sync()
        trainer.update()
        return lv

    # ---- warmup (full API path) ------------------------------------------
    for i in range(Wm):
        api_step(cg, data[i])
    barrier()

    # ---- e2e: public API, host construction + H2D + D2H inside ------------
    c0 = cg._counters()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    t_wall = time.perf_counter()
    step_wall = []
    for i in range(K):
        t_s = time.perf_counter()
        api_step(cg, data[Wm + i])
        step_wall.append(time.perf_counter() - t_s)
    e1.record(stream)
    barrier()
    wall = time.perf_counter() - t_wall
    e2e_ms = maxr(e0.elapsed_time(e1))
    c1 = cg._counters()
    e2e_units = sumr(sum(units[Wm : Wm + K]))
    h2d_per_step = (c1[6] - c0[6]) / K
    d2h_per_step = 4.0

    # ---- value: pre-constructed graphs, device-timed ----------------------
    def build_graphs(offset):
        out = []
        for i in range(K):
            p = dy.new_poolset(mb_pool, mb_pool, 1)
            g = dy.ComputationGraph(p)
            loss = call_loss(task, g, data[offset + i])
            g._prepare()  # hand the node table to the executor before timing
            out.append((g, loss))
        return out

    graphs = build_graphs(Wm + K)
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    launches0 = sum(int(g._counters()[5]) for g, _ in graphs)
    with Clocks(local) as clk:
        barrier()
        for i, (g, loss) in enumerate(graphs):
            flush.zero_()  # L2 flush, outside the step window
            starts[i].record(stream)
            g.backward(loss)
            dp.sync()
            trainer.update()
            ends[i].record(stream)
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_ms = maxr(sum(step_ms))
    launches = sum(int(g._counters()[5]) for g, _ in graphs) - launches0
    launches += K * (1 + len(model.lookups))  # trainer: dense multi-tensor + one per touched table
    value_units = sumr(sum(units[Wm + K : Wm + 2 * K]))
    res = {
        "value": value_units / (dev_ms * 1e-3), "unit": unit_of(cfg), "ms_per_step": dev_ms / K,
        "e2e": {"value": e2e_units / (e2e_ms * 1e-3), "unit": unit_of(cfg), "h2d_bytes_per_step": h2d_per_step,
                "d2h_bytes_per_step": d2h_per_step, "ms_per_step": e2e_ms / K, "wall_s": wall,
                # host wall time of each API step (diagnostic: the loop blocks on value(loss))
                "step_wall_ms": {"median": 1e3 * statistics.median(step_wall), "max": 1e3 * max(step_wall)}},
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    if not profile:
        return res

    # ---- per-class device time (a separate pass: CUDA events around every
    # launch cost host time that must not be inside the value region) ------
    prof_classes = ("gemm_fwd", "gemm_dx", "gemm_dw", "pnls_fwd", "pnls_bwd", "elementwise", "gather",
                    "scatter_add", "bias_colsum", "rnn_fwd", "rnn_bwd", "other")
    del graphs
    graphs = build_graphs(Wm + K)
    for g, _ in graphs:
        g.profile_enable(prof_classes)
        g.profile_reset()
    barrier()
    for g, loss in graphs:
        flush.zero_()
        g.backward(loss)
        dp.sync()
        trainer.update()
    barrier()
    kinds = {}
    for c in prof_classes:
        tot = {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0}
        for g, _ in graphs:
            r = g.profile_read(c)
            for k2 in tot:
                tot[k2] += r[k2]
        kinds[c] = tot
    peaks = _peaks()
    dom = max(kinds, key=lambda c: kinds[c]["ms"])
    res["roofline"] = _roofline(dom, kinds[dom], peaks)
    res["rooflines"] = {c: _roofline(c, kinds[c], peaks) for c in kinds if kinds[c]["ms"] > 0}
    res["kernel_share"] = {c: round(kinds[c]["ms"] / max(1e-9, sum(v["ms"] for v in kinds.values())), 4)
                           for c in kinds}
    res["kernels"] = kinds
    return res


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1701_03980_b200 as dy

    K, Wm = args.steps, args.warmup
    res = measure(dy, cfg, K, Wm, world, rank, local, profile=True)
    # the other BASELINE configs (same contract, shorter runs) beside the headline
    others = {}
    if world == 1 and not args.only:
        for name in ("ptb16", "tree", "tagger", "tiny"):
            if name == args.config:
                continue
            c2 = CONFIGS[name]
            k2 = max(K, 20) if c2["kind"] != "rnnlm" or c2["mb"] == 1 else K
            r2 = measure(dy, c2, k2, max(Wm, 3), world, rank, local, profile=False)
            if not args.no_cpu:
                r2["cpu_baseline"] = cpu_baseline(c2, name, args.other_cpu_budget)
            r2["config"] = bench_config(name, c2, world)
            r2["steps"], r2["warmup"] = k2, max(Wm, 3)
            others[name] = r2

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline(cfg, args.config, args.cpu_budget)
        line = {
            "metric": METRIC,
            "value": res["value"],
            "unit": unit_of(cfg),
            "n_gpus": world,
            "steps": K,
            "warmup": Wm,
            "ms_per_step": res["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": bench_config(args.config, cfg, world),
            "e2e": res["e2e"],
            "gpu_launches": res["gpu_launches"],
            "roofline": res["roofline"],
            "rooflines": res["rooflines"],
            "kernel_share": res["kernel_share"],
            "kernels": res["kernels"],
            "clocks": res["clocks"],
            "cpu_baseline": cpu,
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="ptb64", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=30.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", action="store_true", help="headline config only (skip the other BASELINE configs)")
    ap.add_argument("--other-cpu-budget", type=float, default=3.0)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun
        if args.impl == "b200":
            import torch

            have = torch.cuda.device_count()
            if have < args.gpus:
                sys.exit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
        port = 29500 + (os.getpid() % 2000)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
