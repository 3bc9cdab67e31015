"""`dyngraph <task>` on the B200 backend (reference
pkg/src/dyncore/bench/cli.py, bench/tasks.py, tests/test_bench.py).

The golden runs (tests/golden/cli/runs.json) are the REAL reference CLI on
data files written by the reference generator (tests/golden/
make_cli_golden.py).  Here the same command lines run through
`python -m paper_1701_03980_b200.cli` on the device: same line format,
per-epoch mean loss within rtol 1e-4 and the same dev metric (accuracy to one
example, perplexity within rtol 1e-4); --save / --load resumes."""

import json
import os
import re
import subprocess
import sys

import pytest

from paper_1701_03980_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(ROOT, "tests", "golden", "cli")
RUNS = json.load(open(os.path.join(DATA, "runs.json")))
START_RE = re.compile(r"^startup_secs=[-\d.e+]+$")
EPOCH_RE = re.compile(r"^epoch=(\d+) loss=([-\d.e+]+) metric=([-\d.e+]+) speed=([-\d.e+]+)$")
REF_SRC = "/root/reference/pkg/src"


def files(name):
    return os.path.join(DATA, f"{name}.train"), os.path.join(DATA, f"{name}.dev")


def run(task, data, args, cwd):
    train, dev = files(data)
    return subprocess.run([sys.executable, "-m", "paper_1701_03980_b200.cli", task, "--train", train, "--dev", dev,
                           *args], capture_output=True, text=True, cwd=cwd,
                          env=dict(os.environ, PYTHONPATH=ROOT))


def epochs(proc):
    lines = proc.stdout.strip().splitlines()
    assert START_RE.match(lines[0]), lines[0]
    return [[float(m.group(2)), float(m.group(3))] for m in map(EPOCH_RE.match, lines[1:]) if m]


def n_dev(data):
    from paper_1701_03980_b200.cli import read_labeled_docs, read_pairs, read_tagged, read_token_lines, read_trees

    dev = files(data)[1]
    reader = {"rnnlm": read_token_lines, "tagger": read_tagged, "tagger-char": read_tagged, "treelstm": read_trees,
              "pairclass": read_pairs, "earlystop": read_labeled_docs}[data]
    items = reader(dev)
    return sum(map(len, items)) if data.startswith("tagger") else len(items)


# -- host side (CPU) --------------------------------------------------------------


def test_missing_file_fails_with_diagnostic(tmp_path):
    p = subprocess.run([sys.executable, "-m", "paper_1701_03980_b200.cli", "pairclass", "--train",
                        str(tmp_path / "none"), "--dev", str(tmp_path / "none")], capture_output=True, text=True,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    assert p.returncode == 1 and p.stderr.startswith("error:") and "Traceback" not in p.stderr


def test_sparse_workers_conflict():
    train, dev = files("pairclass")
    p = subprocess.run([sys.executable, "-m", "paper_1701_03980_b200.cli", "pairclass", "--train", train, "--dev",
                        dev, "--workers", "2", "--sparse", "on"], capture_output=True, text=True,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    assert p.returncode == 1 and "sparse" in p.stderr


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
@pytest.mark.parametrize("data", ["rnnlm", "tagger", "tagger-char", "treelstm", "pairclass", "earlystop"])
def test_readers_and_vocab_match_reference(data):
    sys.path.insert(0, REF_SRC)
    try:
        from dyncore.bench import tasks as rt
        from dyncore.bench.vocab import Vocab as RefVocab
    finally:
        sys.path.remove(REF_SRC)
    train = files(data)[0]
    if data == "treelstm":
        ours, ref = cli.read_trees(train), rt.parse_trees(train)

        def key(t):
            return (t.token, t.label, tuple(key(c) for c in t.children))

        assert [key(t) for t in ours] == [key(t) for t in ref]
        toks = [tok for t in ours for tok in cli._leaves(t)]
    else:
        reader = {"rnnlm": ("read_token_lines", "_read_token_lines"), "tagger": ("read_tagged", "_read_tagged"),
                  "tagger-char": ("read_tagged", "_read_tagged"), "pairclass": ("read_pairs", "_read_pairs"),
                  "earlystop": ("read_labeled_docs", "_read_labeled_docs")}[data]
        ours, ref = getattr(cli, reader[0])(train), getattr(rt, reader[1])(train)
        assert [list(map(tuple, x)) if isinstance(x, list) else x for x in ours] == \
               [list(map(tuple, x)) if isinstance(x, list) else x for x in ref] or ours == ref
        toks = [str(x) for item in ours for x in (item if isinstance(item, (list, tuple)) else [item])]
    for thr in (1, 2):
        assert cli.Vocab.build(toks, thr, ("<s>",)).i2t == RefVocab.build(toks, thr, ("<s>",)).i2t


# -- device runs vs the reference CLI ------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("name", [k for k in RUNS if k != "resume"])
def test_cli_matches_reference_run(name, tmp_path):
    spec = RUNS[name]
    p = run(spec["task"], spec["data"], spec["args"], str(tmp_path))
    assert p.returncode == 0, p.stderr
    got, want = epochs(p), spec["epochs"]
    assert len(got) == len(want)
    tol_metric = 1.0 / n_dev(spec["data"]) + 1e-9
    for (gl, gm), (wl, wm) in zip(got, want):
        assert abs(gl - wl) <= 1e-4 * abs(wl), (name, got, want)
        if spec["task"] == "rnnlm":
            assert abs(gm - wm) <= 1e-4 * abs(wm), (name, got, want)
        else:
            assert abs(gm - wm) <= tol_metric, (name, got, want)


@pytest.mark.gpu
def test_cli_save_then_load_continues(tmp_path):
    spec = RUNS["resume"]
    model = str(tmp_path / "m.dyn")
    first = run("pairclass", "pairclass", spec["args"] + ["--save", model], str(tmp_path))
    assert first.returncode == 0, first.stderr
    second = run("pairclass", "pairclass", spec["args"] + ["--load", model], str(tmp_path))
    assert second.returncode == 0, second.stderr
    (l1, _), (l2, _) = epochs(first)[0], epochs(second)[0]
    assert l2 < l1
    assert abs(l1 - spec["first"][0][0]) <= 1e-4 * spec["first"][0][0]
    assert abs(l2 - spec["second"][0][0]) <= 1e-4 * spec["second"][0][0]
