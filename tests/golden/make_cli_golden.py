"""Golden runs of the REAL reference CLI (build container only):

    python tests/golden/make_cli_golden.py

Writes small data files with the reference's own generator
(pkg/src/dyncore/bench/gen.py) into tests/golden/cli/, runs
`python -m dyncore.bench.cli <task> ...` (bench/cli.py) on them and stores the
per-epoch (loss, metric) of every run in tests/golden/cli/runs.json, including
a --save / --load resume pair.  tests/test_cli.py replays the same command
lines through paper_1701_03980_b200.cli on the device.
"""

from __future__ import annotations

import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(HERE, "cli")
REF = "/root/reference/pkg/src"
EPOCH_RE = re.compile(r"^epoch=(\d+) loss=(\S+) metric=(\S+) speed=(\S+)$")

# name: (task, gen seed, gen sizes, extra CLI args)
RUNS = {
    "rnnlm": ("rnnlm", 3, dict(sentences=40), ["--epochs", "2", "--trainer", "adam"]),
    "rnnlm_mb4": ("rnnlm", 3, dict(sentences=40), ["--epochs", "2", "--trainer", "sgd", "--batch-size", "4"]),
    "tagger": ("tagger", 4, dict(sentences=30), ["--epochs", "2", "--trainer", "adam"]),
    "tagger-char": ("tagger-char", 5, dict(sentences=30), ["--epochs", "2", "--unk-threshold", "2"]),
    # (not adagrad: with the reference's eps = 1e-20 the first AdaGrad step is
    # lr * sign(g) even for rounding-level gradients, so a +-1e-9 gradient
    # element that cancels differently under another summation order moves a
    # weight by +-0.1; the AdaGrad kernel has its own known-answer test)
    "treelstm": ("treelstm", 6, dict(sentences=20), ["--epochs", "2", "--trainer", "adam"]),
    "pairclass": ("pairclass", 7, dict(sentences=60), ["--epochs", "3", "--trainer", "sgd", "--seed", "5"]),
    "pairclass_mb8": ("pairclass", 7, dict(sentences=60), ["--epochs", "2", "--trainer", "momentum",
                                                           "--batch-size", "8"]),
    "earlystop": ("earlystop", 8, dict(sentences=40), ["--epochs", "2", "--threshold", "2.0"]),
}


def files(name):
    return os.path.join(DATA, f"{name}.train"), os.path.join(DATA, f"{name}.dev")


def run_cli(task, train, dev, extra, cwd):
    env = dict(os.environ, PYTHONPATH=REF)
    p = subprocess.run([sys.executable, "-m", "dyncore.bench.cli", task, "--train", train, "--dev", dev, *extra],
                       capture_output=True, text=True, env=env, cwd=cwd, check=True)
    eps = [m.groups()[1:3] for m in map(EPOCH_RE.match, p.stdout.splitlines()) if m]
    return [[float(a), float(b)] for a, b in eps]


def main():
    sys.path.insert(0, REF)
    from dyncore.bench.gen import generate

    os.makedirs(DATA, exist_ok=True)
    out = {}
    for name, (task, seed, sizes, extra) in RUNS.items():
        data_name = name.split("_")[0]
        train, dev = files(data_name)
        if not os.path.exists(train):
            generate(task, seed, train, dev, **sizes)
        out[name] = {"task": task, "data": data_name, "args": extra,
                     "epochs": run_cli(task, train, dev, extra, "/tmp")}
    # save -> load resume (tests/test_bench.py:259-272)
    train, dev = files("pairclass")
    model = "/tmp/dg_cli_resume.dyn"
    base = ["--epochs", "1", "--trainer", "sgd", "--lr", "0.1"]
    first = run_cli("pairclass", train, dev, base + ["--save", model], "/tmp")
    second = run_cli("pairclass", train, dev, base + ["--load", model], "/tmp")
    out["resume"] = {"task": "pairclass", "data": "pairclass", "args": base, "first": first, "second": second}
    with open(os.path.join(DATA, "runs.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out)[:2000])


if __name__ == "__main__":
    main()
