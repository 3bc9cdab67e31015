"""Summarise gpurun_out ncu artefacts into profiles/<round>_*.{txt,json}."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PROF, exist_ok=True)

# launch list -> per-kernel totals (second half = steady-state step)
rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
items = [(r[ki], float(r[vi].replace(",", ""))) for r in data if r[vi]]
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, v in items:
    key = k.split("(")[0]
    tot[key] += v
    cnt[key] += 1
T = sum(tot.values())
lines = [f"# ncu --metrics gpu__time_duration.sum launch list of `python bench.py --steps 2 --warmup 1 --only`",
         f"# (cold-cache, serialised by ncu: compare SHARES, not absolutes). launches={len(items)} total={T/1e6:.3f} ms", ""]
share = {}
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"{v/1e6:9.3f} ms {100*v/T:5.1f}%  n={cnt[k]:5d}  avg={v/cnt[k]/1e3:8.1f} us  {k}")
    share[k] = v / T
open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

summary = {"launch_share": share, "launches": len(items), "full": {}}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]
for name in ("full_tma", "full_rnn", "full_row", "full_tc", "full_simt", "full_cell"):
    path = os.path.join(OUT, name + ".ncu-rep")
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h = r[0]
    launches = []
    for row in r[2:]:
        d = {k: row[h.index(k)] for k in want if k in h}
        d["kernel"] = row[h.index("Kernel Name")][:120]
        launches.append(d)
    summary["full"][name] = launches
json.dump(summary, open(os.path.join(PROF, f"{tag}_summary.json"), "w"), indent=1)
print("\n".join(lines[:25]))
for n, ls in summary["full"].items():
    for d in ls:
        print(n, {k: d.get(k) for k in ("kernel", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                          "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")})
