"""Summarise gpurun_out ncu artefacts into profiles/<tag>_launches.txt,
profiles/<tag>_summary.json and profiles/traffic.json.

Every metric of the --set full captures is stored in base units (bytes,
nanoseconds, percent, plain counts): row 1 of `ncu --page raw --csv` holds the
unit of each column and is applied here, so Kbyte / Mbyte / Gbyte figures can
be compared directly.  profiles/traffic.json maps bench.py's op classes to the
measured DRAM bytes (read + write) per launch of their kernel, which bench.py
reports as roofline.traffic."""
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
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
os.makedirs(PROF, exist_ok=True)

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
         "cycle": 1, "Kcycle": 1e3, "Mcycle": 1e6, "%": 1, "": 1,
         "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}
BASE = {"byte": "byte", "nsecond": "ns", "ns": "ns", "cycle": "cycle", "%": "%", "byte/second": "byte/s", "hz": "hz"}


def base_unit(u):
    for b, name in BASE.items():
        if u.endswith(b) and SCALE.get(u) is not None:
            return name
    return u


# launch list -> per-kernel totals
rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
items = [(r[ki], float(r[vi].replace(",", "")) * SCALE[r[ui]]) for r in data if r[vi]]  # ns
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, v in items:
    key = k.split("(")[0]
    tot[key] += v
    cnt[key] += 1
T = sum(tot.values())
lines = ["# ncu --metrics gpu__time_duration.sum launch list of `python bench.py --steps 2 --warmup 1 --only`",
         f"# (cold-cache, serialised by ncu: compare SHARES, not absolutes). launches={len(items)} total={T/1e6:.3f} ms", ""]
share = {}
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"{v/1e6:9.3f} ms {100*v/T:5.1f}%  n={cnt[k]:5d}  avg={v/cnt[k]/1e3:8.1f} us  {k}")
    share[k] = v / T
open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

summary = {"units": "bytes, ns, cycles, % (ncu units normalised)", "launch_share": share, "launches": len(items),
           "full": {}}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__cluster_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum"]
for fn in sorted(os.listdir(OUT)):
    if not (fn.startswith("full_") and fn.endswith(".ncu-rep")):
        continue
    name = fn[: -len(".ncu-rep")]
    raw = subprocess.run(["ncu", "-i", os.path.join(OUT, fn), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    h, units = r[0], r[1]
    launches = []
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")][:120]}
        for k in want:
            if k not in h:
                continue
            j = h.index(k)
            txt = row[j].replace(",", "")
            try:
                d[k] = float(txt) * SCALE.get(units[j], 1.0)
                d.setdefault("_units", {})[k] = base_unit(units[j])
            except ValueError:
                d[k] = txt
        if isinstance(d.get("dram__bytes_read.sum"), float) and isinstance(d.get("dram__bytes_write.sum"), float):
            d["dram_bytes"] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        launches.append(d)
    summary["full"][name] = launches
json.dump(summary, open(os.path.join(PROF, f"{tag}_summary.json"), "w"), indent=1)

# bench op class -> kernel name fragment of its (single) kernel
CLASS_KERNEL = {"rnn_fwd": "rnn_fwd_cl_kernel", "rnn_bwd": "rnn_bwd_cl_kernel", "pnls_fwd": "row_reg_kernel<2",
                "pnls_bwd": "row_reg_kernel<3", "gather": "gather_rows_kernel",
                "scatter_add": "scatter_rows_kernel", "bias_colsum": "colsum_partial_group_kernel"}
traffic = {"source": f"profiles/{tag}_summary.json", "unit": "bytes per launch (dram read + write)", "classes": {}}
for cls, frag in CLASS_KERNEL.items():
    hits = [d for ls in summary["full"].values() for d in ls if frag in d["kernel"] and "dram_bytes" in d]
    if hits:
        traffic["classes"][cls] = {"dram_bytes": sum(d["dram_bytes"] for d in hits) / len(hits),
                                   "launches_captured": len(hits), "kernel": hits[0]["kernel"]}
json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
print("\n".join(lines[:25]))
for n, ls in summary["full"].items():
    for d in ls:
        print(n, {k: d.get(k) for k in ("kernel", "gpu__time_duration.sum", "dram_bytes",
                                          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")})
