"""Print the last step's launches of an ncu launch-list CSV (gpu__time_duration,
grid, block per kernel): tools/launchlist.py gpurun_out/step_launches_tree.csv [steps]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
L = {}
for r in data:
    L.setdefault(r[idi], {"k": r[ki]})[r[mi]] = (r[vi], r[ui])
items = [v for v in L.values() if "spin_kernel" not in v["k"]]
step = items[-(len(items) // nsteps):]
tot = 0.0
for it in step:
    d, u = it["gpu__time_duration.sum"]
    d = float(d.replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[u]
    tot += d
    print("%8.1f us grid %6s blk %4s %s" % (d, it["launch__grid_size"][0], it["launch__block_size"][0], it["k"][:80]))
print("launches %d total %.1f us" % (len(step), tot))
