"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv):
per-kernel totals over the last `--frac` of the launches (steady state)."""
import collections
import csv
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
items = [(r[ki], float(r[vi].replace(",", ""))) for r in data if r[vi]]
tail = items[int(len(items) * (1 - frac)):]
tot, cnt = collections.defaultdict(float), collections.Counter()
for k, v in tail:
    key = k.split("(")[0][:80]
    tot[key] += v
    cnt[key] += 1
T = sum(tot.values())
print(f"launches {len(items)} (summarised {len(tail)}), total {T / 1e6:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"{v / 1e6:8.3f} ms {100 * v / T:5.1f}% n={cnt[k]:5d} avg={v / cnt[k] / 1e3:8.1f}us  {k}")
