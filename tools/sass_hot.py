"""Summarise an ncu `--page source --print-source sass --csv` dump: top SASS
instructions by warp-stall samples with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(float(r[samp] or 0) for r in data)
print(f"total samples {tot:.0f}")
top = sorted(data, key=lambda r: -float(r[samp] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    s = float(r[samp] or 0)
    reasons = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v > 0)
    print(f"{100 * s / tot:5.1f}% {r[ix['Address']]:>6} {r[ix['Source']][:60]:60s} {rs}")
