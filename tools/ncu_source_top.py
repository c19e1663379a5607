#!/usr/bin/env python
"""Top stalled SASS lines of an `ncu --page source --csv` export, with the stall
reasons per line.  python tools/ncu_source_top.py SOURCE.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = rows[2:]
ia = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
f = lambda s: float(s or 0)  # noqa: E731
tot = sum(f(r[ia]) for r in data)
print(f"total samples {tot:.0f}")
for r in sorted(data, key=lambda r: -f(r[ia]))[:n]:
    reasons = sorted(((f(r[i]), hdr[i][6:]) for i in st), reverse=True)[:3]
    rs = " ".join(f"{k}:{v:.0f}" for v, k in reasons if v > 0)
    print(f"{r[0][-5:]} {100 * f(r[ia]) / tot:5.1f}% {r[1][:60]:60s} x{r[ie]:>8s} {rs}")
