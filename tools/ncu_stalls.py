"""Stall reasons by SASS opcode class from an ncu source page (csv):
   ncu -i REP --page source --csv --kernel-name regex:K --print-source sass > src.csv
   python tools/ncu_stalls.py src.csv"""
import csv, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
iSrc = h.index("Source")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tab = defaultdict(lambda: defaultdict(float))
for r in data:
    t = r[iSrc].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    for c in reasons:
        tab[op][c] += f(r[h.index(c)])
tot = sum(sum(v.values()) for v in tab.values())
cols = [c for c in reasons if sum(tab[o][c] for o in tab) / tot > 0.01]
print(f"{'op':8s} {'total%':>7s} " + " ".join(f"{c[6:]:>10s}" for c in cols))
for op, v in sorted(tab.items(), key=lambda x: -sum(x[1].values()))[:16]:
    s = sum(v.values())
    print(f"{op:8s} {s / tot * 100:7.2f} " + " ".join(f"{v[c] / tot * 100:10.2f}" for c in cols))
print(f"{'all':8s} {100:7.2f} " + " ".join(f"{sum(tab[o][c] for o in tab) / tot * 100:10.2f}" for c in cols))
