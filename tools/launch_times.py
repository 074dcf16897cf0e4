"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel name, count and time."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = []
for r in rows[start + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
        per.append((r[ki][:90], v))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = defaultdict(lambda: [0, 0.0])
for name, us in per[skip:]:
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us / 1e3:8.3f} ms {100 * us / tot:5.1f}%  x{n:<4d} {name}")
print(f"{tot / 1e3:8.3f} ms total ({len(per) - skip} launches)")
