"""Per-kernel average of an ncu launch-list CSV: python tools/upd_show.py [csv]."""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/upd.csv").read().splitlines()
i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[i:]))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    if len(r) > vi:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in d.items():
    print(f"{k:70s} n={len(v):3d} avg_us={sum(v) / len(v) / 1000:8.1f}")
