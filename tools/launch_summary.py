"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel totals and
shares (cold-cache, serialised launches: compare shares, not absolute times)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    v = float(r[ival].replace(",", ""))
    u = r[iunit]
    us = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
    name = r[iname].split("(")[0].replace("void ", "").replace("mpk::", "")
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    agg[name].append(us)
tot = sum(sum(v) for v in agg.values())
print(f"{'total us':>12} {'share':>6} {'n':>4} {'avg us':>10}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v):12.1f} {100 * sum(v) / tot:5.1f}% {len(v):4d} {sum(v) / len(v):10.1f}  {k}")
print(f"{tot:12.1f} total")
