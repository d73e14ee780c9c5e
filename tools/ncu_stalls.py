"""Per-instruction stall reasons from an ncu report's source page: totals by reason for the
hottest instructions (by execution count bucket) and the top instructions per reason.
Usage: python tools/ncu_stalls.py report.ncu-rep"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ix = {c: h.index(c) for c in reasons}
i_src, i_ex, i_addr = h.index("Source"), h.index("Instructions Executed"), h.index("Address")
tot = defaultdict(float)
per = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    ex = int(r[i_ex] or 0)
    st = {c: float(r[ix[c]] or 0) for c in reasons}
    per.append((r[i_addr], r[i_src].strip(), ex, st))
    for c in reasons:
        tot[c] += st[c]
T = sum(tot.values())
print("all instructions:", ", ".join(f"{c[6:]} {100 * v / T:.1f}%" for c, v in sorted(tot.items(), key=lambda t: -t[1]) if v > 0))
buckets = defaultdict(lambda: defaultdict(float))
for a, s, ex, st in per:
    for c in reasons:
        buckets[ex][c] += st[c]
print("by execution count (top buckets by samples):")
for ex, st in sorted(buckets.items(), key=lambda t: -sum(t[1].values()))[:8]:
    S = sum(st.values())
    print(f"  exec={ex:>10d} samples={S:8.0f} ({100 * S / T:4.1f}%):",
          ", ".join(f"{c[6:]} {100 * v / S:.0f}%" for c, v in sorted(st.items(), key=lambda t: -t[1])[:6] if v > 0))
for c in sorted(tot, key=lambda c: -tot[c])[:5]:
    top = sorted(per, key=lambda t: -t[3][c])[:6]
    print(f"top {c}:")
    for a, s, ex, st in top:
        print(f"    {st[c]:8.0f} exec={ex:>10d} {s[:90]}")
