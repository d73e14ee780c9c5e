"""Summarise an ncu report: key raw metrics and the SASS hot spots (stall samples)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        print(f"{k:80s} {vals[i]:>16s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src))
h = rows[1]
i_src, i_s, i_ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[i_s]), int(r[i_ex]), r[i_src].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
op, opx = Counter(), Counter()
for s, e, t in data:
    o = t.split()[0] if t else ""
    if o.startswith("@"):
        o = t.split()[1]
    o = o.split(".")[0]
    op[o] += s
    opx[o] += e
print("stall samples by opcode:")
for o, s in op.most_common(15):
    print(f"  {o:12s} {100 * s / tot:5.1f}%  inst={opx[o]}")
print("top instructions:")
for s, e, t in sorted(data, key=lambda x: -x[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"  {100 * s / tot:5.1f}% {e:12d}  {t}")
