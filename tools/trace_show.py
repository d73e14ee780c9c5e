"""Print the per-tile clock64 trace written by MPK_PAIR_TRACE (leader CTA of pair 0).

Columns (cycles relative to the first stamp): MMA thread t_empty_ok / commit_done; epilogue
(warp 4 lane 0) t_full_ok / fold_done / arrived; on the last tile of a row-block also
merge_done / xchg_done / rowend_done (0 when not stamped).
"""
import sys
import numpy as np

for path in sys.argv[1:]:
    a = np.loadtxt(path, dtype=np.int64)
    t0 = a[0, 1]
    r = np.where(a[:, 1:] > 0, a[:, 1:] - t0, 0)
    print(f"--- {path}")
    for i in list(range(0, 8)) + list(range(100, 108)):
        print(i, *r[i], " issue=%d fold=%d" % (r[i, 1] - r[i, 0], r[i, 3] - r[i, 2]))
    print("cycles/tile (tiles 100..200):", (r[200, 2] - r[100, 2]) / 100)
