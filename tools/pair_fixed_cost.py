"""Launch-time decomposition of the pair kernel at the C3 shape (d = 64, k = 256, fp16): a few
kmeans_assign calls at n = 1 row-block per CTA pair and at n = 1M (run under ncu to read the
kernel durations; MPK_PAIR_DBG selects the debug skeleton)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_12208_b200 as mpk  # noqa: E402

for n in (148 * 128, 1_000_000):
    X = torch.randn(n, 64, device="cuda")
    C = X[:256].clone()
    km = mpk.KMeans(n, 64, 256, "fp32", "fp16")
    mpk.kmeans_set_centroids(km.h, C)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(4):
        km.assign(X, lab)
    torch.cuda.synchronize()
    km.close()
print("done")
