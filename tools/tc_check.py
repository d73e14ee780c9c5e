"""Dev check: tcgen05 assign (pair or streaming kernel per MPK_TC_KIND) vs the oracle on a few
shapes, then a timing of kmeans_assign at the C5 shape. Not part of the test suite."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2407_12208_b200 as mpk  # noqa: E402
import synth  # noqa: E402

shapes = [(1000, 64, 256, 'fp16'), (4099, 128, 1024, 'fp16'), (3001, 32, 64, 'e5m2'),
          (2077, 128, 200, 'bf16'), (777, 200, 130, 'fp16'), (5000, 128, 1024, 'e5m2')]
for (n, d, k, dist) in shapes:
    X, _ = synth.blobs(n, d, 10, seed=0, dtype=np.float32)
    Xn, _, _ = oracle.normalize(X, 'zscore', work='fp32')
    Xn = Xn.astype(np.float32)
    C = synth.init_rows(Xn, k, 0)
    km = mpk.KMeans(n, d, k, 'fp32', dist)
    mpk.kmeans_set_centroids(km.h, torch.from_numpy(C).cuda())
    lab = torch.empty(n, dtype=torch.int32, device='cuda')
    sse = km.assign(torch.from_numpy(Xn).cuda(), lab)
    torch.cuda.synchronize()
    ref, dmin, _ = oracle.assign(Xn, C, work='fp32', dist=dist)
    print(n, d, k, dist, 'match', (lab.cpu().numpy() == ref).mean(), 'sse', sse,
          np.maximum(dmin, 0).sum(), flush=True)
    km.close()

n, d, k = 10_000_000, 128, 1024
X = torch.randn(n, d, device='cuda')
C = X[:k].clone()
for dist in ['fp16', 'e5m2']:
    km = mpk.KMeans(n, d, k, 'fp32', dist)
    mpk.kmeans_set_centroids(km.h, C)
    lab = torch.empty(n, dtype=torch.int32, device='cuda')
    for _ in range(2):
        km.assign(X, lab)
    torch.cuda.synchronize()
    t = time.perf_counter()
    R = 5
    for _ in range(R):
        km.assign(X, lab)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / R
    print(dist, 'assign (incl. prep of X each call) ms', dt * 1e3, flush=True)
    km.close()
