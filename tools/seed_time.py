"""Time kmeans_seed_d2: python tools/seed_time.py [cfg] [k]."""
import sys
import time
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_12208_b200 as mpk  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_vq_10m"
cfg = synth.CONFIGS[name]
k = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.k
X, _, _ = synth.make(cfg, n=cfg.n, seed=0)
Xd = torch.from_numpy(X).cuda()
km = mpk.KMeans(cfg.n, cfg.d, k, cfg.work, cfg.dists[0], norm=cfg.norms[0])
u = np.random.default_rng(1).random(k)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    idx = km.seed(Xd, u)
    torch.cuda.synchronize()
    dt = time.time() - t
print(name, "k", k, "seed wall %.3f s" % dt, "per round %.3f ms" % (dt / max(1, k - 1) * 1e3),
      "distinct", len(set(idx.tolist())))
