"""One C5-shaped fit (device input) for profiling: python tools/one_fit.py [iters] [dist]."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_12208_b200 as mpk  # noqa: E402
import synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dist = sys.argv[2] if len(sys.argv) > 2 else "fp16"
cfg = synth.CONFIGS["c5_vq_10m"]
X, _, C0 = synth.make(cfg, n=cfg.n, seed=0)
Xd = torch.from_numpy(X).cuda()
Cd = torch.from_numpy(C0).cuda()
km = mpk.KMeans(cfg.n, cfg.d, cfg.k, "fp32", dist, norm="zscore")
lab = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
for _ in range(2):
    rc, sse, it = km.fit(Xd, Cd, max_iter=iters, tol=-1.0, labels=lab)
torch.cuda.synchronize()
st = km.stats()
print("rc", rc, "sse", sse, "iters", it, {k: v for k, v in st.items() if k.startswith("t_")})
print("changed fraction per iteration:", [round(c / cfg.n, 4) for c in st["changed_t"]])
