"""Time Alg 5 (delta-triggered mixed precision, K6m) fits: python tools/mixed_time.py cfg delta iters."""
import sys
import time
import torch

sys.path.insert(0, ".")
import paper_2407_12208_b200 as mpk  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_blobs_1m_d64"
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = synth.CONFIGS[name]
X, _, C0 = synth.make(cfg, n=cfg.n, seed=0)
Xd, Cd = torch.from_numpy(X).cuda(), torch.from_numpy(C0).cuda()
km = mpk.KMeans(cfg.n, cfg.d, cfg.k, cfg.work, cfg.dists[0], norm=cfg.norms[0], delta=delta)
mpk.kmeans_set_timing(km.h, True)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    rc, sse, it = km.fit(Xd, Cd, max_iter=iters, tol=-1.0)
    torch.cuda.synchronize()
    dt = time.time() - t
st = km.stats()
print(name, "delta", delta, "iters", it, "wall %.3f s" % dt, "eta %.4f" % st["eta"],
      {k: round(v, 3) for k, v in st.items() if k.startswith("t_")})
