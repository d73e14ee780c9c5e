"""NEXT #3: the image-segmentation sweep of PAPER.md:1160-1171 on the synthetic 512 x 512 RGB
image (config C2, min-max = /255): k in {5, 10, 20, 50}; k-means in working precision (fp32),
Alg 3 (all distances in u_l) and Alg 5 (delta = 2) with u_l in {fp16, E5M2}; D^2 seeding in
the same u_l with fixed uniforms; the MX remedy (power-of-two row scaling, reading Z9 B) with
Alg 3; up to 100 Lloyd iterations (tol 1e-4). Prints one JSON line
per run: SSE (final, normalised space), SSE / SSE_working, iterations, eta, underflow and
non-finite counts. Usage: python tools/image_sweep.py [out.json]."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_12208_b200 as mpk  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["c2_image_512"]
X, _, _ = synth.make(cfg, n=cfg.n, seed=0)
n, d = X.shape
Xd = torch.from_numpy(X).cuda()
rows = []
for k in (5, 10, 20, 50):
    u = np.random.default_rng(100 + k).random(k)
    base = None
    for mode, dist in [("working", "fp32"), ("low", "fp16"), ("mp", "fp16"), ("low", "e5m2"),
                       ("mp", "e5m2"), ("mx", "fp16"), ("mx", "e5m2")]:
        # "mx": Alg 3 with the MX remedy of PAPER.md:1166-1171 as power-of-two row scaling
        # (KMEANS_GUARD_POW2, reading Z9 B)
        km = mpk.KMeans(n, d, k, "fp32", dist, norm="minmax",
                        delta=2.0 if mode == "mp" else None,
                        guard="pow2" if mode == "mx" else False)
        idx = km.seed(Xd, u)                      # Alg 1 in u_l (Alg 3 / Alg 5 step 1)
        C0 = Xd[torch.from_numpy(idx).cuda()]
        torch.cuda.synchronize()
        t = time.time()
        rc, sse, it = km.fit(Xd, C0.contiguous(), max_iter=100, tol=1e-4)
        torch.cuda.synchronize()
        dt = time.time() - t
        st = km.stats()
        km.close()
        if mode == "working":
            base = sse
        r = {"k": k, "mode": mode, "dist": dist, "sse": sse, "sse_rel": sse / base,
             "iters": it, "eta": st.get("eta"), "n_underflow": st.get("n_underflow"),
             "n_nonfinite": st.get("n_nonfinite"), "rc": rc, "fit_ms": dt * 1e3}
        rows.append(r)
        print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
