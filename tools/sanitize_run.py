"""Small invocations of every kernel family for compute-sanitizer (memcheck / synccheck /
racecheck): the CTA-pair tcgen05 kernel in ASSIGN, FINAL and CAND modes (fp16, e5m2, guard),
the streaming tcgen05 kernel (MPK_TC_KIND=1), the CUDA-core kernels, the fused small-d
iteration, D^2 seeding and the virtual-rank exchange. Usage:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_12208_b200 as mpk  # noqa: E402
import synth  # noqa: E402


def fit(n, d, k, dist, guard=False, norm="zscore", iters=3, seed=0):
    X, _ = synth.blobs(n, d, max(2, k // 2), sigma=1.5, seed=seed, dtype=np.float32)
    C0 = synth.init_rows(X, k, seed)
    with mpk.KMeans(n, d, k, "fp32", dist, norm=norm, guard=guard) as km:
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        rc, sse, it = km.fit(torch.from_numpy(X).cuda(), torch.from_numpy(C0).cuda(),
                             max_iter=iters, tol=-1.0, labels=lab)
        km.assign(torch.from_numpy(X).cuda(), lab)
        st = km.stats()
    print(f"fit n={n} d={d} k={k} {dist} guard={guard}: sse={sse:.6e} kernel={st['dist_kernel']}"
          f" tc={st['tc_variant']} uncertified={st['n_final_uncertified']}", flush=True)


def main():
    torch.cuda.set_device(0)
    fit(3000, 128, 300, "fp16")                  # pair kernel: ASSIGN + FINAL + CAND
    fit(3000, 128, 300, "e5m2")                  # half split + the fp16 final-pass copy
    fit(2000, 64, 96, "bf16", guard=True)
    os.environ["MPK_TC_KIND"] = "1"
    fit(2000, 64, 96, "fp16")                    # streaming kernel (BN = 96)
    del os.environ["MPK_TC_KIND"]
    fit(1500, 24, 20, "fp16")                    # CUDA-core kernels (d_pad = d)
    fit(5000, 3, 5, "fp16", norm="minmax", iters=10)   # fused small-d iteration (K5g)
    X, _ = synth.blobs(6000, 16, 8, seed=2, dtype=np.float32)
    with mpk.KMeans(6000, 16, 12, "fp32", "fp16") as km:
        idx = km.seed(torch.from_numpy(X).cuda(), np.random.default_rng(1).random(12))
    print("seed", idx[:4], flush=True)
    # two virtual ranks (host threads, device-side reduction)
    grp = mpk.kmeans_vgroup_create(2)
    Xs = [torch.from_numpy(X[:3000]).cuda(), torch.from_numpy(X[3000:]).cuda()]
    C0 = torch.from_numpy(X[:12].copy()).cuda()
    hs = [mpk.kmeans_create_virtual(3000, 16, 12, "fp32", "fp16", 0, grp, r) for r in range(2)]
    th = [threading.Thread(target=mpk.kmeans_fit, args=(hs[r], Xs[r], C0, 3, -1.0))
          for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for h in hs:
        mpk.kmeans_destroy(h)
    mpk.kmeans_vgroup_destroy(grp)
    torch.cuda.synchronize()
    print("sanitize_run: done", flush=True)


if __name__ == "__main__":
    main()
