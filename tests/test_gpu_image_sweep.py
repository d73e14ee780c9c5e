"""NEXT #3: image segmentation of a synthetic RGB image (config C2, /255)
with Alg 1 seeding + Alg 3 (all distances in u_l) or Alg 5 (delta = 2). The paper reports that
fp16 stays close to the working-precision SSE, that q52 (E5M2) degrades badly, and that the
mixed scheme suffers less from the lower precision. Those qualitative statements are checked
here; the paper's cause (underflow under every-operation q52 rounding) does not arise with exact
products and fp32 accumulation (readings Z2/Z3), which the census confirms."""
import numpy as np
import pytest
import torch

import paper_2407_12208_b200 as mpk
import synth

pytestmark = pytest.mark.gpu


def _fit(X, k, dist, delta, u):
    n, d = X.shape
    km = mpk.KMeans(n, d, k, "fp32", dist, norm="minmax", delta=delta)
    idx = km.seed(X, u)
    C0 = X[torch.from_numpy(idx).cuda()].contiguous()
    rc, sse, it = km.fit(X, C0, max_iter=100, tol=1e-4)
    st = km.stats()
    km.close()
    return sse, st


@pytest.mark.parametrize("k", [5, 20])
def test_image_sweep_qualitative(k):
    cfg = synth.CONFIGS["c2_image_512"]
    X, _, _ = synth.make(cfg, n=cfg.n, seed=0)
    Xd = torch.from_numpy(X).cuda()
    u = np.random.default_rng(100 + k).random(k)
    base, _ = _fit(Xd, k, "fp32", None, u)
    mp16, st16 = _fit(Xd, k, "fp16", 2.0, u)
    low8, st8 = _fit(Xd, k, "e5m2", None, u)
    mp8, stm8 = _fit(Xd, k, "e5m2", 2.0, u)
    assert abs(mp16 / base - 1.0) <= 0.05          # fp16: close to the working precision
    assert low8 / base >= 1.5                       # q52 everywhere: significant degradation
    assert mp8 < low8                               # the mixed scheme suffers less
    assert 0.0 < stm8["eta"] < 0.5
    assert st8["n_underflow"] == 0 and st16["n_underflow"] == 0


def test_mx_pow2_scaling_is_a_no_op_on_the_image():
    """NEXT #3's proposed remedy, MX block scaling (a power-of-two scale per block; with d = 3
    the row is the block): KMEANS_GUARD_POW2 divides every pixel by 2^ceil(log2 ||x||_inf), which
    is exact and commutes with rounding to E5M2 as long as nothing under- or overflows — here
    nothing does (census 0), so the scaled fit gives the unscaled fit's labels bit for bit (and
    its SSE): the q52 degradation on images is the 3-bit significand, not range (DESIGN.md NEXT #3)."""
    cfg = synth.CONFIGS["c2_image_512"]
    X, _, _ = synth.make(cfg, n=cfg.n, seed=0)
    Xd = torch.from_numpy(X).cuda()
    n, d = X.shape
    out = []
    for guard in (False, "pow2"):
        km = mpk.KMeans(n, d, 20, "fp32", "e5m2", norm="minmax", guard=guard)
        C0 = Xd[torch.from_numpy(np.arange(0, n, n // 20)[:20]).cuda()].contiguous()
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        rc, sse, it = km.fit(Xd, C0, max_iter=30, tol=-1.0, labels=lab)
        st = km.stats()
        km.close()
        out.append((lab.cpu().numpy(), sse, st))
    assert out[0][2]["n_underflow"] == 0 and out[1][2]["n_underflow"] == 0
    np.testing.assert_array_equal(out[0][0], out[1][0])
    # the final SSE is an fp64 sum whose order may differ between runs: to rounding
    assert abs(out[0][1] - out[1][1]) <= 1e-12 * out[0][1]
