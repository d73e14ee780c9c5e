"""Parity at the size the bench runs (BASELINE.json configs[4], C5: n = 10M, d = 128, k = 1024):
a teacher-forced check along the real 10M-row fit.

For t = 0..4, C_t are the centres after t Lloyd iterations of the GPU fit (C_0 = C0). Then
  * iteration t+1's assignment (Alg 3 step 3) is kmeans_assign(X, C_t) on all
    10M rows; a seeded 200k-row sample is compared with the oracle's assignment of the same rows
    from the same C_t, label by label (admissible under 2 B_acc);
  * C_{t+1} returned by fit(max_iter = t+1) must be eq:center (Alg 3 step 4)
    on those labels: the mean of the rows labelled j (an fp64 sum over all 10M rows, formed here
    on the GPU with torch as the test's own arithmetic), rounded to fp32; empty clusters keep
    c_j.
Finally the final pass (Alg 3 step 7) after 5 iterations: sampled labels against
the oracle's working-precision assignment (within the fp32 evaluation error) and the reported
SSE against the direct formula (eq:dist-eval-alternative) over all rows.

The input is the C5 generator's blobs z-scored by the test (fp64 statistics, one rounding to
fp32) and passed with NORM_NONE, so the oracle sees exactly the rows the kernels see; the
normalisation step itself is pinned by the C2/C3-size tests."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._parity import check_admissible_rows, dev

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
mpk = pytest.importorskip("paper_2407_12208_b200")

T_MAX = 5
SAMPLE = 200_000


@pytest.fixture(scope="module")
def c5_data():
    X, _, C0 = synth.make("c5_vq_10m", seed=0)
    n, d = X.shape
    Xd = torch.from_numpy(X).cuda()
    s1 = torch.zeros(d, dtype=torch.float64, device="cuda")
    for r in range(0, n, 1 << 21):
        s1 += Xd[r:r + (1 << 21)].double().sum(0)
    mu = s1 / n
    s2 = torch.zeros(d, dtype=torch.float64, device="cuda")
    for r in range(0, n, 1 << 21):
        s2 += ((Xd[r:r + (1 << 21)].double() - mu) ** 2).sum(0)
    sd = torch.sqrt(s2 / n)
    for r in range(0, n, 1 << 21):
        Xd[r:r + (1 << 21)] = ((Xd[r:r + (1 << 21)].double() - mu) / sd).float()
    C0n = ((torch.from_numpy(C0).cuda().double() - mu) / sd).float()
    del X
    rng = np.random.default_rng(2024)
    S = np.sort(rng.choice(n, SAMPLE, replace=False))
    Xs = Xd[torch.from_numpy(S).cuda()].cpu().numpy()
    return Xd, C0n, S, Xs


def _means(Xd, lab, k, Cprev):
    d = Xd.shape[1]
    sums = torch.zeros((k, d), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(k, dtype=torch.float64, device="cuda")
    n = Xd.shape[0]
    for r in range(0, n, 1 << 21):
        li = lab[r:r + (1 << 21)].long()
        sums.index_add_(0, li, Xd[r:r + (1 << 21)].double())
        cnt.index_add_(0, li, torch.ones_like(li, dtype=torch.float64))
    want = torch.where(cnt[:, None] > 0, sums / cnt.clamp(min=1)[:, None], Cprev.double())
    return want.float().double().cpu().numpy(), cnt.cpu().numpy()


@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
def test_c5_teacher_forced_along_the_fit(c5_data, dist):
    Xd, C0n, S, Xs = c5_data
    n, d = Xd.shape
    k = C0n.shape[0]
    km = mpk.KMeans(n, d, k, "fp32", dist)
    cents = [C0n.clone()]
    for t in range(1, T_MAX + 1):
        c = torch.empty((k, d), dtype=torch.float32, device="cuda")
        rc, sse, it = km.fit(Xd, C0n, max_iter=t, tol=-1.0, centroids=c)
        assert it == t and km.stats()["tc_variant"] == 2
        cents.append(c)
    final_lab = torch.empty(n, dtype=torch.int32, device="cuda")
    rc, sse_final, _ = km.fit(Xd, C0n, max_iter=T_MAX, tol=-1.0, labels=final_lab)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    for t in range(T_MAX):
        Ct = cents[t]
        mpk.kmeans_set_centroids(km.h, Ct)
        km.assign(Xd, lab)
        # (1) the assignment on the sample vs the oracle, same operands
        Cn = Ct.cpu().numpy()
        ref, _, _ = oracle.assign(Xs, Cn, work="fp32", dist=dist, guard=False)
        g = lab.cpu().numpy()[S]
        frac = check_admissible_rows(Xs, Cn, g, ref, "fp32", dist, False)
        assert frac <= 1e-3, (t, frac)
        # (2) the update of iteration t+1 on the GPU's labels of all 10M rows
        want, cnt = _means(Xd, lab, k, Ct)
        got = cents[t + 1].cpu().numpy().astype(np.float64)
        tol = (np.maximum(cnt, 1)[:, None] * 2.0 ** -52 + 4 * 2.0 ** -24) * np.abs(want) + 1e-30
        bad = np.abs(got - want) > tol
        assert not bad.any(), (t, np.abs(got - want).max(), int(bad.sum()))
    km.close()
    # (3) the final working-precision pass with C_5 on the sample, and the direct-formula SSE
    C5 = cents[T_MAX].cpu().numpy().astype(np.float64)
    want, _ = oracle.final(Xs, C5, work="fp32")
    gl = final_lab.cpu().numpy()
    g = gl[S]
    diff = np.nonzero(g != want)[0]
    if diff.size:
        x = Xs[diff].astype(np.float64)
        D = (x * x).sum(1)[:, None] - 2 * x @ C5.T + (C5 * C5).sum(1)[None, :]
        xn = (x * x).sum(1)
        cmax = (C5 * C5).sum(1).max()
        tol = 2 * (d + 2) * 2.0 ** -24 * (xn + 2 * np.sqrt(xn * cmax) + cmax)
        gap = D[np.arange(diff.size), g[diff]] - D[np.arange(diff.size), want[diff]]
        assert np.all(gap <= tol), gap.max()
    assert diff.size <= 1e-3 * SAMPLE
    Ct = torch.from_numpy(C5).cuda()
    direct = 0.0
    for r in range(0, n, 1 << 21):
        xr = Xd[r:r + (1 << 21)].double()
        direct += float(((xr - Ct[final_lab[r:r + (1 << 21)].long()]) ** 2).sum())
    assert abs(sse_final - direct) <= 1e-9 * direct
