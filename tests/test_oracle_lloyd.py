"""Pins for oracle O1..O9 against things other than the oracle itself: SPEC/paper worked
examples (tests/golden/spec_examples.json), closed forms, exact rational arithmetic, the
paper's error bounds (Thm 5.2, Thm 6.1, Lemma 5.2), Lemma 4.1, Lloyd's monotonicity,
brute-force optimal partitions and sklearn's Lloyd. SURVEY.md §8c.3."""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
U = {"fp64": 2.0 ** -53, "fp32": 2.0 ** -24, "fp16": 2.0 ** -11, "bf16": 2.0 ** -8,
     "e5m2": 2.0 ** -3}


def gamma(m, u):
    return m * u / (1 - m * u)


# ------------------------------------------------------------------ SPEC / paper examples
def test_spec_assign_examples():
    for key in ("assign_1d", "assign_equidistant"):
        g = G[key]
        lab, _, _ = oracle.assign(g["X"], g["C"], work="fp64", dist="fp64")
        assert lab.tolist() == g["labels"], g["_cite"]
        lab16, _, _ = oracle.assign(g["X"], g["C"], work="fp32", dist="fp16")
        assert lab16.tolist() == g["labels"]


def test_spec_update_and_sse_examples():
    g = G["update_mean"]
    st = oracle.step(g["X"], [[5.0, 5.0]], work="fp64", dist="fp64")
    assert st["centroids"][0].tolist() == g["center"], g["_cite"]
    g = G["sse"]
    _, sse = oracle.final(g["X"], g["C"], work="fp64")
    assert sse == g["sse"], g["_cite"]


def test_spec_lemma41_example():
    g = G["lemma41"]
    X = np.array(g["X"])
    _, phi_p = oracle.final(X, [g["p"]], work="fp64")
    _, phi_mu = oracle.final(X, [X.mean(0)], work="fp64")
    assert phi_p == g["phi_p"] and phi_mu == g["phi_mu"]
    assert phi_p == phi_mu + g["S"] * g["dist2"], g["_cite"]


def test_spec_zscore_examples():
    g = G["zscore_2pt"]
    Z, mu, sd = oracle.normalize(g["X"], "zscore")
    assert Z.tolist() == g["Z"], g["_cite"]
    g = G["zscore_4pt"]
    Z, mu, sd = oracle.normalize(g["X"], "zscore")
    assert mu[0] == g["mu"] and abs(sd[0] ** 2 - g["sigma2"]) < 1e-15
    want = (np.array(g["X"]) - 2.5) / np.sqrt(1.25)
    assert np.allclose(Z, want, rtol=0, atol=1e-15)


# ------------------------------------------------------------------ O1 normalisation
def test_zscore_moments_and_constant_feature():
    rng = np.random.default_rng(0)
    X = rng.normal(3.0, 7.0, (5000, 4))
    X[:, 2] = 4.25   # zero variance -> scale 1 (reading Z17)
    Z, mu, sd = oracle.normalize(X, "zscore")
    assert np.all(np.abs(Z[:, [0, 1, 3]].mean(0)) <= 1e-10)
    assert np.all(np.abs(Z[:, [0, 1, 3]].std(0) - 1) <= 1e-10)
    assert sd[2] == 1.0 and np.all(Z[:, 2] == 0.0)


def test_minmax_equals_div255_on_image():
    """channels divided by 255; the generator forces a 0..255 span."""
    X, _ = synth.image(dtype=np.float32)
    Z, mn, rg = oracle.normalize(X.astype(np.float64), "minmax", work="fp32")
    assert np.all(mn == 0.0) and np.all(rg == 255.0)
    want = (X.astype(np.float64) / 255.0).astype(np.float32).astype(np.float64)
    assert np.array_equal(Z, want)


# ------------------------------------------------------------------ O2/O4 distances
def _exact_sq(x, c):
    return sum((Fraction(a) - Fraction(b)) ** 2 for a, b in zip(x, c))


@pytest.mark.parametrize("d", [2, 10, 100])
def test_thm52_expanded_fp64_bound(d):
    """Thm 5.2: |D^ - D| <= gamma_{d+2} (x'x + 2|x|'|c| + c'c), fp64."""
    rng = np.random.default_rng(d)
    X = rng.standard_normal((60, d)) * rng.uniform(0.1, 10, (60, 1))
    c = rng.standard_normal((1, d)) * 3
    _, dmin, _ = oracle.assign(X, c, work="fp64", dist="fp64")
    for i in range(len(X)):
        exact = _exact_sq(X[i], c[0])
        bound = gamma(d + 2, U["fp64"]) * (X[i] @ X[i] + 2 * np.abs(X[i]) @ np.abs(c[0])
                                           + c[0] @ c[0])
        assert abs(Fraction(dmin[i]) - exact) <= Fraction(bound)


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2", "fp32"])
@pytest.mark.parametrize("d", [2, 10, 100])
def test_thm61_mixed_bound(dist, d):
    """Thm 6.1: |D^ - D| <~ (d+2)u(x'x + c'c) + 2(d+2)u_l |x|'|c|, plus an
    underflow allowance d * 2^(e_min - t + 1) |x|'... for subnormal operands (reading Z8)."""
    rng = np.random.default_rng(100 + d)
    X = rng.standard_normal((80, d))
    c = rng.standard_normal((1, d))
    _, dmin, _ = oracle.assign(X, c, work="fp64", dist=dist)
    t, emin, _ = oracle.format_params(dist)
    ul = U[dist]
    for i in range(len(X)):
        exact = float(_exact_sq(X[i], c[0]))
        ax, ac = np.abs(X[i]), np.abs(c[0])
        bound = ((d + 2) * U["fp64"] * (X[i] @ X[i] + c[0] @ c[0])
                 + 2 * (d + 2) * ul * (ax @ ac)
                 + 2 * d * 2.0 ** (emin - t + 1) * (ax.sum() + ac.sum() + 1))
        assert abs(dmin[i] - exact) <= bound


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
def test_low_precision_distance_is_exact_formula_on_rounded_operands(dist):
    """O2/O4 pinned by a library cast + exact rationals: D^ equals x'x - 2 x~'c~ + c'c with
    x~ = torch/numpy single rounding of x, up to fp64 accumulation (gamma_d in fp64)."""
    import torch
    tdt = {"fp16": torch.float16, "bf16": torch.bfloat16, "e5m2": torch.float8_e5m2}[dist]
    rng = np.random.default_rng(7)
    d = 17
    X = rng.standard_normal((40, d)).astype(np.float32)
    C = rng.standard_normal((3, d)).astype(np.float32)
    lab, dmin, d2 = oracle.assign(X, C, work="fp32", dist=dist)
    xl = torch.from_numpy(X).to(tdt).double().numpy()
    cl = torch.from_numpy(C).to(tdt).double().numpy()
    for i in range(len(X)):
        xn = float(np.float32(sum(Fraction(float(v)) ** 2 for v in X[i])))
        Ds = []
        for j in range(3):
            cn = float(np.float32(sum(Fraction(float(v)) ** 2 for v in C[j])))
            dot = sum(Fraction(a) * Fraction(b) for a, b in zip(xl[i], cl[j]))
            Ds.append(Fraction(xn) - 2 * dot + Fraction(cn))
        tolr = 4 * d * U["fp64"] * (abs(xn) + 2 * float(np.abs(xl[i]) @ np.abs(cl).max(0)) + 50)
        best = min(range(3), key=lambda j: (Ds[j], j))
        assert abs(float(Ds[best]) - dmin[i]) <= tolr
        srt = sorted(Ds)
        if float(srt[1] - srt[0]) > 2 * tolr:
            assert lab[i] == best


def test_guard_power_of_two_invariance():
    """Alg 4 scaling: operands x/||x||_inf are invariant under x -> 2^e x,
    norms scale by 2^2e (metamorphic pin 1)."""
    rng = np.random.default_rng(11)
    X = (rng.standard_normal((500, 9)) * 1e3).astype(np.float32).astype(np.float64)
    a = oracle.prep(X, work="fp32", dist="fp16", guard=True)
    b = oracle.prep(X * 2.0 ** 7, work="fp32", dist="fp16", guard=True)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1] * 2.0 ** 14, b[1])
    assert np.array_equal(a[2] * 2.0 ** 7, b[2])
    assert np.all(np.abs(a[0]) <= 1.0)


def test_unguarded_overflow_and_guard_fix():
    """Non-normalised large data overflows fp16/E5M2 operands;
    Alg 4 scaling removes it. Qualitative Table 3 pattern: collapse without the guard."""
    from sklearn.metrics import adjusted_rand_score as ari
    X, y = synth.blobs(3000, 32, 8, (-1e5, 1e5), 1e4, seed=3, dtype=np.float32)
    C0 = synth.init_rows(X, 8, 3)
    xl, _, _ = oracle.prep(X, work="fp32", dist="e5m2", guard=False)
    assert np.isinf(xl).mean() > 0.2
    ref = oracle.fit(X, C0, work="fp32", dist="fp32", max_iter=50)
    for dist in ("e5m2", "fp16"):
        bad = oracle.fit(X, C0, work="fp32", dist=dist, max_iter=50)
        good = oracle.fit(X, C0, work="fp32", dist=dist, guard=True, max_iter=50)
        assert ari(ref["labels"], good["labels"]) > 0.95
        assert abs(good["sse"] / ref["sse"] - 1) < 1e-2
        assert ari(ref["labels"], bad["labels"]) < 0.7       # degraded clustering ...
        assert bad["sse"] > 1.5 * ref["sse"]                 # ... with much larger SSE
        assert bad["empty_t"][-1] > 0                        # overflowed rows pile up


# ------------------------------------------------------------------ O7 update
def test_step_update_matches_groupby_and_lemma52():
    """eq:center: sums/counts equal an independent groupby; the fp32 means obey
    Lemma 5.2: |mu^ - mu| <= gamma_m |mu| elementwise (here: one
    rounding, <= u |mu|)."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((4000, 6)).astype(np.float32).astype(np.float64)
    C = X[:7].copy()
    st = oracle.step(X, C, work="fp32", dist="fp16")
    lab = st["labels"]
    assert np.array_equal(st["counts"], np.bincount(lab, minlength=7))
    ref = np.zeros((7, 6))
    np.add.at(ref, lab, X)
    assert np.allclose(st["sums"], ref, rtol=1e-13, atol=1e-12)
    for j in range(7):
        exact = [sum(Fraction(v) for v in X[lab == j, t]) / int((lab == j).sum())
                 for t in range(6)]
        mu = st["centroids"][j]
        for t in range(6):
            assert abs(Fraction(mu[t]) - exact[t]) <= Fraction(U["fp32"]) * abs(exact[t])
    # step labels = assign labels (same definition)
    lab2, _, _ = oracle.assign(X, C, work="fp32", dist="fp16")
    assert np.array_equal(lab, lab2)


def test_empty_cluster_keeps_centroid():
    X = np.array([[0.0], [1.0], [2.0]])
    C = np.array([[0.5], [100.0]])
    st = oracle.step(X, C, work="fp64", dist="fp64")
    assert st["counts"].tolist() == [3, 0]
    assert st["centroids"][1, 0] == 100.0 and st["centroids"][0, 0] == 1.0


# ------------------------------------------------------------------ Lloyd loop
def test_k1_mean_and_sse_closed_form():
    rng = np.random.default_rng(9)
    X = rng.standard_normal((3000, 5)) * 4 + 2
    r = oracle.fit(X, X[:1], max_iter=5)
    mu = X.mean(0)
    assert np.allclose(r["centroids"][0], mu, rtol=1e-13, atol=1e-13)
    want = float(np.sum((X - mu) ** 2))
    assert abs(r["sse"] - want) <= 1e-12 * want


@pytest.mark.parametrize("work,dist", [("fp64", "fp64"), ("fp32", "fp16"), ("fp32", "e5m2")])
def test_iteration_sse_k1_closed_form(work, dist):
    """O6 (SSE_t = sum_i max(0, min_j D^_ij), eq:sse PAPER.md:130-133) pinned by value with
    k = 1: from C0 = x_0, SSE_1 = sum_i ||x_i - x_0||^2 and then SSE_2 = sum_i ||x_i - mu||^2
    (mu the mean, eq:center). The data are small integers (exact in fp16 and E5M2, every
    product and sum exact), so the expanded formula of O4 equals the direct one exactly and
    SSE_1 is an exact integer. A dropped ||x||^2 or ||c||^2 term, a wrong sign of the cross
    term or a missing clamp changes SSE_1."""
    rng = np.random.default_rng(21)
    X = rng.integers(-3, 4, size=(64, 5)).astype(np.float64)
    X[0] = [1, -2, 0, 3, -1]
    # column sums divisible by 64 make mu an exact dyadic value
    X[-1] -= X.sum(0) - 64 * np.round(X.sum(0) / 64)
    X[-1] = np.clip(X[-1], -3, 3)
    r = oracle.fit(X, X[:1], work=work, dist=dist, max_iter=2, tol=-1.0)
    exact1 = sum(sum((Fraction(a) - Fraction(b)) ** 2 for a, b in zip(x, X[0])) for x in X)
    assert r["sse_t"][0] == float(exact1)
    mu = [sum(Fraction(v) for v in X[:, t]) / len(X) for t in range(X.shape[1])]
    exact2 = sum(sum((Fraction(a) - m) ** 2 for a, m in zip(x, mu)) for x in X)
    # the centroid is mu rounded to the working precision; SSE_2 from the low-precision
    # operand c~ = round_l(mu): bound the effect of both roundings on the sum
    u = U[dist]
    slack = 4 * u * float(sum(sum(abs(Fraction(a)) + abs(m) for a, m in zip(x, mu)) for x in X)) \
        * max(1.0, float(max(abs(m) for m in mu)))
    assert abs(r["sse_t"][1] - float(exact2)) <= slack + 1e-12 * float(exact2)
    if dist == "fp64":
        assert abs(r["sse_t"][1] - float(exact2)) <= 1e-12 * float(exact2)
    assert r["changed_t"].tolist() == [64, 0]


def test_guard_scale_by_value():
    """Alg 4 lines 1-5: s = ||x||_inf and x~ = round_l(x / s). Pinned by
    value: (3, -4, 1) -> s = 4, x~ = (0.75, -1, 0.25); (3, 1, -2) -> s = 3 (not the 2-norm
    sqrt(14), not a power of two), x~ = fp16(1, 1/3, -2/3); a zero row -> s = 1 (Z10). Norms are
    the unscaled ||x||^2."""
    X = np.array([[3.0, -4.0, 1.0], [3.0, 1.0, -2.0], [0.0, 0.0, 0.0], [-0.5, 0.25, 0.125]])
    xl, nrm, sc = oracle.prep(X, work="fp32", dist="fp16", guard=True)
    assert sc.tolist() == [4.0, 3.0, 1.0, 0.5]
    assert nrm.tolist() == [26.0, 14.0, 0.0, 0.328125]
    want = np.array([[0.75, -1.0, 0.25],
                     [1.0, float(np.float16(1.0 / 3.0)), float(np.float16(-2.0 / 3.0))],
                     [0.0, 0.0, 0.0], [-1.0, 0.5, 0.25]])
    assert np.array_equal(xl, want)
    # unguarded: s = 1, x~ = round_l(x)
    xl0, _, sc0 = oracle.prep(X, work="fp32", dist="e5m2", guard=False)
    assert sc0.tolist() == [1.0] * 4
    assert np.array_equal(xl0, X)   # every value is exact in E5M2


def test_k_equals_n_zero_sse():
    rng = np.random.default_rng(10)
    X = rng.standard_normal((50, 3))
    r = oracle.fit(X, X, max_iter=3)
    assert r["sse"] == 0.0 and np.array_equal(r["labels"], np.arange(50))


def _best_partition(X, k):
    best = (np.inf, None)
    n = len(X)
    for lab in itertools.product(range(k), repeat=n):
        lab = np.array(lab)
        if len(np.unique(lab)) < k:
            continue
        s = 0.0
        for j in range(k):
            P = X[lab == j]
            s += float(np.sum((P - P.mean(0)) ** 2))
        if s < best[0] - 1e-12:
            best = (s, lab)
    return best


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bruteforce_optimal_partition(seed):
    """n=9, k=3: Lloyd's SSE >= the optimum; started from the optimal partition's means it
    returns that partition with SSE equal to the optimum (SURVEY §8c.3 brute force)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((9, 2)) * 3
    opt, lab = _best_partition(X, 3)
    r = oracle.fit(X, X[[0, 4, 8]], max_iter=100)
    assert r["sse"] >= opt * (1 - 1e-12)
    C = np.stack([X[lab == j].mean(0) for j in range(3)])
    r2 = oracle.fit(X, C, max_iter=100)
    assert np.array_equal(r2["labels"], lab)
    assert abs(r2["sse"] - opt) <= 1e-12 * opt


def test_sse_monotone_and_fixed_point():
    """Lloyd's local-improvement property: SSE_t non-increasing up
    to the Thm 5.2 rounding slack; the returned centroids are a fixed point."""
    X, _ = synth.blobs(4000, 4, 6, sigma=2.5, seed=4, dtype=np.float64)
    C0 = synth.init_rows(X, 6, 4)
    r = oracle.fit(X, C0, max_iter=200, tol=0.0)
    s = r["sse_t"]
    xn = np.sum(X * X, 1)
    slack = gamma(6, U["fp64"]) * float(np.sum(xn + 2 * np.sqrt(xn) * 20 + 400))
    assert np.all(np.diff(s) <= slack)
    assert r["changed_t"][-1] == 0
    st = oracle.step(X, r["centroids"], work="fp64", dist="fp64")
    assert np.array_equal(st["labels"], r["labels"])
    assert np.array_equal(st["centroids"], r["centroids"])


def test_matches_sklearn_lloyd():
    """fp64 working mode vs sklearn.cluster.KMeans(lloyd, init=C0, n_init=1) on well-separated
    blobs without empty clusters; sklearn is the library the paper cites."""
    from sklearn.cluster import KMeans
    X, _ = synth.blobs(5000, 3, 5, sigma=1.0, seed=12, dtype=np.float64)
    C0 = synth.init_rows(X, 5, 12)
    r = oracle.fit(X, C0, max_iter=300, tol=0.0)
    km = KMeans(5, init=C0, n_init=1, algorithm="lloyd", tol=0.0, max_iter=300).fit(X)
    assert np.mean(km.labels_ == r["labels"]) >= 0.999
    assert abs(km.inertia_ - r["sse"]) <= 1e-9 * r["sse"]


def test_fp16_normalised_quality_close_to_fp64():
    """Normalised data tolerates fp16 distances (Table 3 normalised S1
    1.547e2 vs 1.546e2): SSE within 1e-2 relative of the fp64 run, ARI > 0.95."""
    from sklearn.metrics import adjusted_rand_score as ari
    X, _ = synth.blobs(6000, 8, 10, sigma=1.5, seed=13, dtype=np.float32)
    C0 = synth.init_rows(X, 10, 13)
    a = oracle.fit(X, C0, work="fp32", dist="fp32", norm="zscore", max_iter=100)
    b = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=100)
    assert abs(a["sse"] - b["sse"]) <= 1e-2 * a["sse"]
    assert ari(a["labels"], b["labels"]) > 0.95


def test_iteration_counting_and_tol():
    """Reading Z22: a fixed-point C0 stops after one iteration; tol < 0 runs max_iter."""
    X = np.array([[0.0], [1.0], [10.0], [11.0]])
    r = oracle.fit(X, [[0.5], [10.5]], max_iter=10, tol=0.0)
    assert r["iters"] == 1 and r["changed_t"].tolist() == [4]      # shift 0 <= tol
    r = oracle.fit(X, [[0.0], [11.0]], max_iter=10, tol=0.0)
    assert r["iters"] == 2 and r["changed_t"].tolist() == [4, 0]   # no label changed
    r = oracle.fit(X, [[0.5], [10.5]], max_iter=7, tol=-1.0)
    assert r["iters"] == 7


def test_guard_pow2_reading_b():
    """Reading Z9 B (KMEANS_GUARD_POW2): s = 2^ceil(log2 ||x||_inf) — a power of two in
    [||x||_inf, 2 ||x||_inf) — so x / s is exact and x~ = round_l(x / s). Pins: (1) the scale by
    value; (2) where every infinity norm is a power of two, B equals A bit for bit; (3) scaling
    by a power of two commutes with rounding, so away from the format's subnormal and overflow
    ranges the significands of x~ are those of round_l(x): B changes nothing but the exponent
    range (the MX block scale's only effect)."""
    X = np.array([[3.0, -4.0, 1.0], [0.75, 0.5, -0.25], [0.0, 0.0, 0.0], [5.0, 1.0, 1.0]])
    xl, nrm, sc = oracle.prep(X, work="fp32", dist="fp16", guard="pow2")
    assert sc.tolist() == [4.0, 1.0, 1.0, 8.0]
    assert np.array_equal(xl[0], [0.75, -1.0, 0.25])
    assert np.array_equal(xl[3], [0.625, 0.125, 0.125])
    rng = np.random.default_rng(31)
    P = rng.standard_normal((300, 9))
    P[:, 0] = np.sign(P[:, 0]) * 2.0 ** rng.integers(1, 6, 300)   # the max is a power of 2
    P[:, 1:] = np.clip(P[:, 1:], -1.9, 1.9)
    a = oracle.prep(P, work="fp64", dist="e5m2", guard=True)
    b = oracle.prep(P, work="fp64", dist="e5m2", guard="pow2")
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    Q = rng.uniform(0.05, 1.0, (400, 3)) * rng.choice([-1, 1], (400, 3))
    ql, _, _ = oracle.prep(Q, work="fp64", dist="e5m2", guard=False)
    pl, _, ps = oracle.prep(Q, work="fp64", dist="e5m2", guard="pow2")
    assert np.all(np.log2(ps) == np.round(np.log2(ps)))
    np.testing.assert_array_equal(pl * ps[:, None], ql)
