"""Pins for the oracle's Alg 4 / Alg 5 mode (O4m: the delta-triggered per-pair precision switch,
PAPER.md:613-645, 674-699). Each pin ties O4m to something other than its own formula: the two
limits that reduce it to other oracle routines, a column-by-column recomposition from those
routines, the exact scale invariance of the trigger, and the trigger-rate curve the paper states
for Fig 2."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def _data(n=600, d=8, k=12, seed=1, sigma=1.0):
    X, _ = synth.blobs(n, d, k, (-10.0, 10.0), sigma, seed=seed)
    Xn, _, _ = oracle.normalize(X, "zscore", "fp32")
    C = Xn[np.random.default_rng(seed + 7).choice(n, k, replace=False)].copy()
    return Xn, C


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
def test_delta_one_is_all_low_precision_with_scaling(dist):
    """delta = 1: eq:prec-delta always holds ("for delta = 1 the algorithm computes the distance
    fully in the low precision"): eta = 1 and the assignment equals the guarded
    (Alg 4 scaled) low-precision assignment."""
    X, C = _data()
    lab, dm, d2, nl = oracle.assign(X, C, "fp32", dist, delta=1.0, return_n_low=True)
    lab0, dm0, d20 = oracle.assign(X, C, "fp32", dist, guard=True)
    assert nl == X.shape[0] * C.shape[0]
    np.testing.assert_array_equal(lab, lab0)
    np.testing.assert_array_equal(dm, dm0)
    np.testing.assert_array_equal(d2, d20)


@pytest.mark.parametrize("work", ["fp32", "fp64"])
def test_huge_delta_is_working_precision(work):
    """delta -> inf: the condition never holds (eta = 0), every pair uses the working-precision
    formula (Alg 4 line 8), i.e. the assignment with dist = work."""
    X, C = _data()
    lab, dm, d2, nl = oracle.assign(X, C, work, "fp16", delta=1e150, return_n_low=True)
    lab0, dm0, d20 = oracle.assign(X, C, work, work)
    assert nl == 0
    np.testing.assert_array_equal(lab, lab0)
    np.testing.assert_array_equal(dm, dm0)


def test_mixed_assignment_recomposes_from_the_two_limits():
    """For a delta where both branches occur, each D_ij must be the low-precision value when
    eq:prec-delta holds for (x_i, c_j) and the working-precision value otherwise: rebuild the
    whole D matrix one centroid at a time from the two limit routines and the O2 norms, then
    check the mixed argmin, minimum and trigger count against it."""
    X, C = _data(n=300, d=6, k=9, sigma=2.0)
    Xr = X * np.linspace(0.2, 3.0, X.shape[0])[:, None]      # spread the norms: both branches
    Xr = oracle.round_to("fp32", Xr)
    delta = 1.3
    n, k = Xr.shape[0], C.shape[0]
    D_low, D_work = np.empty((n, k)), np.empty((n, k))
    for j in range(k):
        _, D_low[:, j], _ = oracle.assign(Xr, C[j:j + 1], "fp32", "fp16", guard=True)
        _, D_work[:, j], _ = oracle.assign(Xr, C[j:j + 1], "fp32", "fp32")
    _, xn, _ = oracle.prep(Xr, "fp32", "fp32")
    _, cn, _ = oracle.prep(C, "fp32", "fp32")
    hi = np.maximum(xn[:, None], cn[None, :])
    lo = np.minimum(xn[:, None], cn[None, :])
    trig = hi >= delta * delta * lo
    assert 0 < trig.sum() < n * k
    D = np.where(trig, D_low, D_work)
    lab, dm, _, nl = oracle.assign(Xr, C, "fp32", "fp16", delta=delta, return_n_low=True)
    assert nl == int(trig.sum())
    np.testing.assert_array_equal(lab, np.argmin(D, axis=1))
    np.testing.assert_array_equal(dm, D.min(axis=1))


def test_trigger_is_scale_invariant():
    """eq:prec-delta compares a ratio of squared norms, so scaling the data by a power of two
    (exact in floating point) leaves every decision unchanged (the curves on
    scaled and unscaled data coincide)."""
    X, C = _data(n=400, d=5, k=10, sigma=1.5)
    for delta in (1.2, 2.0, 5.0):
        a = oracle.assign(X, C, "fp32", "fp16", delta=delta, return_n_low=True)[3]
        b = oracle.assign(4.0 * X, 4.0 * C, "fp32", "fp16", delta=delta, return_n_low=True)[3]
        assert a == b


@pytest.mark.parametrize("sigma", [0.5, 1.0, 2.0])
def test_fig2_trigger_rate_curve(sigma):
    """Fig 2: 2,000 Gaussian points in 10 blobs (d = 2, reading Z24). The
    trigger rate eta is 1 at delta = 1, decreases with delta, and is close to 0 at delta = 80,
    on raw and on z-scored data alike."""
    X, _ = synth.blobs(2000, 2, 10, (-10.0, 10.0), sigma, seed=3)
    deltas = [1.0, 1.5, 2.0, 5.0, 10.0, 20.0, 40.0, 80.0]
    curves = []
    for norm in ("none", "zscore"):
        Xn, _, _ = oracle.normalize(X, norm, "fp32")
        C = Xn[:10].copy()
        eta = [oracle.assign(Xn, C, "fp32", "fp16", delta=dl, return_n_low=True)[3] / (2000 * 10)
               for dl in deltas]
        assert eta[0] == 1.0
        assert all(a >= b for a, b in zip(eta, eta[1:]))
        assert eta[-1] < 0.01
        curves.append(np.array(eta))
    # "almost identical" on normalised and non-normalised data
    assert np.max(np.abs(curves[0] - curves[1])) < 0.15


def test_fit_counts_triggered_pairs_over_iterations():
    """Alg 5: every iteration computes all n k distances; n_low sums the triggered ones, so
    eta_fit = n_low / (iters n k) lies in [0, 1], and delta = 1 gives exactly iters n k."""
    X, _ = synth.blobs(500, 4, 6, (-10.0, 10.0), 1.0, seed=5)
    C0 = X[:6].copy()
    r1 = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=4, tol=-1.0,
                    delta=1.0)
    assert r1["n_low"] == r1["iters"] * 500 * 6
    r2 = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=4, tol=-1.0,
                    delta=2.0)
    assert 0 <= r2["n_low"] <= r2["iters"] * 500 * 6
    r3 = oracle.fit(X, C0, work="fp32", dist="fp32", norm="zscore", max_iter=4, tol=-1.0)
    rh = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=4, tol=-1.0,
                    delta=1e150)
    assert rh["n_low"] == 0
    np.testing.assert_array_equal(rh["labels"], r3["labels"])
    np.testing.assert_array_equal(rh["centroids"], r3["centroids"])


def test_delta_below_one_is_rejected():
    X, C = _data(n=50, d=3, k=4)
    with pytest.raises(ValueError):
        oracle.assign(X, C, "fp32", "fp16", delta=0.5)
