"""GPU parity of Alg 4 / Alg 5's per-pair precision switch (kmeans_set_delta, K6m) against the
oracle's O4m (tests/test_oracle_mixed.py pins it): exact trigger counts, admissible labels under
the per-pair error bounds, and the two limits (delta = 1: the scaled low-precision CUDA-core
kernel; delta -> inf: the working-precision kernel) bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import paper_2407_12208_b200 as mpk
import synth
from tests._parity import check_labels_admissible, dev, distances_on_rounded_operands

pytestmark = pytest.mark.gpu

NP = {"fp32": np.float32, "fp64": np.float64}


def _spread(n, d, k, work, seed=2):
    """z-scored blobs with rows rescaled over [0.15, 3]: pairs on both sides of eq:prec-delta."""
    X, _ = synth.blobs(n, d, 8, sigma=2.0, seed=seed, dtype=NP[work])
    Xn, _, _ = oracle.normalize(X, "zscore", work=work)
    Xn = Xn * np.linspace(0.15, 3.0, n)[np.random.default_rng(seed).permutation(n)][:, None]
    Xn = oracle.round_to(work, Xn).astype(NP[work])
    C = synth.init_rows(Xn, k, seed)
    return Xn, C


def _gpu_assign(Xn, C, work, dist, delta=None, guard=False, force_simt=False):
    n, d = Xn.shape
    k = C.shape[0]
    km = mpk.KMeans(n, d, k, work, dist, guard=guard, force_simt=force_simt, delta=delta)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    mpk.kmeans_set_centroids(km.h, dev(C))
    km.assign(dev(Xn), lab)
    st = km.stats()
    km.close()
    return lab.cpu().numpy(), st


def _mixed_reference(Xn, C, work, dist, delta):
    D_low, B_low = distances_on_rounded_operands(Xn, C, work, dist, True)
    D_w, B_w = distances_on_rounded_operands(Xn, C, work, work, False)
    _, xn, _ = oracle.prep(Xn, work, work)
    _, cn, _ = oracle.prep(C, work, work)
    hi = np.maximum(xn[:, None], cn[None, :])
    lo = np.minimum(xn[:, None], cn[None, :])
    trig = hi >= delta * delta * lo
    return np.where(trig, D_low, D_w), np.where(trig, B_low, B_w), int(trig.sum())


@pytest.mark.parametrize("work,dist", [("fp32", "fp16"), ("fp32", "bf16"), ("fp32", "e5m2"),
                                       ("fp64", "fp16"), ("fp64", "fp32")])
@pytest.mark.parametrize("delta", [1.3, 2.0])
def test_mixed_assign_parity(work, dist, delta):
    n, d, k = 3001, 19, 23                        # ragged against the 64 x 64 x 16 tiles
    Xn, C = _spread(n, d, k, work)
    lab, st = _gpu_assign(Xn, C, work, dist, delta=delta)
    ref_lab, _, _, ref_low = oracle.assign(Xn, C, work, dist, delta=delta, return_n_low=True)
    D, B, n_trig = _mixed_reference(Xn, C, work, dist, delta)
    assert n_trig == ref_low
    assert 0 < ref_low < n * k                    # both branches exercised
    assert st["n_dist"] == n * k
    assert st["n_dist_low"] == ref_low            # the trigger decisions, bit-exact
    frac = check_labels_admissible(lab, ref_lab, D, B)
    assert frac <= 2e-3


@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
def test_delta_one_equals_scaled_low_precision_kernel(dist):
    """delta = 1 triggers every pair: the same labels as the guarded CUDA-core kernel (K6)."""
    Xn, C = _spread(2000, 17, 21, "fp32")
    lab, st = _gpu_assign(Xn, C, "fp32", dist, delta=1.0)
    lab0, _ = _gpu_assign(Xn, C, "fp32", dist, guard=True, force_simt=True)
    assert st["n_dist_low"] == st["n_dist"] == 2000 * 21
    np.testing.assert_array_equal(lab, lab0)


def test_huge_delta_equals_working_precision_kernel():
    """delta -> inf triggers nothing: the same labels as the fp32 working-mode kernel."""
    Xn, C = _spread(2000, 17, 21, "fp32")
    lab, st = _gpu_assign(Xn, C, "fp32", "fp16", delta=1e30)
    lab0, _ = _gpu_assign(Xn, C, "fp32", "fp32")
    assert st["n_dist_low"] == 0
    np.testing.assert_array_equal(lab, lab0)


def test_mixed_fit_matches_oracle():
    """Alg 5 end to end (Alg 3 steps 2-7 with Alg 4 in the loop): SSE and eta against the
    oracle's fit; the normalisation statistics may differ in the last bits, so eta is compared
    within a small tolerance."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=20011, seed=4)
    C0 = C0[:48].copy()
    ref = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=6, tol=-1.0,
                     delta=1.05)
    km = mpk.KMeans(len(X), 64, 48, "fp32", "fp16", norm="zscore", delta=1.05)
    lab = torch.empty(len(X), dtype=torch.int32, device="cuda")
    rc, sse, it = km.fit(dev(X), dev(C0), max_iter=6, tol=-1.0, labels=lab)
    st = km.stats()
    km.close()
    assert it == ref["iters"] == 6
    eta_ref = ref["n_low"] / (6 * len(X) * 48)
    assert 0.0 < eta_ref < 1.0
    assert abs(st["eta"] - eta_ref) <= 1e-3
    assert abs(sse - ref["sse"]) <= 1e-3 * ref["sse"]


def test_set_delta_rejects_values_below_one():
    km = mpk.KMeans(100, 4, 3, "fp32", "fp16")
    with pytest.raises(mpk.KMeansError):
        mpk.kmeans_set_delta(km.h, 0.5)
    with pytest.raises(mpk.KMeansError):
        mpk.kmeans_set_delta(km.h, float("inf"))
    mpk.kmeans_set_delta(km.h, 0.0)
    km.close()


@pytest.mark.parametrize("dist", ["fp16", "bf16"])
def test_mixed_tile_classes(dist):
    """Rows sorted by norm and several centroid tiles (k = 300): the fp32 kernel sees tiles in
    which no pair, every pair and some pairs trigger (its per-tile shortcut); trigger counts stay
    exact and labels admissible."""
    n, d, k, delta = 4099, 40, 300, 1.5
    Xn, _ = _spread(n, d, 8, "fp32", seed=7)
    order = np.argsort((Xn.astype(np.float64) ** 2).sum(1))
    Xn = np.ascontiguousarray(Xn[order])
    C = synth.init_rows(Xn, k, 3)
    C = np.ascontiguousarray(C[np.argsort((C.astype(np.float64) ** 2).sum(1))])
    lab, st = _gpu_assign(Xn, C, "fp32", dist, delta=delta)
    ref_lab, _, _, ref_low = oracle.assign(Xn, C, "fp32", dist, delta=delta, return_n_low=True)
    D, B, n_trig = _mixed_reference(Xn, C, "fp32", dist, delta)
    assert 0 < ref_low < n * k
    assert st["n_dist_low"] == ref_low
    assert check_labels_admissible(lab, ref_lab, D, B) <= 2e-3
