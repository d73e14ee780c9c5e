"""GPU D^2 seeding (kmeans_seed_d2, k_seed.cu) against the oracle's O10 (pinned in
tests/test_oracle_seed.py). Alg 1 defines a sampling law, not a summation
order: the GPU forms the weights with fp32-accumulated dot products and sums them in a parallel
fixed order, so each draw is checked teacher-forced for ADMISSIBILITY — given the GPU's own
earlier centres, u_j * S must fall inside the chosen index's cumulative-weight interval of the
oracle's weights (oracle.seed_weights), widened by a rigorous bound on the weight and sum
rounding differences — and the centres must be distinct."""
import numpy as np
import pytest
import torch

import oracle
import paper_2407_12208_b200 as mpk
import synth
from tests._parity import dev

pytestmark = pytest.mark.gpu

NP = {"fp32": np.float32, "fp64": np.float64}


def _normalised(n, d, k_true, work, seed):
    X, _ = synth.blobs(n, d, k_true, sigma=2.0, seed=seed, dtype=NP[work])
    Xn, _, _ = oracle.normalize(X, "zscore", work=work)
    return Xn.astype(NP[work])


def check_seed_admissible(Xn, idx, u, work, dist, guard):
    """Every draw j >= 1 of a seeding whose earlier centres are idx[:j]: with the oracle's weights
    W (O10, Alg 1 line 2) and P = cumsum(W), S = P[-1]: P[c-1] - T <= u_j S <= P[c] + T for the
    chosen c, T bounding |W_gpu - W| summed over all rows (fp32 dot accumulation,
    gamma_d(2^-24) |x~|.|c~| per pair, plus the fp64 combination) and the order of the fp64 sums."""
    n, d = Xn.shape
    xl, xn, sx = oracle.prep(Xn, work=work, dist=dist, guard=guard)
    u_acc = 2.0 ** -53 if dist == "fp64" else 2.0 ** -24
    gam = d * u_acc / (1 - d * u_acc)
    absx = np.abs(xl)
    assert len(set(np.asarray(idx).tolist())) == len(idx)
    E = np.zeros(n)
    for j in range(1, len(idx)):
        c_new = idx[j - 1]
        ss = sx * sx[c_new]
        e_new = 2 * ss * gam * (absx @ absx[c_new]) + 8 * 2.0 ** -53 * (
            np.abs(xn) + 2 * ss * np.abs(xl @ xl[c_new]) + abs(xn[c_new]))
        E = np.maximum(E, e_new)
        W = oracle.seed_weights(Xn, idx[:j], work=work, dist=dist, guard=guard)
        P = np.cumsum(W)
        S = P[-1]
        T = E.sum() * (1 + u[j]) + 4 * n * 2.0 ** -53 * S
        c = int(idx[j])
        lo = P[c - 1] if c > 0 else 0.0
        assert lo - T <= u[j] * S <= P[c] + T, (j, c, lo, P[c], u[j] * S, T)
        assert W[c] + E[c] > 0.0, (j, c)


@pytest.mark.parametrize("work,dist,guard", [("fp32", "fp16", False), ("fp32", "bf16", False),
                                             ("fp32", "e5m2", True), ("fp32", "fp32", False),
                                             ("fp32", "fp16", True), ("fp64", "fp16", False),
                                             ("fp64", "fp64", False)])
def test_seed_draws_admissible(work, dist, guard):
    n, d, k = 20011, 24, 40                       # 5 seeding blocks, ragged tail
    Xn = _normalised(n, d, 12, work, seed=3)
    u = np.random.default_rng(11).random(k)
    km = mpk.KMeans(n, d, k, work, dist, guard=guard)
    idx, rc = mpk.kmeans_seed_d2(km.h, dev(Xn), u)
    km.close()
    assert rc == 0
    check_seed_admissible(Xn, idx, u, work, dist, guard)
    # the oracle's own draws (sequential sums, fp64 dots) mostly coincide
    ref, _ = oracle.seed_d2(Xn, k, u, work, dist, guard=guard)
    assert ref[0] == idx[0]


def test_seed_many_blocks_two_level_pick():
    """n = 5M rows (1221 seeding blocks: the pick's first level holds several block sums per
    thread), fp16 operands of 16-byte rows."""
    n, d, k = 5_000_003, 8, 5
    rng = np.random.default_rng(21)
    Xn = rng.standard_normal((n, d)).astype(np.float32)
    Xn[rng.integers(0, n, 50)] *= 30.0            # a few far points carry much of the weight
    u = rng.random(k)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    idx, rc = mpk.kmeans_seed_d2(km.h, dev(Xn), u)
    km.close()
    assert rc == 0
    check_seed_admissible(Xn, idx, u, "fp32", "fp16", False)


def test_seed_from_host_buffer_and_tc_handle():
    """Host input and a C5-shaped handle (tcgen05 distance kernel, padded operand rows)."""
    n, d, k = 9000, 128, 64
    Xn = _normalised(n, d, 20, "fp32", seed=4)
    u = np.random.default_rng(5).random(k)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    idx = km.seed(Xn, u)
    km.close()
    check_seed_admissible(Xn, idx, u, "fp32", "fp16", False)


def test_seed_degenerate_data_warns_and_draws_uniformly():
    X = np.ones((64, 3), np.float32)
    km = mpk.KMeans(64, 3, 3, "fp32", "fp16")
    idx, rc = mpk.kmeans_seed_d2(km.h, dev(X), [0.0, 0.5, 0.75])
    km.close()
    assert rc & mpk.KMEANS_WARN_SEED_UNIFORM
    assert idx.tolist() == [0, 32, 48]


def test_seed_rejects_bad_uniforms():
    km = mpk.KMeans(100, 3, 2, "fp32", "fp16")
    X = np.random.default_rng(0).random((100, 3)).astype(np.float32)
    with pytest.raises(mpk.KMeansError):
        mpk.kmeans_seed_d2(km.h, dev(X), [0.5, 1.0])
    km.close()


def test_alg3_end_to_end_seed_then_fit():
    """Alg 3 steps 1-7: D^2 seeding in u_l (admissible draws), then the Lloyd loop and the final
    pass from those centres, against the oracle's fit from the same C0."""
    n, d, k = 30011, 16, 24
    Xn = _normalised(n, d, 10, "fp32", seed=6)
    u = np.random.default_rng(7).random(k)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    idx = km.seed(dev(Xn), u)
    check_seed_admissible(Xn, idx, u, "fp32", "fp16", False)
    ref = oracle.fit(Xn, Xn[idx], work="fp32", dist="fp16", max_iter=8, tol=-1.0)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    rc, sse, it = km.fit(dev(Xn), dev(Xn[idx]), max_iter=8, tol=-1.0, labels=lab)
    km.close()
    assert abs(sse - ref["sse"]) <= 1e-3 * ref["sse"]
