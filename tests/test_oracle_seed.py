"""Pins for the oracle's D^2 seeding (O10: Alg 1, with Alg 3 step 1's low
precision; reading R6 fixes the draw order). The pins tie it to the paper's
sampling law (probability D(p)^2 / sum D^2, checked by sweeping the uniform), to the O4
assignment routine (the D^2 weights), and to SPEC's worked examples."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def test_k1_is_the_uniform_draw():
    X, _ = synth.blobs(1000, 3, 4, seed=1)
    for u0 in (0.0, 0.3141, 0.999999):
        idx, w = oracle.seed_d2(X, 1, [u0], "fp32", "fp16")
        assert idx[0] == int(u0 * 1000) and w == 0


def test_k_equals_n_chooses_every_point_once():
    """k = n -> every point becomes a centre."""
    X, _ = synth.blobs(50, 2, 3, seed=2)
    u = np.random.default_rng(3).random(50)
    idx, w = oracle.seed_d2(X, 50, u, "fp32", "fp16")
    assert w == 0
    assert sorted(idx.tolist()) == list(range(50))


def test_duplicate_groups_second_centre_in_the_other_group():
    """{a, a, b, b}, k = 2: the D^2 weights inside the first centre's group are 0,
    so the second centre lies in the other group for every draw."""
    X = np.array([[0.0, 0.0], [0.0, 0.0], [9.0, 9.0], [9.0, 9.0]])
    for u0 in (0.1, 0.6):
        first = int(u0 * 4) // 2
        for u1 in np.linspace(0.0, 0.999, 37):
            idx, w = oracle.seed_d2(X, 2, [u0, u1], "fp32", "fp16")
            assert idx[1] // 2 != first and w == 0


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
def test_sampling_law_matches_d2_weights(dist):
    """Line 2 of Alg 1: the next centre is p' with probability D(p')^2 / sum D(p)^2. Sweep u_1
    over a fine grid: the share of u_1 values choosing each index equals its weight. The weights
    come from the independent O4 routine (assignment of every point to the single first centre,
    D = max(0, D_min))."""
    X, _ = synth.blobs(9, 2, 3, seed=4)
    Xn, _, _ = oracle.normalize(X, "zscore", "fp32")
    u0 = 0.5
    c0 = int(u0 * 9)
    _, dmin, _ = oracle.assign(Xn, Xn[c0:c0 + 1], "fp32", dist)
    wts = np.maximum(dmin, 0.0)
    wts[c0] = 0.0            # R6: a chosen centre's own weight is 0 (dist(c, c) = 0)
    M = 20000
    counts = np.zeros(9)
    for m in range(M):
        idx, _ = oracle.seed_d2(Xn, 2, [u0, (m + 0.5) / M], "fp32", dist)
        counts[idx[1]] += 1
    assert counts[c0] == 0
    np.testing.assert_allclose(counts / M, wts / wts.sum(), atol=2.0 / M)


def test_chosen_centres_are_distinct_and_have_positive_weight():
    X, _ = synth.blobs(3000, 5, 7, seed=5)
    u = np.random.default_rng(6).random(40)
    idx, w, d2 = oracle.seed_d2(X, 40, u, "fp32", "fp16", norm="zscore", return_d2=True)
    assert w == 0 and len(set(idx.tolist())) == 40
    # every chosen point is at distance 0 from itself once chosen
    assert np.all(d2[idx] == 0.0)


def test_all_points_identical_falls_back_to_uniform():
    X = np.ones((20, 3))
    idx, w = oracle.seed_d2(X, 3, [0.0, 0.5, 0.75], "fp32", "fp16")
    assert w == 1
    assert idx.tolist() == [0, 10, 15]


def test_seed_weights_are_the_o4_distances_to_the_nearest_centre():
    """oracle.seed_weights (the D^2 of Alg 1 line 2 for given centres) against the independent
    O4 assignment routine: min over the centres of max(0, D^) — from a single-centre assignment
    per centre — with 0 at the centres themselves; and the O10 draw is the inverse-CDF index of
    those weights (numpy's sequential cumulative sum)."""
    X, _ = synth.blobs(2000, 6, 5, seed=12)
    Xn, _, _ = oracle.normalize(X, "zscore", "fp32")
    cen = [17, 1500, 3]
    w = oracle.seed_weights(Xn, cen, "fp32", "fp16")
    want = np.full(len(Xn), np.inf)
    for c in cen:
        _, dmin, _ = oracle.assign(Xn, Xn[c:c + 1], "fp32", "fp16")
        want = np.minimum(want, np.maximum(dmin, 0.0))
    want[cen] = 0.0
    np.testing.assert_array_equal(w, want)
    u = np.array([cen[0] / 2000 + 1e-9, 0.37])
    idx, _ = oracle.seed_d2(Xn, 2, u, "fp32", "fp16")
    w1 = oracle.seed_weights(Xn, [idx[0]], "fp32", "fp16")
    P = np.cumsum(w1)
    assert idx[1] == int(np.argmax(P > u[1] * P[-1]))


def test_multi_block_order_and_determinism():
    """n = 10000: the result does not depend on threads (the sums are sequential by definition)
    and is reproducible."""
    X, _ = synth.blobs(10000, 4, 6, seed=8)
    u = np.random.default_rng(9).random(12)
    a = oracle.seed_d2(X, 12, u, "fp32", "bf16", norm="zscore")
    b = oracle.seed_d2(X, 12, u, "fp32", "bf16", norm="zscore")
    np.testing.assert_array_equal(a[0], b[0])
    assert len(set(a[0].tolist())) == 12
