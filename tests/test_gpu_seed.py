"""GPU D^2 seeding (kmeans_seed_d2, k_seed.cu) against the oracle's O10 (pinned in
tests/test_oracle_seed.py). Reading R6 makes the draw a deterministic function of (X, u) with the
weights formed in fp64 from the stored low-precision operands on both sides, so the chosen
indices must be identical, not merely admissible."""
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


@pytest.mark.parametrize("work,dist,guard", [("fp32", "fp16", False), ("fp32", "bf16", False),
                                             ("fp32", "e5m2", True), ("fp32", "fp32", False),
                                             ("fp32", "fp16", True), ("fp64", "fp16", False),
                                             ("fp64", "fp64", False)])
def test_seed_indices_match_oracle(work, dist, guard):
    n, d, k = 20011, 24, 40                       # 5 seeding blocks, ragged tail
    Xn = _normalised(n, d, 12, work, seed=3)
    u = np.random.default_rng(11).random(k)
    ref, w = oracle.seed_d2(Xn, k, u, work, dist, guard=guard)
    km = mpk.KMeans(n, d, k, work, dist, guard=guard)
    idx = km.seed(dev(Xn), u)
    km.close()
    assert w == 0
    np.testing.assert_array_equal(idx, ref)
    assert len(set(idx.tolist())) == k


def test_seed_from_host_buffer_and_tc_handle():
    """Host input and a C5-shaped handle (tcgen05 distance kernel, padded operand rows)."""
    n, d, k = 9000, 128, 64
    Xn = _normalised(n, d, 20, "fp32", seed=4)
    u = np.random.default_rng(5).random(k)
    ref, _ = oracle.seed_d2(Xn, k, u, "fp32", "fp16")
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    idx = km.seed(Xn, u)
    km.close()
    np.testing.assert_array_equal(idx, ref)


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
    """Alg 3 steps 1-7: D^2 seeding in u_l, then the Lloyd loop and the final pass, against the
    oracle's O10 + fit on the same data and uniforms."""
    n, d, k = 30011, 16, 24
    Xn = _normalised(n, d, 10, "fp32", seed=6)
    u = np.random.default_rng(7).random(k)
    ref_idx, _ = oracle.seed_d2(Xn, k, u, "fp32", "fp16")
    ref = oracle.fit(Xn, Xn[ref_idx], work="fp32", dist="fp16", max_iter=8, tol=-1.0)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    idx = km.seed(dev(Xn), u)
    np.testing.assert_array_equal(idx, ref_idx)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    rc, sse, it = km.fit(dev(Xn), dev(Xn[idx]), max_iter=8, tol=-1.0, labels=lab)
    km.close()
    assert abs(sse - ref["sse"]) <= 1e-3 * ref["sse"]
