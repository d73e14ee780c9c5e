"""Parity of the tcgen05 distance + argmin kernel (K4) against the oracle, element by element
(labels admissible under the fp32-accumulation bound B_acc), across tile
shapes: swizzle 32/64/128 B, one or several K-blocks, ragged n (not a multiple of 128 rows or of
the R-row group), ragged k (not a multiple of the 128-column N tile), tiny k."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._parity import check_labels_admissible, dev, distances_on_rounded_operands

pytestmark = pytest.mark.gpu
mpk = pytest.importorskip("paper_2407_12208_b200")

SHAPES = [  # (n, d, k)
    (1000, 64, 256),
    (4099, 128, 1024),
    (2077, 128, 200),
    (3001, 32, 64),
    (1500, 16, 40),
    (777, 200, 130),
    (5000, 8, 16),
    (129, 64, 17),
]


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("guard", [False, True])
def test_tc_assign_matches_oracle(dist, shape, guard):
    n, d, k = shape
    X, _ = synth.blobs(n, d, max(2, k // 3), sigma=1.5, seed=n + d + k, dtype=np.float32)
    Xn, _, _ = oracle.normalize(X, "zscore", work="fp32")
    Xn = Xn.astype(np.float32)
    C = synth.init_rows(Xn, k, 3)
    km = mpk.KMeans(n, d, k, "fp32", dist, guard=guard)
    mpk.kmeans_set_centroids(km.h, dev(C))
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    sse = km.assign(dev(Xn), lab)
    km.close()
    ref, dmin, _ = oracle.assign(Xn, C, work="fp32", dist=dist, guard=guard)
    D, B = distances_on_rounded_operands(Xn, C, "fp32", dist, guard)
    frac = check_labels_admissible(lab.cpu().numpy(), ref, D, B)
    assert frac <= 2e-3
    want = np.maximum(dmin, 0).sum()
    assert abs(sse - want) <= 1e-4 * want


def test_tc_kernel_is_selected():
    X, _ = synth.blobs(3000, 64, 10, seed=1, dtype=np.float32)
    C0 = synth.init_rows(X, 64, 1)
    km = mpk.KMeans(3000, 64, 64, "fp32", "fp16")
    km.fit(dev(X), dev(C0), max_iter=2, tol=-1.0)
    assert km.stats()["dist_kernel"] == "tcgen05"
    km.close()


@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
def test_tc_vs_simt_same_fit(dist):
    """The tensor-core and CUDA-core paths implement the same arithmetic model (rounded
    operands, fp32 accumulation): whole fits agree to the SSE gate."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=20000, seed=5)
    C0 = C0[:128].copy()
    res = []
    for fs in (False, True):
        km = mpk.KMeans(len(X), 64, 128, "fp32", dist, norm="zscore", force_simt=fs)
        lab = torch.empty(len(X), dtype=torch.int32, device="cuda")
        rc, sse, it = km.fit(dev(X), dev(C0), max_iter=10, tol=-1.0, labels=lab)
        res.append((sse, lab.cpu().numpy(), km.stats()["dist_kernel"]))
        km.close()
    assert res[0][2] == "tcgen05" and res[1][2] == "simt_low"
    assert abs(res[0][0] - res[1][0]) <= 1e-4 * res[1][0]
    assert np.mean(res[0][1] == res[1][1]) > 0.995
