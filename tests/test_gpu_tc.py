"""Parity of the tcgen05 distance + argmin kernel (K4) against the oracle, element by element
(labels admissible under the fp32-accumulation bound B_acc), across tile
shapes: swizzle 32/64/128 B, one or several K-blocks, ragged n (not a multiple of 128 rows or of
the R-row group), ragged k (not a multiple of the 128-column N tile), tiny k."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._parity import (check_admissible_rows, check_labels_admissible, dev,
                           distances_on_rounded_operands)

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
    (3001, 64, 96),     # streaming kernel: a 96-column tile (three 32-column chunks)
]


def _set_kind(monkeypatch, kind):
    """kind 2: the CTA-pair kernel (k_assign_tc2.cu) wherever its resident centroid halves fit;
    kind 1: the streaming kernel (k_assign_tc.cu), forced with MPK_TC_KIND=1 (it is selected
    on its own when k is too large for the pair kernel, see test_tc_large_k_streaming)."""
    if kind == 1:
        monkeypatch.setenv("MPK_TC_KIND", "1")
    else:
        monkeypatch.delenv("MPK_TC_KIND", raising=False)


def _assign_vs_oracle(n, d, k, dist, guard, seed, want_variant=None, max_frac=2e-3):
    X, _ = synth.blobs(n, d, max(2, k // 3), sigma=1.5, seed=seed, dtype=np.float32)
    Xn, _, _ = oracle.normalize(X, "zscore", work="fp32")
    Xn = Xn.astype(np.float32)
    C = synth.init_rows(Xn, k, 3)
    km = mpk.KMeans(n, d, k, "fp32", dist, guard=guard)
    mpk.kmeans_set_centroids(km.h, dev(C))
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    sse = km.assign(dev(Xn), lab)
    st = km.stats()
    km.close()
    assert st["dist_kernel"] == "tcgen05"
    if want_variant is not None:
        assert st["tc_variant"] == want_variant
    ref, dmin, _ = oracle.assign(Xn, C, work="fp32", dist=dist, guard=guard)
    frac = check_admissible_rows(Xn, C, lab.cpu().numpy(), ref, "fp32", dist, guard)
    assert frac <= max_frac
    want = np.maximum(dmin, 0).sum()
    assert abs(sse - want) <= 1e-4 * want
    return frac


@pytest.mark.parametrize("kind", [2, 1])
@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("guard", [False, True])
def test_tc_assign_matches_oracle(dist, shape, guard, kind, monkeypatch):
    _set_kind(monkeypatch, kind)
    n, d, k = shape
    es = 1 if dist == "e5m2" else 2
    variant = None
    if kind == 1:
        # the streaming kernel holds rows of at most 256 bytes; 512-byte rows stay on the pair
        # kernel even when kind 1 is requested
        variant = 1 if mpk_row_bytes(d, es) <= 256 else 2
    _assign_vs_oracle(n, d, k, dist, guard, n + d + k, want_variant=variant)


def mpk_row_bytes(d, es):
    """Padded operand row length in bytes (k_assign_tc.cu tc_dpad)."""
    rb = (d * es + 31) // 32 * 32
    return (rb + 127) // 128 * 128 if rb > 64 else rb


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
@pytest.mark.parametrize("guard", [False, True])
def test_tc_deep_row_blocks_c5_shape(dist, guard, monkeypatch):
    """The C5 shape (d = 128, k = 1024) with n = 200 003: every CTA pair of the 74 runs >= 10
    row-blocks of 256 rows, so the X~ ring wraps (SA slots, phase flips) and the partial
    buffers are reused (part_free, row-block index >= 2) many times, as at the bench size —
    against the oracle label by label (admissible under 2 B_acc), with a ragged tail."""
    _set_kind(monkeypatch, 2)
    _assign_vs_oracle(200_003, 128, 1024, dist, guard, 77, want_variant=2)


@pytest.mark.parametrize("dist", ["fp16", "bf16", "e5m2"])
@pytest.mark.parametrize("guard", [False, True])
@pytest.mark.parametrize("shape", [(200_003, 64, 256), (120_001, 32, 64), (90_007, 16, 40)])
def test_tc_deep_row_blocks_one_tile(dist, guard, shape, monkeypatch):
    """One centroid tile per row-block (the C3 / C4 shapes: k <= 256): the two epilogue
    warpgroups alternate row-blocks and each does its own row-block end (k_assign_tc2.cu
    "row-block alternation"); >= 4 row-blocks per CTA pair, so both warpgroups cycle through
    every accumulator more than once — against the oracle label by label, ragged tail."""
    _set_kind(monkeypatch, 2)
    n, d, k = shape
    _assign_vs_oracle(n, d, k, dist, guard, n + k, want_variant=2)


@pytest.mark.parametrize("dist", ["fp16", "bf16"])
@pytest.mark.parametrize("shape", [(150_001, 200, 16), (150_001, 256, 40)])
def test_tc_row_block_groups_with_few_row_slots(dist, shape, monkeypatch):
    """512-byte operand rows leave room for only 3 X~ row-block slots, fewer than a group of
    4 row-blocks per accumulator (k <= 64): the plan halves the group (k_assign_tc2.cu
    pair_plan) — before, the MMA issuer waited for a slot that no one could free. Padded columns
    (d = 200 -> d_pad = 256), many row-blocks per CTA pair, against the oracle."""
    _set_kind(monkeypatch, 2)
    n, d, k = shape
    _assign_vs_oracle(n, d, k, dist, False, n + d, want_variant=2)


@pytest.mark.parametrize("dist,shape", [("fp16", (200_003, 64, 256)), ("e5m2", (120_001, 32, 64))])
def test_tc_one_tile_alternation_equals_column_split(dist, shape, monkeypatch):
    """The row-block alternation and the column split (MPK_PAIR_DBG bit 5) fold the same values
    in the same reverse order: identical labels, the SSE equal up to its summation order."""
    n, d, k = shape
    X, _ = synth.blobs(n, d, max(2, k // 3), sigma=1.5, seed=5, dtype=np.float32)
    C = synth.init_rows(X, k, 3)
    out = []
    for dbg in ("0", "32"):
        monkeypatch.setenv("MPK_PAIR_DBG", dbg)
        km = mpk.KMeans(n, d, k, "fp32", dist, guard=True)
        mpk.kmeans_set_centroids(km.h, dev(C))
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        sse = km.assign(dev(X), lab)
        assert km.stats()["tc_variant"] == 2
        km.close()
        out.append((lab.cpu().numpy(), sse))
    monkeypatch.delenv("MPK_PAIR_DBG")
    assert np.array_equal(out[0][0], out[1][0])
    assert abs(out[0][1] - out[1][1]) <= 1e-9 * abs(out[1][1])


@pytest.mark.parametrize("dist,guard", [("fp16", False), ("bf16", True)])
def test_tc_row_block_halves_equal_column_split(dist, guard, monkeypatch):
    """C5 shape (four 256-column tiles per row-block): the warpgroups' own half-tile
    accumulators ("rbh") and the column split (MPK_PAIR_DBG bit 6) visit the same values in the
    same decreasing column order: identical labels, the SSE equal up to its summation order."""
    n, d, k = 120_011, 128, 1024
    X, _ = synth.blobs(n, d, 300, sigma=1.5, seed=9, dtype=np.float32)
    C = synth.init_rows(X, k, 2)
    out = []
    for dbg in ("0", "64"):
        monkeypatch.setenv("MPK_PAIR_DBG", dbg)
        km = mpk.KMeans(n, d, k, "fp32", dist, guard=guard)
        mpk.kmeans_set_centroids(km.h, dev(C))
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        sse = km.assign(dev(X), lab)
        assert km.stats()["tc_variant"] == 2
        km.close()
        out.append((lab.cpu().numpy(), sse))
    monkeypatch.delenv("MPK_PAIR_DBG")
    assert np.array_equal(out[0][0], out[1][0])
    assert abs(out[0][1] - out[1][1]) <= 1e-9 * abs(out[1][1])


@pytest.mark.parametrize("dist,k,variant", [("fp16", 2048, 1), ("bf16", 2048, 1),
                                            ("e5m2", 2048, 2), ("e5m2", 4096, 1)])
def test_tc_large_k_streaming(dist, k, variant, monkeypatch):
    """k beyond the pair kernel's resident centroid halves (d = 128: k > ~1300 at fp16, > ~2600
    at E5M2) selects the streaming kernel without any override; parity as above."""
    _set_kind(monkeypatch, 2)
    _assign_vs_oracle(20_011, 128, k, dist, False, k + 5, want_variant=variant)


def test_wide_rows_large_k_use_cuda_cores():
    """fp16 rows of 512 bytes (d = 256) with k = 1024: neither tcgen05 plan fits in shared
    memory, so the handle takes the CUDA-core low-precision kernel (same arithmetic model) —
    created without error and parity-green."""
    n, d, k = 3001, 256, 1024
    X, _ = synth.blobs(n, d, 50, sigma=1.5, seed=3, dtype=np.float32)
    Xn, _, _ = oracle.normalize(X, "zscore", work="fp32")
    Xn = Xn.astype(np.float32)
    C = synth.init_rows(Xn, k, 3)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    mpk.kmeans_set_centroids(km.h, dev(C))
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    km.assign(dev(Xn), lab)
    st = km.stats()
    km.close()
    assert st["dist_kernel"] == "simt_low" and st["tc_variant"] == 0
    ref, _, _ = oracle.assign(Xn, C, work="fp32", dist="fp16", guard=False)
    assert check_admissible_rows(Xn, C, lab.cpu().numpy(), ref, "fp32", "fp16", False) <= 2e-3


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


@pytest.mark.parametrize("kind", [2, 1])
@pytest.mark.parametrize("dist,guard", [("fp16", False), ("bf16", False), ("e5m2", False),
                                        ("fp16", True), ("e5m2", True)])
def test_final_pass_certified_filter(dist, guard, kind, monkeypatch):
    """Alg 3 step 7 via the certified tensor-core filter: the final labels equal the
    working-precision argmin for the returned centroids (checked against an fp64 evaluation,
    mismatches allowed only within the fp32 evaluation error), with few CUDA-core fallbacks."""
    _set_kind(monkeypatch, kind)
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=25000, seed=3)
    C0 = C0[:96].copy()
    km = mpk.KMeans(len(X), 64, 96, "fp32", dist, norm="zscore", guard=guard)
    lab = torch.empty(len(X), dtype=torch.int32, device="cuda")
    cent = torch.empty((96, 64), dtype=torch.float32, device="cuda")
    rc, sse, it = km.fit(dev(X), dev(C0), max_iter=6, tol=-1.0, labels=lab, centroids=cent)
    st = km.stats()
    shift = np.empty(64, np.float32)
    scale = np.empty(64, np.float32)
    mpk.kmeans_get_transform(km.h, shift, scale)
    km.close()
    assert st["dist_kernel"] == "tcgen05" and st["tc_variant"] == kind
    if kind == 2:
        # uncertified rows are resolved from their candidate columns (R2)
        assert 0 <= st["n_final_fallback"] <= 0.01 * len(X)
    else:
        # the streaming kernel has no candidate mode: every uncertified row is re-evaluated
        # over all k centroids on CUDA cores
        assert st["n_final_fallback"] == st["n_final_uncertified"] <= 0.3 * len(X)
    ref = oracle.fit(X, C0, work="fp32", dist=dist, norm="zscore", guard=guard, max_iter=6,
                     tol=-1.0)
    Xn = oracle.apply_normalization(X, ref["shift"], ref["scale"], "fp32")
    C = cent.cpu().numpy().astype(np.float64)
    g = lab.cpu().numpy()
    want, _ = oracle.final(Xn, C, work="fp32")
    D = (Xn * Xn).sum(1)[:, None] - 2 * Xn @ C.T + (C * C).sum(1)[None, :]
    bad = np.nonzero(g != want)[0]
    if bad.size:
        tol = 2 * (66 * 2.0 ** -24) * ((Xn * Xn).sum(1) + 2 * np.sqrt((Xn * Xn).sum(1) * (C * C).sum(1).max())
                                       + (C * C).sum(1).max())
        gap = D[bad, g[bad]] - D[bad, want[bad]]
        assert np.all(gap <= tol[bad]), gap.max()
    direct = float(np.sum((Xn - C[g]) ** 2))
    assert abs(sse - direct) <= 1e-6 * direct


@pytest.mark.parametrize("dist,guard", [("fp16", False), ("e5m2", False), ("fp16", True)])
def test_final_pass_candidates_match_full_evaluation(dist, guard, monkeypatch):
    """DESIGN.md R2: the final pass resolves uncertified rows from their candidate columns
    (v^_j <= T). The labels must be bit-identical to the full CUDA-core evaluation of every
    uncertified row (MPK_NO_CAND=1), on a workload with many near-ties (1024 clusters in 128-d,
    the C5 shape) so that the candidate path is exercised."""
    X, _, C0 = synth.make("c5_vq_10m", n=60000, seed=11)
    labs, stats = [], []
    for no_cand in (False, True):
        if no_cand:
            monkeypatch.setenv("MPK_NO_CAND", "1")
        else:
            monkeypatch.delenv("MPK_NO_CAND", raising=False)
        km = mpk.KMeans(len(X), 128, 1024, "fp32", dist, norm="zscore", guard=guard)
        lab = torch.empty(len(X), dtype=torch.int32, device="cuda")
        km.fit(dev(X), dev(C0), max_iter=3, tol=-1.0, labels=lab)
        labs.append(lab.cpu().numpy())
        stats.append(km.stats())
        km.close()
    cand, full = stats
    assert cand["dist_kernel"] == "tcgen05"
    assert cand["n_final_uncertified"] == full["n_final_uncertified"] > 100
    # most uncertified rows are resolved from their candidates
    assert cand["n_final_fallback"] < 0.2 * cand["n_final_uncertified"]
    assert full["n_final_fallback"] == full["n_final_uncertified"]
    np.testing.assert_array_equal(labs[0], labs[1])


@pytest.mark.parametrize("dist,guard", [("fp16", False), ("e5m2", False), ("bf16", True)])
@pytest.mark.parametrize("k", [1024, 200])
def test_tc_exact_ties_take_the_first_column(dist, guard, k):
    """Duplicated centroids give bit-identical distances (same operands, same accumulation):
    the argmin must take the FIRST of the tied columns (the sequential scan's rule, Alg 3 step 3,
    PAPER.md:546), wherever the duplicates sit (same chain, same tile, other tiles). The ASSIGN
    kernel scans columns in reverse (fold_rev_m3), so this pins its non-strict tie rule."""
    n, d = 6000, 128
    rng = np.random.default_rng(k)
    C = rng.standard_normal((k, d)).astype(np.float32)
    pairs = [(0, 8), (3, k - 1), (5, 13), (17, k // 2 + 1), (k // 2, k // 2 + 8), (40, 41)]
    later = set()
    for a, b in pairs:
        C[b] = C[a]
        later.add(b)
    src = np.array([a for a, _ in pairs])
    X = C[src[rng.integers(0, len(src), n)]] + 0.05 * rng.standard_normal((n, d)).astype(np.float32)
    X[: n // 4] = rng.standard_normal((n // 4, d)).astype(np.float32)
    km = mpk.KMeans(n, d, k, "fp32", dist, guard=guard)
    mpk.kmeans_set_centroids(km.h, dev(C))
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    km.assign(dev(X), lab)
    km.close()
    g = lab.cpu().numpy()
    assert not np.isin(g, list(later)).any()
    ref, _, _ = oracle.assign(X, C, work="fp32", dist=dist, guard=guard)
    D, B = distances_on_rounded_operands(X, C, "fp32", dist, guard)
    assert check_labels_admissible(g, ref, D, B) <= 2e-3


@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
def test_tc_nonfinite_rows_match_the_scan(dist):
    """Rows whose distances are all NaN / +inf take column 0 and rows with a -inf distance take
    the first such column — the sequential scan's results, as the oracle computes them."""
    n, d, k = 600, 64, 300
    rng = np.random.default_rng(7)
    X = rng.standard_normal((n, d)).astype(np.float32)
    C = rng.standard_normal((k, d)).astype(np.float32)
    X[0] = np.nan
    X[1, 3] = np.inf
    X[2, 5] = -np.inf
    X[3, :] = 1e30
    km = mpk.KMeans(n, d, k, "fp32", dist)
    mpk.kmeans_set_centroids(km.h, dev(C))
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    km.assign(dev(X), lab)
    km.close()
    g = lab.cpu().numpy()
    ref, _, _ = oracle.assign(X, C, work="fp32", dist=dist, guard=False)
    assert g[0] == 0
    assert np.array_equal(g[:4], ref[:4]), (g[:4], ref[:4])


@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
@pytest.mark.parametrize("shape", [(4099, 128, 1024), (3001, 32, 64), (1500, 16, 40)])
def test_tc_guard_pow2_matches_oracle(dist, shape):
    """Reading Z9 B (KMEANS_GUARD_POW2, s = 2^ceil(log2 ||x||_inf)) on the tensor-core kernels,
    label by label against the oracle's O2 with the same reading."""
    n, d, k = shape
    _assign_vs_oracle(n, d, k, dist, "pow2", n + 3 * d + k)
