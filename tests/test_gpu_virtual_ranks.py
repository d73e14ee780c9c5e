"""The point-sharded path with g ranks on the one GPU a box has: virtual
ranks (kmeans_vgroup_create / kmeans_create_virtual) run every per-rank step of the NCCL path —
shard statistics, per-shard fixed-point totals and counts, SSE_t partials, the final SSE — each
rank's kmeans_fit on its own host thread, and only the collective differs (a device-side sum in
rank order). eq:center is a sum over points, so summing per-shard partials
must give the single-rank result: with fp32 work the totals are exact integers, so labels and
centres are bit-identical for every g."""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2407_12208_b200 import dist as pd
from tests._parity import dev

pytestmark = pytest.mark.gpu
mpk = pytest.importorskip("paper_2407_12208_b200")


def _plain_fit(X, C0, work, dist, flags, max_iter):
    n, d = X.shape
    k = C0.shape[0]
    h = mpk.kmeans_create(n, d, k, work, dist, flags)
    wt = torch.float64 if work == "fp64" else torch.float32
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    cent = torch.empty((k, d), dtype=wt, device="cuda")
    rc, sse, it = mpk.kmeans_fit(h, dev(X), dev(C0), max_iter, -1.0, lab, cent)
    st = mpk.stats_dict(mpk.kmeans_get_stats(h))
    mpk.kmeans_destroy(h)
    return lab.cpu().numpy(), cent.cpu().numpy(), sse, st


def _virtual_fit(X, C0, work, dist, flags, max_iter, g):
    n, d = X.shape
    k = C0.shape[0]
    grp = mpk.kmeans_vgroup_create(g)
    wt = torch.float64 if work == "fp64" else torch.float32
    ranges = [pd.shard_range(n, g, r) for r in range(g)]
    hs = [mpk.kmeans_create_virtual(r1 - r0, d, k, work, dist, flags, grp, r)
          for r, (r0, r1) in enumerate(ranges)]
    Xs = [dev(X[r0:r1]) for r0, r1 in ranges]
    Cd = dev(C0)
    labs = [torch.empty(r1 - r0, dtype=torch.int32, device="cuda") for r0, r1 in ranges]
    cents = [torch.empty((k, d), dtype=wt, device="cuda") for _ in ranges]
    out = [None] * g
    errs = []

    def run(r):
        try:
            out[r] = mpk.kmeans_fit(hs[r], Xs[r], Cd, max_iter, -1.0, labs[r], cents[r])
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(g)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert all(not t.is_alive() for t in th)
    torch.cuda.synchronize()
    stats = [mpk.stats_dict(mpk.kmeans_get_stats(h)) for h in hs]
    for h in hs:
        mpk.kmeans_destroy(h)
    mpk.kmeans_vgroup_destroy(grp)
    return (np.concatenate([l.cpu().numpy() for l in labs]), [c.cpu().numpy() for c in cents],
            [o[1] for o in out], [o[2] for o in out], stats)


@pytest.mark.parametrize("g", [2, 3, 8])
@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
def test_virtual_ranks_fp32_fx_bit_identical(g, dist):
    """fp32 work (exact fixed-point totals, R9): the g-rank fit equals the 1-rank fit bit for
    bit in labels and centres; the SSE (an fp64 sum over ranks) to 1e-12. The tcgen05 kernel
    runs on every shard (ragged shard sizes)."""
    X, _, C0 = synth.make("c5_vq_10m", n=40_003, seed=4)
    C0 = C0[:256].copy()
    flags = mpk.KMEANS_NORM_NONE
    lab1, cent1, sse1, st1 = _plain_fit(X, C0, "fp32", dist, flags, 6)
    labg, cents, sses, iters, stats = _virtual_fit(X, C0, "fp32", dist, flags, 6, g)
    assert st1["dist_kernel"] == "tcgen05"
    assert all(s["dist_kernel"] == "tcgen05" and s["n_ranks"] == g for s in stats)
    assert iters == [6] * g
    np.testing.assert_array_equal(labg, lab1)
    for c in cents:
        np.testing.assert_array_equal(c.view(np.uint32), cent1.view(np.uint32))
    for s in sses:
        assert s == sses[0]
        assert abs(s - sse1) <= 1e-12 * sse1
    # per-iteration traces: SSE_t and changed are global (allreduced) on every rank
    for s in stats:
        assert s["changed_t"] == st1["changed_t"]
        np.testing.assert_allclose(s["sse_t"], st1["sse_t"], rtol=1e-12)


@pytest.mark.parametrize("g", [2, 3])
@pytest.mark.parametrize("dist", ["fp16", "bf16"])
def test_virtual_ranks_row_block_halves_bit_identical(g, dist):
    """The C5 shape (d = 128, k = 1024: four 256-column tiles per row-block, the warpgroups'
    own half-tile accumulators, k_assign_tc2.cu "rbh") on every shard: the g-rank fit equals the
    1-rank fit bit for bit."""
    X, _, C0 = synth.make("c5_vq_10m", n=60_013, seed=8)
    flags = mpk.KMEANS_NORM_NONE
    lab1, cent1, sse1, st1 = _plain_fit(X, C0, "fp32", dist, flags, 3)
    labg, cents, sses, iters, stats = _virtual_fit(X, C0, "fp32", dist, flags, 3, g)
    assert st1["dist_kernel"] == "tcgen05" and st1["tc_variant"] == 2
    np.testing.assert_array_equal(labg, lab1)
    for c in cents:
        np.testing.assert_array_equal(c.view(np.uint32), cent1.view(np.uint32))
    for s in sses:
        assert abs(s - sse1) <= 1e-12 * sse1


@pytest.mark.parametrize("g", [2, 3])
@pytest.mark.parametrize("dist", ["fp16", "e5m2"])
def test_virtual_ranks_one_tile_groups_bit_identical(g, dist):
    """k = 64 (one 64-column tile per row-block: the warpgroups alternate groups of four
    row-blocks, k_assign_tc2.cu) with >= 4 row-blocks per CTA pair on every shard: the g-rank
    fit equals the 1-rank fit bit for bit."""
    X, _, C0 = synth.make("c5_vq_10m", n=240_007, seed=6)
    C0 = C0[:64].copy()
    flags = mpk.KMEANS_NORM_NONE
    lab1, cent1, sse1, st1 = _plain_fit(X, C0, "fp32", dist, flags, 4)
    labg, cents, sses, iters, stats = _virtual_fit(X, C0, "fp32", dist, flags, 4, g)
    assert st1["dist_kernel"] == "tcgen05" and st1["tc_variant"] == 2
    np.testing.assert_array_equal(labg, lab1)
    for c in cents:
        np.testing.assert_array_equal(c.view(np.uint32), cent1.view(np.uint32))
    for s in sses:
        assert abs(s - sse1) <= 1e-12 * sse1


@pytest.mark.parametrize("g", [2, 3])
def test_virtual_ranks_zscore_matches_oracle(g):
    """z-score statistics allreduced across ranks (two passes, fp64 sums, eq:z-norm
    PAPER.md:119-126): the g-rank fit agrees with the oracle's single-process fit to the fp16
    gates of SURVEY §8c.4 (SSE 1e-3 relative, ARI >= 0.99)."""
    from sklearn.metrics import adjusted_rand_score as ari
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=30_011, seed=6)
    C0 = C0[:64].copy()
    labg, cents, sses, _, _ = _virtual_fit(X, C0, "fp32", "fp16", mpk.KMEANS_NORM_ZSCORE, 8, g)
    ref = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=8, tol=-1.0)
    assert abs(sses[0] - ref["sse"]) <= 1e-3 * ref["sse"]
    assert ari(ref["labels"], labg) >= 0.99
    lab1, cent1, sse1, _ = _plain_fit(X, C0, "fp32", "fp16", mpk.KMEANS_NORM_ZSCORE, 8)
    assert abs(sses[0] - sse1) <= 1e-6 * sse1
    assert np.mean(labg == lab1) >= 0.999


def test_virtual_ranks_fp64_packed_allreduce():
    """fp64 work: the packed fp64 [sums | counts | SSE_t | changed] allreduce (R7 sums per rank,
    summed across ranks): identical centres on every rank, within gamma_m (Lemma 5.2,
    PAPER.md:429-434) of the 1-rank fit (the fp64 sums only change order)."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=12_000, seed=8)
    C0 = C0[:48].copy()
    X = X.astype(np.float64)
    C0 = C0.astype(np.float64)
    lab1, cent1, sse1, _ = _plain_fit(X, C0, "fp64", "fp16", mpk.KMEANS_NORM_NONE, 5)
    labg, cents, sses, _, _ = _virtual_fit(X, C0, "fp64", "fp16", mpk.KMEANS_NORM_NONE, 5, 4)
    assert np.mean(labg == lab1) >= 0.999
    m = len(X)
    for c in cents:
        np.testing.assert_array_equal(c, cents[0])
        np.testing.assert_allclose(c, cent1, rtol=m * 2.0 ** -53 * 4, atol=1e-13)
    assert abs(sses[0] - sse1) <= 1e-12 * sse1


def test_virtual_ranks_small_d_image():
    """The fused small-d kernel (C2's d = 3 image, min-max) on 3 ranks: min/max statistics
    reduced with min/max allreduces, the packed accumulator summed across ranks."""
    X, _, C0 = synth.make("c2_image_512", seed=0)
    labg, cents, sses, _, stats = _virtual_fit(X, C0, "fp32", "fp16", mpk.KMEANS_NORM_MINMAX,
                                               10, 3)
    lab1, cent1, sse1, st1 = _plain_fit(X, C0, "fp32", "fp16", mpk.KMEANS_NORM_MINMAX, 10)
    assert st1["dist_kernel"] == "smalld_fused"
    assert np.mean(labg == lab1) >= 0.9999
    assert abs(sses[0] - sse1) <= 1e-6 * sse1
    for c in cents:
        np.testing.assert_array_equal(c, cents[0])


def test_vgroup_destroy_refused_while_handles_live():
    grp = mpk.kmeans_vgroup_create(2)
    h = mpk.kmeans_create_virtual(100, 8, 4, "fp32", "fp32", 0, grp, 0)
    with pytest.raises(mpk.KMeansError):
        mpk.kmeans_vgroup_destroy(grp)
    mpk.kmeans_destroy(h)
    mpk.kmeans_vgroup_destroy(grp)
    with pytest.raises(mpk.KMeansError):
        mpk.kmeans_vgroup_create(0)
