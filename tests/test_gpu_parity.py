"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs. Gates from BASELINE.json north_star / SURVEY §8c.4:
  fp64 distance: labels equal except near-ties (gap <= 1e-12 (xn + cn)); SSE rel <= 1e-10
  fp32: SSE rel <= 1e-5;  fp16/bf16 (normalised): SSE rel <= 1e-3, ARI >= 0.99;  E5M2: <= 5e-2
Teacher-forced single steps are compared label by label with the accumulation bound B_acc."""
import numpy as np
import pytest
import torch
from sklearn.metrics import adjusted_rand_score as ari

import oracle
import synth
from tests._parity import U, check_labels_admissible, dev, distances_on_rounded_operands

pytestmark = pytest.mark.gpu

mpk = pytest.importorskip("paper_2407_12208_b200")

TDT = {"fp64": torch.float64, "fp32": torch.float32}
NP = {"fp64": np.float64, "fp32": np.float32}


def gpu_fit(X, C0, work, dist, norm="none", guard=False, max_iter=50, tol=-1.0,
            force_simt=False, on_device=True):
    n, d = X.shape
    k = C0.shape[0]
    km = mpk.KMeans(n, d, k, work, dist, norm=norm, guard=guard, force_simt=force_simt)
    if on_device:
        Xd, Cd = dev(X), dev(C0)
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        cent = torch.empty((k, d), dtype=TDT[work], device="cuda")
    else:
        Xd, Cd = np.ascontiguousarray(X), np.ascontiguousarray(C0)
        lab = np.empty(n, np.int32)
        cent = np.empty((k, d), NP[work])
    rc, sse, iters = km.fit(Xd, Cd, max_iter=max_iter, tol=tol, labels=lab, centroids=cent)
    st = km.stats()
    km.close()
    to_np = (lambda t: t.cpu().numpy()) if on_device else (lambda t: t)
    return dict(rc=rc, sse=sse, iters=iters, labels=to_np(lab), centroids=to_np(cent), stats=st)


# ------------------------------------------------------------------ cast kernel: bit exact
@pytest.mark.parametrize("src", ["fp32", "fp64"])
@pytest.mark.parametrize("dst", ["fp16", "bf16", "e5m2", "fp32"])
def test_cast_bit_exact(src, dst):
    rng = np.random.default_rng(0)
    x = rng.standard_normal(400000) * 10.0 ** rng.integers(-9, 6, 400000)
    t, emin, emax = oracle.format_params(dst)
    special = [0.0, -0.0, np.inf, -np.inf, 65504.0, 65519.99, 65520.0, 57344.0, 61439.0,
               61440.0, -61440.0, 2.0 ** -24, 2.0 ** -25, 1.5 * 2.0 ** -24, 2.0 ** -16,
               2.0 ** -17, 1.5 * 2.0 ** -16, 1.125 + 2.0 ** -40, 1 + 2.0 ** -8 + 2.0 ** -40,
               3.3961e38, 3.3895e38]
    # midpoints between consecutive representable values around many binades
    vals = np.unique(oracle.round_to(dst, x[:2000]))
    vals = vals[np.isfinite(vals)]
    mids = (vals[:-1] + vals[1:]) / 2
    x = np.concatenate([x, special, mids, -mids])
    if src == "fp32":
        with np.errstate(over="ignore"):
            x = x.astype(np.float32).astype(np.float64)
    want = oracle.round_to(dst, x)
    xs = dev(x.astype(NP[src]))
    out_dtype = {"fp16": torch.float16, "bf16": torch.bfloat16, "e5m2": torch.float8_e5m2,
                 "fp32": torch.float32}[dst]
    out = torch.empty(len(x), dtype=out_dtype, device="cuda")
    mpk.kmeans_cast(src, dst, xs, len(x), out)
    got = out.to(torch.float64).cpu().numpy()
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], want[~nan])
    assert np.array_equal(np.signbit(got[~nan]), np.signbit(want[~nan]))


# ------------------------------------------------------------------ C1: n=1000, d=2, k=3
@pytest.mark.parametrize("norm", ["none", "zscore"])
@pytest.mark.parametrize("force_simt", [False, True])
def test_c1_fp64_parity(norm, force_simt):
    X, _, C0 = synth.make("c1_blobs_small", seed=0)
    ref = oracle.fit(X, C0, work="fp64", dist="fp64", norm=norm, max_iter=100, tol=1e-12)
    g = gpu_fit(X, C0, "fp64", "fp64", norm=norm, max_iter=100, tol=1e-12,
                force_simt=force_simt)
    assert g["iters"] == ref["iters"]
    Xn = oracle.apply_normalization(X, ref["shift"], ref["scale"], "fp64") if norm != "none" \
        else X
    D = ((Xn[:, None, :] - ref["centroids"][None, :, :]) ** 2).sum(-1)
    srt = np.sort(D, 1)
    xn = (Xn * Xn).sum(1)
    near = (srt[:, 1] - srt[:, 0]) <= 1e-12 * (xn + (ref["centroids"] ** 2).sum(1).max())
    assert np.all((g["labels"] == ref["labels"]) | near)
    assert abs(g["sse"] - ref["sse"]) <= 1e-10 * ref["sse"]
    assert np.allclose(g["centroids"], ref["centroids"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("norm", ["none", "zscore"])
def test_c1_fp16_parity(norm):
    X, _, C0 = synth.make("c1_blobs_small", seed=0)
    ref = oracle.fit(X, C0, work="fp64", dist="fp16", norm=norm, max_iter=100, tol=1e-12)
    for fs in (False, True):
        g = gpu_fit(X, C0, "fp64", "fp16", norm=norm, max_iter=100, tol=1e-12, force_simt=fs)
        assert abs(g["sse"] - ref["sse"]) <= 1e-3 * ref["sse"]
        assert ari(ref["labels"], g["labels"]) >= 0.99


# ------------------------------------------------------------------ teacher-forced steps
@pytest.mark.parametrize("work,dist", [("fp32", "fp32"), ("fp32", "fp16"), ("fp32", "bf16"),
                                       ("fp32", "e5m2"), ("fp64", "fp64"), ("fp64", "fp16")])
@pytest.mark.parametrize("guard", [False, True])
@pytest.mark.parametrize("force_simt", [False, True])
def test_step_parity(work, dist, guard, force_simt):
    """One Lloyd step from the same centroids: labels admissible under B_acc, counts exact
    where labels agree, centroids within gamma_m (Lemma 5.2)."""
    n, d, k = 5003, 37, 29          # ragged against every tile size
    X, _ = synth.blobs(n, d, 12, sigma=2.0, seed=1, dtype=NP[work])
    Xn, _, _ = oracle.normalize(X, "zscore", work=work)
    Xn = Xn.astype(NP[work])
    C = synth.init_rows(Xn, k, 1)
    ref = oracle.step(Xn, C, work=work, dist=dist, guard=guard)
    km = mpk.KMeans(n, d, k, work, dist, guard=guard, force_simt=force_simt)
    # low-precision labels through kmeans_assign
    km_lab = torch.empty(n, dtype=torch.int32, device="cuda")
    mpk.kmeans_set_centroids(km.h, dev(C))
    km.assign(dev(Xn), km_lab)
    lab = km_lab.cpu().numpy()
    D, B = distances_on_rounded_operands(Xn, C, work, dist, guard)
    frac = check_labels_admissible(lab, ref["labels"], D, B)
    assert frac <= 1e-3
    # one fit iteration from C (update in working precision)
    cent = torch.empty((k, d), dtype=TDT[work], device="cuda")
    km.fit(dev(Xn), dev(C), max_iter=1, tol=-1.0, centroids=cent)
    cg = cent.cpu().numpy().astype(np.float64)
    if frac == 0:
        assert np.array_equal(np.bincount(lab, minlength=k), ref["counts"])
        m = np.maximum(ref["counts"], 1)[:, None]
        tolr = (m * U[work] * 4 + 4 * U[work]) * np.abs(ref["centroids"]) + 1e-30
        assert np.all(np.abs(cg - ref["centroids"]) <= tolr)
    # whatever the labels, the update is eq:center on the GPU's OWN labels (Alg 3 step 4,
    # PAPER.md:547): round_u(mean of the rows labelled j), empty clusters keep c_j — so the
    # counts behind the centres are exactly the label counts, never checked only "on agreement"
    cnt = np.bincount(lab, minlength=k)
    sums = np.zeros((k, d))
    np.add.at(sums, lab, Xn.astype(np.float64))
    want = np.where(cnt[:, None] > 0, sums / np.maximum(cnt, 1)[:, None], C.astype(np.float64))
    want = want.astype(NP[work]).astype(np.float64)
    tolr = (np.maximum(cnt, 1)[:, None] * 2.0 ** -52 + 4 * U[work]) * np.abs(want) + 1e-30
    assert np.all(np.abs(cg - want) <= tolr), np.abs(cg - want).max()
    km.close()


# ------------------------------------------------------------------ end-to-end fits
@pytest.mark.parametrize("dist,gate", [("fp32", 1e-5), ("fp16", 1e-3), ("bf16", 1e-3)])
def test_c3_reduced_fit(dist, gate):
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=30011, seed=0)
    C0 = C0[:64].copy()
    ref = oracle.fit(X, C0, work="fp32", dist=dist, norm="zscore", max_iter=15, tol=-1.0)
    g = gpu_fit(X, C0, "fp32", dist, norm="zscore", max_iter=15, tol=-1.0)
    assert g["iters"] == 15
    assert abs(g["sse"] - ref["sse"]) <= gate * ref["sse"], (g["sse"], ref["sse"])
    assert ari(ref["labels"], g["labels"]) >= 0.99


@pytest.mark.parametrize("variant", ["guard-fp16", "guard-e5m2", "zscore-e5m2", "none-e5m2",
                                     "none-fp16"])
def test_c4_reduced_overflow_modes(variant):
    norm_guard, dist = variant.split("-")
    norm = "zscore" if norm_guard == "zscore" else "none"
    guard = norm_guard == "guard"
    X, _, C0 = synth.make("c4_blobs_1m_large", n=20000, seed=0)
    ref = oracle.fit(X, C0, work="fp32", dist=dist, norm=norm, guard=guard, max_iter=12,
                     tol=-1.0)
    g = gpu_fit(X, C0, "fp32", dist, norm=norm, guard=guard, max_iter=12, tol=-1.0)
    gate = 5e-2 if dist == "e5m2" else 1e-3
    assert abs(g["sse"] - ref["sse"]) <= gate * ref["sse"], (g["sse"], ref["sse"])
    if norm_guard == "none":
        # the paper's failure mode: non-finite operands, flagged, not an error
        assert g["rc"] & mpk.KMEANS_WARN_NONFINITE
        assert g["stats"]["n_nonfinite"] > 0


def test_c2_image_smalld_parity():
    X, truth, C0 = synth.make("c2_image_512", seed=0)
    ref = oracle.fit(X, C0, work="fp32", dist="fp16", norm="minmax", max_iter=20, tol=-1.0)
    g = gpu_fit(X, C0, "fp32", "fp16", norm="minmax", max_iter=20, tol=-1.0)
    assert g["stats"]["dist_kernel"] == "smalld_fused"
    assert abs(g["sse"] - ref["sse"]) <= 1e-3 * ref["sse"]
    assert ari(ref["labels"], g["labels"]) >= 0.99
    # per-iteration SSE trace agrees too
    assert np.allclose(g["stats"]["sse_t"], ref["sse_t"], rtol=1e-3)


# ------------------------------------------------------------------ host buffers / assign / edge cases
def test_host_buffers_equal_device_buffers():
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=8000, seed=2)
    C0 = C0[:32].copy()
    a = gpu_fit(X, C0, "fp32", "fp16", norm="zscore", max_iter=5, on_device=True)
    b = gpu_fit(X, C0, "fp32", "fp16", norm="zscore", max_iter=5, on_device=False)
    assert np.array_equal(a["labels"], b["labels"])
    assert abs(a["sse"] - b["sse"]) <= 1e-9 * a["sse"]


def test_assign_chunks_rows_beyond_n():
    n, d, k = 3000, 16, 10
    X, _ = synth.blobs(n, d, 5, seed=3, dtype=np.float32)
    C = synth.init_rows(X, k, 3)
    Y, _ = synth.blobs(7777, d, 5, seed=4, dtype=np.float32)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    mpk.kmeans_set_centroids(km.h, dev(C))
    lab = torch.empty(len(Y), dtype=torch.int32, device="cuda")
    sse = km.assign(dev(Y), lab)
    ref_lab, dmin, _ = oracle.assign(Y, C, work="fp32", dist="fp16")
    D, B = distances_on_rounded_operands(Y, C, "fp32", "fp16", False)
    check_labels_admissible(lab.cpu().numpy(), ref_lab, D, B)
    assert abs(sse - np.maximum(dmin, 0).sum()) <= 1e-5 * sse
    km.close()


def test_edge_k1_and_k_equals_n():
    X, _ = synth.blobs(777, 5, 3, seed=5, dtype=np.float32)
    g = gpu_fit(X, X[:1].copy(), "fp32", "fp16", max_iter=4)
    mu = X.astype(np.float64).mean(0)
    assert np.allclose(g["centroids"][0], mu, rtol=1e-5, atol=1e-6)
    assert np.all(g["labels"] == 0)
    Xs = X[:50].copy()
    g = gpu_fit(Xs, Xs.copy(), "fp32", "fp32", max_iter=3)
    assert np.array_equal(g["labels"], np.arange(50)) and g["sse"] == 0.0


def test_edge_far_dummy_centroids_stay_empty():
    """Metamorphic pin 4: appended far centroids stay empty, are kept, and
    raise KMEANS_WARN_EMPTY; labels of the real centroids are unchanged."""
    X, _ = synth.blobs(4000, 8, 6, seed=6, dtype=np.float32)
    C0 = synth.init_rows(X, 6, 6)
    a = gpu_fit(X, C0, "fp32", "fp16", max_iter=10)
    far = np.full((3, 8), 1e3 * np.abs(X).max(), np.float32)
    b = gpu_fit(X, np.vstack([C0, far]), "fp32", "fp16", max_iter=10)
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(b["centroids"][6:], far)
    assert b["rc"] & mpk.KMEANS_WARN_EMPTY


def test_metamorphic_power_of_two_scaling():
    """Metamorphic pin 1: (2^e X, 2^e C0) gives identical labels and SSE * 2^(2e)."""
    X, _ = synth.blobs(5000, 24, 10, seed=7, dtype=np.float32)
    C0 = synth.init_rows(X, 10, 7)
    a = gpu_fit(X, C0, "fp32", "fp16", max_iter=8)
    b = gpu_fit(X * np.float32(4.0), C0 * np.float32(4.0), "fp32", "fp16", max_iter=8)
    assert np.array_equal(a["labels"], b["labels"])
    assert abs(b["sse"] - 16 * a["sse"]) <= 1e-6 * b["sse"]


def test_metamorphic_row_permutation():
    X, _ = synth.blobs(6000, 12, 7, seed=8, dtype=np.float32)
    C0 = synth.init_rows(X, 7, 8)
    perm = np.random.default_rng(0).permutation(len(X))
    a = gpu_fit(X, C0, "fp32", "bf16", max_iter=6)
    b = gpu_fit(X[perm].copy(), C0, "fp32", "bf16", max_iter=6)
    assert np.array_equal(a["labels"][perm], b["labels"])
    assert np.allclose(a["centroids"], b["centroids"], rtol=1e-5, atol=1e-6)


def test_nonfinite_inputs_do_not_crash():
    X, _ = synth.blobs(1000, 4 * 5, 4, seed=9, dtype=np.float32)
    X[3, 2] = np.nan
    X[5, 1] = np.inf
    C0 = synth.init_rows(X[10:], 4, 9)
    g = gpu_fit(X, C0, "fp32", "fp16", max_iter=3)
    assert g["labels"].min() >= 0 and g["labels"].max() < 4


def test_convergence_stops_early():
    X, _, C0 = synth.make("c1_blobs_small", seed=1)
    g = gpu_fit(X, C0, "fp64", "fp16", max_iter=300, tol=1e-4)
    assert g["stats"]["converged"] and g["iters"] < 300
    assert not (g["rc"] & mpk.KMEANS_WARN_MAXITER)


def test_dist_handle_single_rank_matches_plain_handle():
    """The NCCL path (kmeans_create_dist: allreduced normalisation statistics, the fixed-point
    update's grid and exact int64 totals, SSE_t / changed and the final SSE) with a 1-rank
    communicator gives the plain handle's results: exercises every collective call site on the
    one GPU a gpurun box has."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=20000, seed=9)
    C0 = C0[:64].copy()
    n, d, k = X.shape[0], 64, 64
    outs = []
    for use_dist in (False, True):
        flags = mpk.KMEANS_NORM_ZSCORE
        if use_dist:
            h = mpk.kmeans_create_dist(n, d, k, "fp32", "fp16", flags, mpk.kmeans_nccl_unique_id(),
                                       1, 0)
        else:
            h = mpk.kmeans_create(n, d, k, "fp32", "fp16", flags)
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        cent = torch.empty((k, d), dtype=torch.float32, device="cuda")
        rc, sse, it = mpk.kmeans_fit(h, dev(X), dev(C0), 8, -1.0, lab, cent)
        outs.append((lab.cpu().numpy(), cent.cpu().numpy(), sse))
        mpk.kmeans_destroy(h)
    # the fixed-point totals (R9) are integers: the NCCL path (int64 allreduce of the totals,
    # max-allreduce of the grid) gives bit-identical labels and centres
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
    assert abs(outs[0][2] - outs[1][2]) <= 1e-12 * outs[0][2]


def test_center_update_bound_trace_matches_oracle():
    """Thm 5.3's per-iteration bound (kmeans_stats.u_bound_t) against the oracle's O11 on the
    same fit; the centres agree to the update's rounding, so the early (large-movement)
    iterations agree closely."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=20011, seed=2)
    C0 = C0[:32].copy()
    ref = oracle.fit(X, C0, work="fp32", dist="fp32", norm="zscore", max_iter=6, tol=-1.0)
    km = mpk.KMeans(len(X), 64, 32, "fp32", "fp32", norm="zscore")
    km.fit(dev(X), dev(C0), max_iter=6, tol=-1.0)
    st = km.stats()
    km.close()
    ub = np.array(st["u_bound_t"])
    assert len(ub) == 6
    np.testing.assert_allclose(ub[:3], ref["u_bound_t"][:3], rtol=1e-3)
    assert st["n_update_prec_short"] == int(np.sum(ub < 2.0 ** -24))


@pytest.mark.parametrize("work,dist,k", [("fp32", "fp16", 300), ("fp64", "fp64", 40),
                                         ("fp32", "fp32", 1)])
def test_update_is_bit_reproducible(work, dist, k):
    """The update (stable bucket sort + ordered boundary reduction, no floating-point atomics)
    gives bit-identical centres, labels and traces on repeated fits — clusters that span many
    segsum chunks (k = 1) and many small clusters (k = 300) alike."""
    X, _, _ = synth.make("c3_blobs_1m_d64", n=250007, seed=11)
    X = X.astype(NP[work])
    C0 = X[np.random.default_rng(k).choice(len(X), k, replace=False)].copy()
    runs = [gpu_fit(X, C0, work, dist, norm="zscore", max_iter=5) for _ in range(3)]
    for r in runs[1:]:
        np.testing.assert_array_equal(r["centroids"], runs[0]["centroids"])
        np.testing.assert_array_equal(r["labels"], runs[0]["labels"])
        assert r["sse"] == pytest.approx(runs[0]["sse"], rel=1e-12)   # atomic fp64 SSE sum
        assert r["stats"]["u_bound_t"] == runs[0]["stats"]["u_bound_t"]



@pytest.mark.parametrize("d", [128, 256])
@pytest.mark.parametrize("dist,guard", [("fp16", False), ("e5m2", True), ("bf16", False)])
def test_wide_rows_zscore_fit_parity(d, dist, guard):
    """Rows of 128 / 256 columns take the vectorised prep (normalise + ||x||^2 + guard scale +
    operand rounding, one pass): z-score transform, per-iteration SSE trace and final SSE agree
    with the oracle (Alg 3 on eq:z-norm data); labels ARI >= 0.99."""
    from sklearn.metrics import adjusted_rand_score
    n, k = 4099, 40
    X, _ = synth.blobs(n, d, 16, sigma=1.5, seed=d, dtype=np.float32)
    X = (X * 3.0 + 5.0).astype(np.float32)
    C0 = synth.init_rows(X, k, 2)
    g = gpu_fit(X, C0, "fp32", dist, norm="zscore", guard=guard, max_iter=4)
    ref = oracle.fit(X, C0, work="fp32", dist=dist, norm="zscore", guard=guard, max_iter=4,
                     tol=-1.0)
    assert abs(g["sse"] - ref["sse"]) <= 1e-3 * ref["sse"]
    st = g["stats"]
    for a, b in zip(st["sse_t"], ref["sse_t"]):
        assert abs(a - b) <= 1e-3 * b
    assert adjusted_rand_score(ref["labels"], g["labels"]) >= 0.99


def _fit_env(env, X, C0, work, dist, **kw):
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return gpu_fit(X, C0, work, dist, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("dist,norm", [("fp16", "zscore"), ("e5m2", "none"), ("fp32", "none")])
def test_fx_incremental_equals_full_resummation(dist, norm):
    """R9: the exact fixed-point totals make a cluster's centre a function of its members only,
    so updating them from the changed rows (MPK_FX_CAP = n: always incremental) and re-summing
    all rows every iteration (MPK_FX_CAP = 0: always the full path) give bit-identical labels,
    centres, SSE traces and counts — over a whole fit in which labels keep changing."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=30000, seed=4)
    C0 = C0[:200].copy()
    a = _fit_env({"MPK_FX_CAP": "0"}, X, C0, "fp32", dist, norm=norm, max_iter=12)
    b = _fit_env({"MPK_FX_CAP": str(len(X))}, X, C0, "fp32", dist, norm=norm, max_iter=12)
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["centroids"].view(np.uint32), b["centroids"].view(np.uint32))
    assert a["stats"]["sse_t"] == b["stats"]["sse_t"]
    assert a["stats"]["changed_t"] == b["stats"]["changed_t"]
    # several iterations after the first two moved labels (the incremental path had work)
    assert sum(1 for c in a["stats"]["changed_t"][2:] if c > 0) >= 2


@pytest.mark.parametrize("dist,k", [("fp16", 1024), ("fp16", 256), ("e5m2", 64), ("bf16", 1024),
                                    ("e5m2", 1024)])
def test_fx_changed_rows_listed_by_the_distance_kernel(dist, k):
    """The CTA-pair kernel lists the changed rows itself (PairParams::fx_list, by 32-row segment,
    from every ASSIGN row end — column split / half split through warp 3, row-block alternation
    and groups, row-block halves) instead of the update's fx_diff pass (MPK_NO_FX_LIST=1): the
    same integer updates, so bit-identical labels, centres and traces over a fit whose labels
    keep changing (incremental and full paths)."""
    X, _, C0 = synth.make("c5_vq_10m", n=70_001, seed=11)
    C0 = C0[:k].copy()
    a = _fit_env({}, X, C0, "fp32", dist, norm="zscore", max_iter=10)
    b = _fit_env({"MPK_NO_FX_LIST": "1"}, X, C0, "fp32", dist, norm="zscore", max_iter=10)
    assert a["stats"]["dist_kernel"] == "tcgen05" and a["stats"]["tc_variant"] == 2
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["centroids"].view(np.uint32), b["centroids"].view(np.uint32))
    assert a["stats"]["sse_t"] == b["stats"]["sse_t"]
    assert a["stats"]["changed_t"] == b["stats"]["changed_t"]
    assert sum(1 for c in a["stats"]["changed_t"][2:] if c > 0) >= 2
    # one launch (fx_diff) fewer per iteration
    assert a["stats"]["n_kernel_launches"] == b["stats"]["n_kernel_launches"] - 10


def test_fx_matches_fp64_summation_path():
    """The fixed-point totals (default) and the fp64 summation of R7 (MPK_NO_FX) agree: the means
    differ at most by the fp64 path's own rounding (a few fp32 ulps), labels essentially equal."""
    X, _, C0 = synth.make("c3_blobs_1m_d64", n=30000, seed=6)
    C0 = C0[:64].copy()
    a = _fit_env({}, X, C0, "fp32", "fp16", norm="zscore", max_iter=8)
    b = _fit_env({"MPK_NO_FX": "1"}, X, C0, "fp32", "fp16", norm="zscore", max_iter=8)
    assert np.mean(a["labels"] == b["labels"]) > 0.999
    assert np.allclose(a["centroids"], b["centroids"], rtol=4 * 2.0 ** -24, atol=1e-6)
    assert abs(a["sse"] - b["sse"]) <= 1e-6 * b["sse"]


def test_fx_centres_are_the_rounded_exact_means():
    """R9: eq:center in precision u (Alg 3 step 4) from the fixed-point totals
    is the exact mean of the members rounded once to fp32 (the quotient is formed exactly,
    k_update.cu fx_quot_rn): every centre equals RN_fp32(exact mean) unless the grid (2^-46 of
    max |x_t| per member) straddles a rounding boundary, checked against exact rationals."""
    n, d, k = 40000, 48, 37
    X, _ = synth.blobs(n, d, 12, sigma=2.0, seed=11, dtype=np.float32)
    X[:, 3] *= 1e-3                                   # features of different magnitudes
    X[:, 7] += 100.0
    C0 = synth.init_rows(X, k, 5)
    km = mpk.KMeans(n, d, k, "fp32", "fp16")
    mpk.kmeans_set_centroids(km.h, dev(C0))
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    km.assign(dev(X), lab)
    cent = torch.empty((k, d), dtype=torch.float32, device="cuda")
    km.fit(dev(X), dev(C0), max_iter=1, tol=-1.0, centroids=cent)
    km.close()
    g = lab.cpu().numpy()
    C = cent.cpu().numpy()
    # exact means: fp32 values are integers times 2^-149, summed as Python integers
    from fractions import Fraction
    XI = np.ldexp(X.astype(np.float64), 149)
    amax = np.abs(X).max(0).astype(np.float64)
    grid = np.ldexp(1.0, np.frexp(amax)[1] - 45)        # g_t = 2^(e_t - 45), 2^e_t > max |x_t|
    n_exact = n_near = 0
    for j in range(k):
        rows = np.nonzero(g == j)[0]
        if rows.size == 0:
            assert np.array_equal(C[j], C0[j])
            continue
        for t in range(d):
            mean = Fraction(sum(int(v) for v in XI[rows, t]), rows.size << 149)
            c = np.float32(float(mean))
            lo, hi = np.nextafter(c, np.float32(-np.inf)), np.nextafter(c, np.float32(np.inf))
            want = min((lo, c, hi), key=lambda v: (abs(Fraction(float(v)) - mean),
                                                   int(np.array(v).view(np.int32)) & 1))
            if C[j, t] == want:
                n_exact += 1
                continue
            # only the grid (|x - q g| <= g / 2 per member) may move the mean across a rounding
            # boundary: then the exact mean lies within g / 2 of the midpoint of C and want
            mid = (Fraction(float(C[j, t])) + Fraction(float(want))) / 2
            assert abs(mean - mid) <= Fraction(float(grid[t])) / 2, (j, t, C[j, t], want)
            n_near += 1
    assert n_near <= 1e-3 * (n_exact + n_near)


def test_one_pass_zscore_matches_two_pass_and_oracle():
    """R4: the one-pass z-score moments (about row 0) give eq:z-norm's mu and sigma (PAPER.md:
    119-126) like the two-pass statistics and the oracle's — the same fp32 transform (the
    handle reports it in the working type) — even with means 1000 sigma away from 0 (the shift
    by a data value removes that cancellation)."""
    rng = np.random.default_rng(3)
    n, d = 50000, 64
    X = (rng.standard_normal((n, d)) * rng.uniform(0.5, 3.0, d) + 1000.0 * rng.uniform(-1, 1, d))
    X = X.astype(np.float32)
    C0 = synth.init_rows(X, 16, 1)
    out = {}
    for name, env in (("one", {}), ("two", {"MPK_TWO_PASS_ZSCORE": "1"})):
        import os
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            km = mpk.KMeans(n, d, 16, "fp32", "fp16", norm="zscore")
            km.fit(dev(X), dev(C0), max_iter=1, tol=-1.0)
            sh, sc = np.empty(d, np.float32), np.empty(d, np.float32)   # working type
            mpk.kmeans_get_transform(km.h, sh, sc)
            km.close()
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        out[name] = (sh, sc)
    ref = oracle.fit(X, C0, work="fp32", dist="fp16", norm="zscore", max_iter=1, tol=-1.0)
    def ulps(a, b):
        return np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))
    want_sh = np.asarray(ref["shift"], np.float64).astype(np.float32)
    want_sc = np.asarray(ref["scale"], np.float64).astype(np.float32)
    for sh, sc in out.values():      # the fp64 statistics agree far below fp32's rounding
        assert ulps(sh, want_sh).max() <= 1 and ulps(sc, want_sc).max() <= 1
        assert np.mean(ulps(sh, want_sh) == 0) >= 0.95 and np.mean(ulps(sc, want_sc) == 0) >= 0.95
