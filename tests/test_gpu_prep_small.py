"""The d <= 4 kernels — one row per thread — against the general ones on the same fits.

K1 prep for d <= 4 (the image workload's rows): prep_small_kernel, one row
per thread, against prep_fast_kernel, one row per warp (MPK_PREP_NO_SMALL=1). Both compute the
normalisation O1, ||x||^2, the guard scale and the low-precision operands with the same
arithmetic in the same order (k_prep.cu), so whole fits — labels, centres, the per-iteration
trace and the operand census — must be bit-identical; the oracle parity of that arithmetic is
test_gpu_parity.py's C1 / C2 tests."""
import numpy as np
import pytest
import torch

from tests._parity import dev

pytestmark = pytest.mark.gpu
mpk = pytest.importorskip("paper_2407_12208_b200")


def _fit(X, C0, dist, norm, guard, iters):
    n, d = X.shape
    k = C0.shape[0]
    km = mpk.KMeans(n, d, k, "fp32", dist, norm=norm, guard=guard)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    cent = torch.empty((k, d), dtype=torch.float32, device="cuda")
    rc, sse, it = km.fit(dev(X), dev(C0), max_iter=iters, tol=-1.0, labels=lab, centroids=cent)
    st = km.stats()
    lab2 = torch.empty(n, dtype=torch.int32, device="cuda")
    km.assign(dev(X), lab2)
    km.close()
    return dict(rc=rc, sse=sse, iters=it, labels=lab.cpu().numpy(), centroids=cent.cpu().numpy(),
                relabel=lab2.cpu().numpy(), stats=st)


def _same(a, b):
    assert a["rc"] == b["rc"] and a["iters"] == b["iters"]
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["relabel"], b["relabel"])
    assert np.array_equal(a["centroids"], b["centroids"], equal_nan=True)
    # the final pass's SSE is an fp64 atomic sum (order not fixed): equal up to rounding
    assert abs(a["sse"] - b["sse"]) <= 1e-12 * abs(b["sse"])
    for key in ("n_nonfinite", "n_underflow", "dist_kernel"):
        assert a["stats"][key] == b["stats"][key], key
    t = a["iters"]
    assert np.array_equal(np.asarray(a["stats"]["changed_t"])[:t], np.asarray(b["stats"]["changed_t"])[:t])
    # on the k > 8 paths the per-iteration SSE and shift^2 are fp64 atomic sums across blocks
    # (finalize_kernel): equal up to the order of the additions
    for key in ("sse_t", "shift2_t"):
        np.testing.assert_allclose(np.asarray(a["stats"][key])[:t], np.asarray(b["stats"][key])[:t],
                                   rtol=1e-12, atol=0, err_msg=key)


def _both(monkeypatch, *args, env="MPK_PREP_NO_SMALL"):
    monkeypatch.delenv(env, raising=False)
    a = _fit(*args)
    monkeypatch.setenv(env, "1")
    b = _fit(*args)
    monkeypatch.delenv(env)
    return a, b


@pytest.mark.parametrize("d", [1, 2, 3, 4])
@pytest.mark.parametrize("dist,norm,guard", [("fp16", "minmax", False), ("e5m2", "none", True),
                                             ("bf16", "zscore", "pow2"), ("fp32", "none", False)])
def test_small_d_prep_equals_warp_per_row(d, dist, norm, guard, monkeypatch):
    rng = np.random.default_rng(10 + d)
    n = 148 * 256 * 3 + 91                       # several grid sweeps and a ragged tail
    X = (rng.standard_normal((n, d)) * 40.0 + 7.0).astype(np.float32)
    for k in (6, 20):                            # the fused small-d loop (k <= 8) and K2 / K4
        C0 = X[rng.choice(n, k, replace=False)].copy()
        a, b = _both(monkeypatch, X, C0, dist, norm, guard, 4)
        _same(a, b)


def test_small_d_census_overflow_and_underflow(monkeypatch):
    """Unnormalised, unguarded rows beyond E5M2's range and below its subnormals: both kernels
    count the same operands as non-finite / underflowed."""
    rng = np.random.default_rng(3)
    n = 50_000
    X = rng.standard_normal((n, 3)).astype(np.float32)
    X[::7, 0] *= 1e6                             # overflows E5M2 (max 57344)
    X[::5, 2] *= 1e-9                            # below E5M2's smallest subnormal
    C0 = X[:5].copy()
    a, b = _both(monkeypatch, X, C0, "e5m2", "none", False, 2)
    assert a["stats"]["n_nonfinite"] > 0 and a["stats"]["n_underflow"] > 0
    for key in ("n_nonfinite", "n_underflow"):
        assert a["stats"][key] == b["stats"][key], key
    assert np.array_equal(a["labels"], b["labels"])


@pytest.mark.parametrize("d", [1, 3, 4])
@pytest.mark.parametrize("dist,k", [("fp16", 6), ("fp32", 6), ("fp32", 40), ("bf16", 200)])
def test_small_d_assign_equals_register_tiled(d, dist, k, monkeypatch):
    """assign_simt_small_kernel (d <= 4, k <= 256) against K6b, the 8 x 8 register-tiled kernel
    (MPK_SIMT_NO_SMALL=1): the final pass in working precision (A8) and, for fp32 distances,
    every Lloyd iteration. Labels and centres bit-identical; the final SSE
    (final_sse_small_kernel vs final_sse_fast_kernel, both compensated sums) within 1e-12."""
    rng = np.random.default_rng(20 + d)
    n = 148 * 256 * 2 + 333
    X = (rng.standard_normal((n, d)) * 3.0).astype(np.float32)
    X[:50] = X[50:100]                           # duplicate rows: equal distances, tie order
    C0 = X[rng.choice(n, k, replace=False)].copy()
    a, b = _both(monkeypatch, X, C0, dist, "minmax", False, 5, env="MPK_SIMT_NO_SMALL")
    _same(a, b)


@pytest.mark.parametrize("d,norm,dist", [(64, "zscore", "fp16"), (3, "minmax", "fp16"),
                                         (32, "minmax", "e5m2"), (200, "zscore", "bf16")])
def test_warp_combine_equals_thread_combine(d, norm, dist, monkeypatch):
    """The normalisation statistics' cross-block combine (O1): one warp per column staging the
    partials in shared memory vs one thread per column (MPK_COMBINE_THREAD=1). Same additions
    in the same block order: the transform, and so the whole fit, bit-identical."""
    rng = np.random.default_rng(30 + d)
    n = 300_000 if d <= 64 else 60_000
    X = (rng.standard_normal((n, d)) * 5.0 + 100.0).astype(np.float32)
    C0 = X[rng.choice(n, 16, replace=False)].copy()
    a, b = _both(monkeypatch, X, C0, dist, norm, False, 3, env="MPK_COMBINE_THREAD")
    _same(a, b)


@pytest.mark.parametrize("d,norm,dist,guard", [(64, "zscore", "fp16", False), (32, "none", "e5m2", True),
                                               (64, "minmax", "bf16", "pow2"), (32, "zscore", "fp16", False)])
def test_grouped_prep_matches_warp_per_row(d, norm, dist, guard, monkeypatch):
    """prep_vecg_kernel (d = 32 / 64: G = d/4 lanes per row) against prep_fast_kernel
    (MPK_PREP_NO_VECG=1). The normalised rows, the low operands and the guard scales are the
    same per element; ||x||^2 is summed over the lanes in another grouping (both exact-product
    compensated sums, rounded once to fp32), so a norm may differ by one ulp in rare rows:
    labels equal up to near-ties, the fit's SSE to 1e-9."""
    rng = np.random.default_rng(40 + d)
    n = 200_003
    X = (rng.standard_normal((n, d)) * 3.0 + 1.0).astype(np.float32)
    C0 = X[rng.choice(n, 48, replace=False)].copy()
    a, b = _both(monkeypatch, X, C0, dist, norm, guard, 4, env="MPK_PREP_NO_VECG")
    assert a["iters"] == b["iters"] and a["rc"] == b["rc"]
    assert (a["labels"] != b["labels"]).mean() <= 1e-4
    assert abs(a["sse"] - b["sse"]) <= 1e-9 * abs(b["sse"])
    for key in ("n_nonfinite", "n_underflow"):
        assert a["stats"][key] == b["stats"][key], key
