"""K5p — the small-d Lloyd loop (d <= 4, k <= 8: the image workload) with all
iterations in one cooperative launch — against K5g, one launch per iteration (MPK_NO_PERSIST=1).
Both run the same per-iteration arithmetic in the same order (k_smalld_loop.cu), so labels,
centres, the per-iteration trace and the stopping iteration (Alg 3 step 6) must be
bit-identical; the oracle parity of that arithmetic is test_gpu_parity.py's C1 / C2 tests."""
import numpy as np
import pytest
import torch

import synth
from tests._parity import dev

pytestmark = pytest.mark.gpu
mpk = pytest.importorskip("paper_2407_12208_b200")

TDT = {"fp32": torch.float32, "fp64": torch.float64}


def _fit(X, C0, work, dist, norm, guard, max_iter, tol):
    n, d = X.shape
    k = C0.shape[0]
    km = mpk.KMeans(n, d, k, work, dist, norm=norm, guard=guard)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    cent = torch.empty((k, d), dtype=TDT[work], device="cuda")
    rc, sse, iters = km.fit(dev(X), dev(C0), max_iter=max_iter, tol=tol, labels=lab,
                            centroids=cent)
    st = km.stats()
    km.close()
    assert st["dist_kernel"] == "smalld_fused"
    return dict(rc=rc, sse=sse, iters=iters, labels=lab.cpu().numpy(),
                centroids=cent.cpu().numpy(), stats=st)


def _both(monkeypatch, *args):
    monkeypatch.delenv("MPK_NO_PERSIST", raising=False)
    a = _fit(*args)
    monkeypatch.setenv("MPK_NO_PERSIST", "1")
    b = _fit(*args)
    monkeypatch.delenv("MPK_NO_PERSIST")
    return a, b


def _same(a, b):
    assert a["iters"] == b["iters"]
    assert a["rc"] == b["rc"]
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["centroids"], b["centroids"])
    # the final pass's SSE is an fp64 atomic sum (order not fixed): equal up to rounding
    assert abs(a["sse"] - b["sse"]) <= 1e-12 * abs(b["sse"])
    t = a["iters"]
    for key in ("sse_t", "shift2_t", "changed_t"):
        assert np.array_equal(np.asarray(a["stats"][key])[:t], np.asarray(b["stats"][key])[:t]), key


@pytest.mark.parametrize("dist,guard", [("fp16", False), ("e5m2", False), ("fp16", True),
                                        ("fp32", False)])
def test_c2_persistent_equals_per_launch(dist, guard, monkeypatch):
    X, _, C0 = synth.make("c2_image_512", seed=0)
    a, b = _both(monkeypatch, X, C0, "fp32", dist, "minmax", guard, 20, -1.0)
    _same(a, b)
    assert a["iters"] == 20
    # one launch for the whole loop instead of one per iteration
    assert a["stats"]["n_kernel_launches"] <= b["stats"]["n_kernel_launches"] - 18


@pytest.mark.parametrize("work,dist", [("fp64", "fp64"), ("fp64", "fp16"), ("fp32", "bf16")])
def test_c1_persistent_converges_at_the_same_iteration(work, dist, monkeypatch):
    """With tol >= 0 the loop stops on the device (no label changed, or the shift <= tol):
    the persistent launch leaves at the same iteration, with the same result."""
    X, _, C0 = synth.make("c1_blobs_small", seed=0)
    X = X.astype(np.float64 if work == "fp64" else np.float32)
    C0 = C0.astype(X.dtype)
    a, b = _both(monkeypatch, X, C0, work, dist, "zscore", False, 100, 1e-12)
    _same(a, b)
    assert a["iters"] < 100 and a["stats"]["converged"]


def test_ragged_tiles_and_several_tiles_per_block(monkeypatch):
    """n not a multiple of the 2048-row tile (the ragged last tile is read with plain loads)
    and more tiles than blocks (up to three resident tiles per block, the shared-memory limit
    with the cached operands at d = 3)."""
    rng = np.random.default_rng(4)
    n = 148 * 2048 * 2 + 777
    X = rng.random((n, 3), dtype=np.float32)
    C0 = X[rng.choice(n, 6, replace=False)].copy()
    a, b = _both(monkeypatch, X, C0, "fp32", "fp16", "none", True, 7, -1.0)
    _same(a, b)
    assert a["stats"]["n_kernel_launches"] <= b["stats"]["n_kernel_launches"] - 5


def test_too_large_for_shared_memory_falls_back(monkeypatch):
    """Rows beyond what the blocks' shared memory holds: K5g runs."""
    rng = np.random.default_rng(5)
    n = 148 * 2048 * 9
    X = rng.random((n, 3), dtype=np.float32)
    C0 = X[:5].copy()
    a, b = _both(monkeypatch, X, C0, "fp32", "fp16", "none", False, 3, -1.0)
    _same(a, b)
    assert a["stats"]["n_kernel_launches"] == b["stats"]["n_kernel_launches"]
