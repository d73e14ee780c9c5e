"""Python binding of the B200 mixed-precision k-means C ABI (include/kmeans.h).

Argument marshalling only: every step of the hot path runs in the sm_100a kernels of
libmpkmeans.so. Names follow the C ABI. Arrays may be torch tensors (CUDA or CPU) or numpy
arrays; their data pointers are handed to the library, which detects host vs device memory.
If the shared library is missing this module raises ImportError — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpkmeans.so")

KMEANS_FP64, KMEANS_FP32, KMEANS_FP16, KMEANS_BF16, KMEANS_E5M2 = 0, 1, 2, 3, 4
KMEANS_NORM_NONE, KMEANS_NORM_MINMAX, KMEANS_NORM_ZSCORE = 0, 1, 2
KMEANS_GUARD_SCALE = 0x100
KMEANS_FORCE_SIMT = 0x200
KMEANS_GUARD_POW2 = 0x400
KMEANS_OK, KMEANS_EINVAL, KMEANS_ENOMEM, KMEANS_ECUDA, KMEANS_ENCCL, KMEANS_ENODEV = \
    0, -1, -2, -3, -4, -5
KMEANS_WARN_NONFINITE, KMEANS_WARN_EMPTY, KMEANS_WARN_MAXITER, KMEANS_WARN_UNDERFLOW = 1, 2, 4, 8
KMEANS_WARN_SEED_UNIFORM = 16
KMEANS_MAX_TRACE = 1024

PREC = {"fp64": KMEANS_FP64, "fp32": KMEANS_FP32, "fp16": KMEANS_FP16, "bf16": KMEANS_BF16,
        "e5m2": KMEANS_E5M2}
NORM = {"none": KMEANS_NORM_NONE, "minmax": KMEANS_NORM_MINMAX, "zscore": KMEANS_NORM_ZSCORE}
DIST_KERNELS = {0: "simt_work", 1: "simt_low", 2: "tcgen05", 3: "smalld_fused"}
EXPORTS = ["kmeans_create", "kmeans_fit", "kmeans_assign", "kmeans_set_centroids",
           "kmeans_get_centroids", "kmeans_get_transform", "kmeans_get_stats",
           "kmeans_set_stream", "kmeans_set_timing", "kmeans_set_delta", "kmeans_seed_d2",
           "kmeans_destroy",
           "kmeans_last_error",
           "kmeans_cast", "kmeans_create_dist", "kmeans_nccl_unique_id", "kmeans_version",
           "kmeans_vgroup_create", "kmeans_create_virtual", "kmeans_vgroup_destroy"]


class kmeans_stats(ct.Structure):
    _fields_ = [("iters", ct.c_int32), ("converged", ct.c_int32), ("warnings", ct.c_int32),
                ("dist_kernel", ct.c_int32), ("n_nonfinite", ct.c_int64),
                ("n_underflow", ct.c_int64), ("t_prep_ms", ct.c_double),
                ("t_loop_ms", ct.c_double), ("t_final_ms", ct.c_double),
                ("t_dist_ms", ct.c_double), ("t_update_ms", ct.c_double),
                ("t_finalize_ms", ct.c_double), ("t_allreduce_ms", ct.c_double),
                ("n_dist_launches", ct.c_int32), ("trace_len", ct.c_int32),
                ("sse_t", ct.c_double * KMEANS_MAX_TRACE),
                ("shift2_t", ct.c_double * KMEANS_MAX_TRACE),
                ("changed_t", ct.c_int64 * KMEANS_MAX_TRACE),
                ("empty_t", ct.c_int32 * KMEANS_MAX_TRACE),
                ("n_kernel_launches", ct.c_int64), ("n_final_fallback", ct.c_int64),
                ("n_final_uncertified", ct.c_int64), ("n_dist", ct.c_int64),
                ("n_dist_low", ct.c_int64), ("u_bound_t", ct.c_double * KMEANS_MAX_TRACE),
                ("n_update_prec_short", ct.c_int32), ("tc_variant", ct.c_int32),
                ("n_ranks", ct.c_int32), ("eta", ct.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    lib = ct.CDLL(LIB_PATH)
    P, i32, i64, dbl = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_double
    sig = {
        "kmeans_create": (i32, [i64, i32, i32, i32, i32, i32, ct.POINTER(P)]),
        "kmeans_fit": (i32, [P, P, P, i32, dbl, P, P, P, P]),
        "kmeans_assign": (i32, [P, P, i64, P, P]),
        "kmeans_set_centroids": (i32, [P, P]),
        "kmeans_get_centroids": (i32, [P, P]),
        "kmeans_get_transform": (i32, [P, P, P]),
        "kmeans_get_stats": (i32, [P, ct.POINTER(kmeans_stats)]),
        "kmeans_set_stream": (i32, [P, P]),
        "kmeans_set_timing": (i32, [P, i32]),
        "kmeans_set_delta": (i32, [P, ct.c_double]),
        "kmeans_seed_d2": (i32, [P, P, P, P]),
        "kmeans_destroy": (i32, [P]),
        "kmeans_last_error": (ct.c_char_p, [P]),
        "kmeans_cast": (i32, [i32, i32, P, i64, P]),
        "kmeans_create_dist": (i32, [i64, i32, i32, i32, i32, i32, P, i32, i32, ct.POINTER(P)]),
        "kmeans_nccl_unique_id": (i32, [P]),
        "kmeans_vgroup_create": (i32, [i32, ct.POINTER(P)]),
        "kmeans_create_virtual": (i32, [i64, i32, i32, i32, i32, i32, P, i32, ct.POINTER(P)]),
        "kmeans_vgroup_destroy": (i32, [P]),
        "kmeans_version": (ct.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()


class KMeansError(RuntimeError):
    def __init__(self, rc: int, msg: str):
        super().__init__(f"rc={rc}: {msg}")
        self.rc = rc


def _ptr(a):
    """Data pointer of a torch tensor / numpy array (must be contiguous), or None."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported array type {type(a)}")


def _prec(p) -> int:
    return PREC[p] if isinstance(p, str) else int(p)


def _check(rc: int, h=None) -> int:
    if rc < 0:
        raise KMeansError(rc, _lib.kmeans_last_error(h).decode())
    return rc


def kmeans_version() -> str:
    return _lib.kmeans_version().decode()


def kmeans_create(n, d, k, work_prec, dist_prec, flags=0):
    h = ct.c_void_p()
    _check(_lib.kmeans_create(int(n), int(d), int(k), _prec(work_prec), _prec(dist_prec),
                              int(flags), ct.byref(h)), None)
    return h


def kmeans_create_dist(n_local, d, k, work_prec, dist_prec, flags, nccl_id: bytes, nranks, rank):
    h = ct.c_void_p()
    buf = ct.create_string_buffer(bytes(nccl_id), 128)
    _check(_lib.kmeans_create_dist(int(n_local), int(d), int(k), _prec(work_prec),
                                   _prec(dist_prec), int(flags), buf, int(nranks), int(rank),
                                   ct.byref(h)), None)
    return h


def kmeans_vgroup_create(nranks):
    g = ct.c_void_p()
    _check(_lib.kmeans_vgroup_create(int(nranks), ct.byref(g)), None)
    return g


def kmeans_create_virtual(n_local, d, k, work_prec, dist_prec, flags, group, rank):
    h = ct.c_void_p()
    _check(_lib.kmeans_create_virtual(int(n_local), int(d), int(k), _prec(work_prec),
                                      _prec(dist_prec), int(flags), group, int(rank),
                                      ct.byref(h)), None)
    return h


def kmeans_vgroup_destroy(group):
    _check(_lib.kmeans_vgroup_destroy(group), None)


def kmeans_nccl_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    _check(_lib.kmeans_nccl_unique_id(buf))
    return buf.raw


def kmeans_fit(h, X, C0, max_iter, tol, labels=None, centroids=None):
    """Returns (rc, sse, iters); rc >= 0 is the warning mask."""
    sse = ct.c_double()
    iters = ct.c_int32()
    rc = _lib.kmeans_fit(h, _ptr(X), _ptr(C0), int(max_iter), float(tol), _ptr(labels),
                         _ptr(centroids), ct.byref(sse), ct.byref(iters))
    _check(rc, h)
    return rc, sse.value, iters.value


def kmeans_assign(h, X, m, labels, want_sse=True):
    sse = ct.c_double()
    rc = _lib.kmeans_assign(h, _ptr(X), int(m), _ptr(labels), ct.byref(sse) if want_sse else None)
    _check(rc, h)
    return sse.value if want_sse else None


def kmeans_set_centroids(h, C):
    _check(_lib.kmeans_set_centroids(h, _ptr(C)), h)


def kmeans_get_centroids(h, C):
    _check(_lib.kmeans_get_centroids(h, _ptr(C)), h)


def kmeans_get_transform(h, shift, scale):
    _check(_lib.kmeans_get_transform(h, _ptr(shift), _ptr(scale)), h)


def kmeans_get_stats(h) -> kmeans_stats:
    st = kmeans_stats()
    _check(_lib.kmeans_get_stats(h, ct.byref(st)), h)
    return st


def kmeans_set_stream(h, stream_ptr: int | None):
    _check(_lib.kmeans_set_stream(h, stream_ptr), h)


def kmeans_set_timing(h, enable: bool):
    _check(_lib.kmeans_set_timing(h, int(bool(enable))), h)


def kmeans_seed_d2(h, X, u):
    """Alg 1 D^2 seeding in the low precision (R6): returns (indices int64[k], rc)."""
    import numpy as np
    uu = np.ascontiguousarray(np.asarray(u, dtype=np.float64))   # exactly k values
    idx = np.empty(uu.shape[0], np.int64)
    rc = _lib.kmeans_seed_d2(h, _ptr(X), uu.ctypes.data_as(ct.c_void_p),
                             idx.ctypes.data_as(ct.c_void_p))
    _check(rc, h)
    return idx, rc


def kmeans_set_delta(h, delta: float):
    """Alg 4 / Alg 5 per-pair precision switch (0 = off, else delta >= 1)."""
    _check(_lib.kmeans_set_delta(h, float(delta)), h)


def kmeans_destroy(h):
    return _lib.kmeans_destroy(h)


def kmeans_last_error(h=None) -> str:
    return _lib.kmeans_last_error(h).decode()


def kmeans_cast(src_prec, dst_prec, src, count, dst):
    _check(_lib.kmeans_cast(_prec(src_prec), _prec(dst_prec), _ptr(src), int(count), _ptr(dst)))


def stats_dict(st: kmeans_stats) -> dict:
    t = st.trace_len
    return dict(iters=st.iters, converged=bool(st.converged), warnings=st.warnings,
                dist_kernel=DIST_KERNELS.get(st.dist_kernel, st.dist_kernel),
                n_nonfinite=st.n_nonfinite, n_underflow=st.n_underflow,
                t_prep_ms=st.t_prep_ms, t_loop_ms=st.t_loop_ms, t_final_ms=st.t_final_ms,
                t_dist_ms=st.t_dist_ms, t_update_ms=st.t_update_ms,
                t_finalize_ms=st.t_finalize_ms, t_allreduce_ms=st.t_allreduce_ms,
                sse_t=list(st.sse_t[:t]), shift2_t=list(st.shift2_t[:t]),
                changed_t=list(st.changed_t[:t]), empty_t=list(st.empty_t[:t]),
                u_bound_t=list(st.u_bound_t[:t]), n_update_prec_short=st.n_update_prec_short,
                n_kernel_launches=st.n_kernel_launches, n_final_fallback=st.n_final_fallback,
                n_final_uncertified=st.n_final_uncertified, n_dist=st.n_dist,
                n_dist_low=st.n_dist_low, eta=st.eta, tc_variant=st.tc_variant,
                n_ranks=st.n_ranks)


class KMeans:
    """Convenience wrapper owning one handle."""

    def __init__(self, n, d, k, work="fp32", dist="fp16", norm="none", guard=False,
                 force_simt=False, delta=None):
        # guard: False, True (s = ||x||_inf) or "pow2" (s = 2^ceil(log2 ||x||_inf))
        flags = NORM[norm] | (KMEANS_GUARD_SCALE if guard else 0) | \
            (KMEANS_GUARD_POW2 if guard == "pow2" else 0) | \
            (KMEANS_FORCE_SIMT if force_simt else 0)
        self.n, self.d, self.k = int(n), int(d), int(k)
        self.work = work
        self.h = kmeans_create(n, d, k, work, dist, flags)
        if delta is not None:
            kmeans_set_delta(self.h, delta)

    def fit(self, X, C0, max_iter=300, tol=1e-4, labels=None, centroids=None):
        return kmeans_fit(self.h, X, C0, max_iter, tol, labels, centroids)

    def assign(self, X, labels, m=None):
        return kmeans_assign(self.h, X, X.shape[0] if m is None else m, labels)

    def seed(self, X, u):
        """Alg 1 D^2 seeding with the k uniforms u (returns int64 row indices)."""
        if len(u) != self.k:
            raise ValueError(f"need exactly k = {self.k} uniforms")
        return kmeans_seed_d2(self.h, X, u)[0]

    def stats(self) -> dict:
        return stats_dict(kmeans_get_stats(self.h))

    def close(self):
        if self.h is not None:
            kmeans_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
