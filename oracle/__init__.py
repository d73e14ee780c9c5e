"""CPU oracle for the mixed-precision Lloyd hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference legs) may
import this package. The CUDA product path (paper_2407_12208_b200) never imports it and shares
no code with it. The arithmetic lives in mpkmeans_oracle.c (plain C, fp64, software rounding),
each step citing the PAPER.md passage it follows; this file only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpkmeans_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

PREC = {"fp64": 0, "fp32": 1, "fp16": 2, "bf16": 3, "e5m2": 4}
NORM = {"none": 0, "minmax": 1, "zscore": 2}
GUARD = 0x100


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ct.CDLL(_LIB)
            P = ct.c_void_p
            i64, i32, dbl = ct.c_int64, ct.c_int, ct.c_double
            lib.oracle_round.restype = dbl
            lib.oracle_round.argtypes = [i32, dbl]
            lib.oracle_round_array.argtypes = [i32, P, P, i64]
            lib.oracle_format_params.argtypes = [i32, P, P, P]
            lib.oracle_normalize_stats.argtypes = [i32, i64, i32, P, P, P]
            lib.oracle_normalize_apply.argtypes = [i32, i64, i32, P, P, P, P]
            lib.oracle_fit.argtypes = [i64, i32, i32, i32, i32, i32, P, P, i32, dbl, P, P, P, P,
                                       P, P, P, P, P, P, dbl, P, P]
            lib.oracle_step.argtypes = [i64, i32, i32, i32, i32, i32, P, P, P, P, P, P, P, P,
                                        dbl, P]
            lib.oracle_assign.argtypes = [i64, i32, i32, i32, i32, i32, P, P, P, P, P, dbl, P]
            lib.oracle_prep.argtypes = [i64, i32, i32, i32, i32, P, P, P, P]
            lib.oracle_final.argtypes = [i64, i32, i32, i32, P, P, P, P]
            lib.oracle_num_threads.restype = i32
            lib.oracle_seed_d2.argtypes = [i64, i32, i32, i32, i32, i32, P, P, P, P, P]
            lib.oracle_seed_weights.argtypes = [i64, i32, i32, i32, i32, P, P, i32, P]
            _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p)


def _prec(p) -> int:
    return PREC[p] if isinstance(p, str) else int(p)


GUARD_POW2 = 0x400


def _guard(guard) -> int:
    """False -> 0; True -> 1 (s = ||x||_inf, reading Z9 A); "pow2" -> 2 (Z9 B)."""
    return 2 if guard == "pow2" else (1 if guard else 0)


def _flags(norm="none", guard=False) -> int:
    f = NORM[norm] if isinstance(norm, str) else int(norm)
    return f | (GUARD if guard else 0) | (GUARD_POW2 if guard == "pow2" else 0)


def num_threads() -> int:
    return _load().oracle_num_threads()


def round_to(fmt, v) -> np.ndarray:
    """O0: round fp64 values once (RNE, subnormals, overflow to inf) to format `fmt`."""
    lib = _load()
    x = _f64(v)
    out = np.empty_like(x)
    lib.oracle_round_array(_prec(fmt), _p(x), _p(out), x.size)
    return out


def format_params(fmt) -> tuple[int, int, int]:
    lib = _load()
    t, a, b = ct.c_int(), ct.c_int(), ct.c_int()
    lib.oracle_format_params(_prec(fmt), ct.byref(t), ct.byref(a), ct.byref(b))
    return t.value, a.value, b.value


def normalize(X, norm: str, work="fp64"):
    """O1: returns (X_normalised_in_work_precision, shift[d], scale[d])."""
    lib = _load()
    X = _f64(X)
    n, d = X.shape
    shift, scale = np.empty(d), np.empty(d)
    lib.oracle_normalize_stats(NORM[norm], n, d, _p(X), _p(shift), _p(scale))
    out = np.empty_like(X)
    if NORM[norm] == 0:
        out[:] = round_to(work, X)
    else:
        lib.oracle_normalize_apply(_prec(work), n, d, _p(shift), _p(scale), _p(X), _p(out))
    return out, shift, scale


def apply_normalization(X, shift, scale, work="fp64"):
    lib = _load()
    X = _f64(X)
    out = np.empty_like(X)
    lib.oracle_normalize_apply(_prec(work), X.shape[0], X.shape[1], _p(_f64(shift)),
                               _p(_f64(scale)), _p(X), _p(out))
    return out


def fit(X, C0, work="fp64", dist="fp64", norm="none", guard=False, max_iter=300, tol=1e-4,
        delta=None):
    """Full Lloyd run (O1..O9). Returns a dict with labels, centroids, sse, iters, shift,
    scale and per-iteration traces (sse_t, changed_t, shift2_t, empty_t). delta >= 1 runs Alg 5
    (Alg 4's per-pair precision switch, O4m); n_low counts the triggered low-precision pairs
    over all iterations (eta = n_low / (iters * n * k))."""
    lib = _load()
    X, C0 = _f64(X), _f64(C0)
    n, d = X.shape
    k = C0.shape[0]
    labels = np.empty(n, np.int32)
    cent = np.empty((k, d))
    sse = ct.c_double()
    iters = ct.c_int()
    shift, scale = np.empty(d), np.empty(d)
    tr_sse, tr_ch = np.zeros(max_iter), np.zeros(max_iter, np.int64)
    tr_sh, tr_em = np.zeros(max_iter), np.zeros(max_iter, np.int32)
    n_low = ct.c_int64()
    tr_ub = np.zeros(max_iter)
    rc = lib.oracle_fit(n, d, k, _prec(work), _prec(dist), _flags(norm, guard), _p(X), _p(C0),
                        max_iter, tol, _p(labels), _p(cent), ct.byref(sse), ct.byref(iters),
                        _p(shift), _p(scale), _p(tr_sse), _p(tr_ch), _p(tr_sh), _p(tr_em),
                        float(delta or 0.0), ct.byref(n_low), _p(tr_ub))
    if rc != 0:
        raise ValueError(f"oracle_fit rc={rc}")
    it = iters.value
    return dict(labels=labels, centroids=cent, sse=sse.value, iters=it, shift=shift,
                scale=scale, sse_t=tr_sse[:it], changed_t=tr_ch[:it], shift2_t=tr_sh[:it],
                empty_t=tr_em[:it], n_low=n_low.value, u_bound_t=tr_ub[:it])


def step(X, C, work="fp32", dist="fp16", guard=False, delta=None):
    """One teacher-forced step (O3..O7) on normalised X from centroids C (delta: O4m)."""
    lib = _load()
    X, Cc = _f64(X), _f64(C)
    n, d = X.shape
    k = Cc.shape[0]
    labels = np.empty(n, np.int32)
    dmin, d2 = np.empty(n), np.empty(n)
    sums = np.empty((k, d))
    counts = np.empty(k, np.int64)
    cnext = np.empty((k, d))
    n_low = ct.c_int64()
    rc = lib.oracle_step(n, d, k, _prec(work), _prec(dist), _guard(guard), _p(X), _p(Cc),
                         _p(labels), _p(dmin), _p(d2), _p(sums), _p(counts), _p(cnext),
                         float(delta or 0.0), ct.byref(n_low))
    if rc != 0:
        raise ValueError(f"oracle_step rc={rc}")
    return dict(labels=labels, dmin=dmin, d2nd=d2, sums=sums, counts=counts, centroids=cnext,
                n_low=n_low.value)


def assign(X, C, work="fp32", dist="fp16", guard=False, delta=None, return_n_low=False):
    """Low-precision assignment (O2..O5; O4m with delta): labels, best and second-best expanded
    distance (and the number of triggered low-precision pairs if return_n_low)."""
    lib = _load()
    X, Cc = _f64(X), _f64(C)
    n, d = X.shape
    labels = np.empty(n, np.int32)
    dmin, d2 = np.empty(n), np.empty(n)
    n_low = ct.c_int64()
    rc = lib.oracle_assign(n, d, Cc.shape[0], _prec(work), _prec(dist), _guard(guard), _p(X),
                           _p(Cc), _p(labels), _p(dmin), _p(d2), float(delta or 0.0),
                           ct.byref(n_low))
    if rc != 0:
        raise ValueError(f"oracle_assign rc={rc}")
    if return_n_low:
        return labels, dmin, d2, n_low.value
    return labels, dmin, d2


def prep(X, work="fp32", dist="fp16", guard=False):
    """O2: (low-precision operands, norms x^T x in u, guard scales)."""
    lib = _load()
    X = _f64(X)
    n, d = X.shape
    xl, nrm, sc = np.empty_like(X), np.empty(n), np.empty(n)
    lib.oracle_prep(n, d, _prec(work), _prec(dist), _guard(guard), _p(X), _p(xl), _p(nrm), _p(sc))
    return xl, nrm, sc


def final(X, C, work="fp32"):
    """O9: final working-precision assignment and direct-formula SSE."""
    lib = _load()
    X, Cc = _f64(X), _f64(C)
    labels = np.empty(X.shape[0], np.int32)
    sse = ct.c_double()
    lib.oracle_final(X.shape[0], X.shape[1], Cc.shape[0], _prec(work), _p(X), _p(Cc),
                     _p(labels), ct.byref(sse))
    return labels, sse.value


def seed_d2(X, k, u, work="fp32", dist="fp16", norm="none", guard=False, return_d2=False):
    """O10: D^2 seeding (Alg 1) in the low precision with the caller's uniforms u[k] (reading
    R6). Returns (indices int64[k], warn) — or (indices, warn, final D2) with return_d2."""
    lib = _load()
    X = _f64(X)
    n, d = X.shape
    uu = _f64(u)
    assert uu.shape == (k,)
    idx = np.empty(k, np.int64)
    d2 = np.empty(n) if return_d2 else None
    warn = ct.c_int()
    rc = lib.oracle_seed_d2(n, d, k, _prec(work), _prec(dist), _flags(norm, guard), _p(X),
                            _p(uu), _p(idx), _p(d2) if return_d2 else None, ct.byref(warn))
    if rc != 0:
        raise ValueError(f"oracle_seed_d2 rc={rc}")
    if return_d2:
        return idx, warn.value, d2
    return idx, warn.value


def seed_weights(X, centres, work="fp32", dist="fp16", norm="none", guard=False):
    """O10's D^2 weights (Alg 1 line 2) for the given chosen centres (row indices): min over the
    centres of the low-precision expanded D^2, 0 at the centres — for teacher-forced checks of a
    seeding whose draws were made elsewhere."""
    lib = _load()
    X = _f64(X)
    n, d = X.shape
    c = np.ascontiguousarray(np.asarray(centres, dtype=np.int64))
    out = np.empty(n)
    rc = lib.oracle_seed_weights(n, d, _prec(work), _prec(dist), _flags(norm, guard), _p(X),
                                 _p(c), c.size, _p(out))
    if rc != 0:
        raise ValueError(f"oracle_seed_weights rc={rc}")
    return out
