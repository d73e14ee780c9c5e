"""Shared helpers of the GPU parity tests (test-side arithmetic only; never imported by the
product path)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

U = {"fp64": 2.0 ** -53, "fp32": 2.0 ** -24, "fp16": 2.0 ** -11, "bf16": 2.0 ** -8,
     "e5m2": 2.0 ** -3}


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def distances_on_rounded_operands(X, C, work, dist, guard):
    """D_ij = xn_i - 2 s_i s_j x~_i.c~_j + cn_j in fp64 from the oracle's O2/O3 operands, plus
    the accumulation bound B_acc: 2 s_i s_j gamma_d(2^-24) |x~_i|.|c~_j| +
    3 u_ep (xn_i + cn_j + 2 s_i s_j |x~_i . c~_j|)."""
    xl, xn, sx = oracle.prep(X, work=work, dist=dist, guard=guard)
    cl, cn, sc = oracle.prep(C, work=work, dist=dist, guard=guard)
    dot = xl @ cl.T
    ss = sx[:, None] * sc[None, :]
    D = xn[:, None] - 2.0 * ss * dot + cn[None, :]
    d = X.shape[1]
    u_acc = 2.0 ** -53 if dist == "fp64" else 2.0 ** -24
    u_ep = 2.0 ** -53 if work == "fp64" else 2.0 ** -24
    gam = d * u_acc / (1 - d * u_acc)
    B = 2 * ss * gam * (np.abs(xl) @ np.abs(cl).T) + 3 * u_ep * (
        np.abs(xn)[:, None] + np.abs(cn)[None, :] + 2 * ss * np.abs(dot))
    return D, B


def check_labels_admissible(lab_gpu, lab_ref, D, B, slack=2.0):
    """Labels may differ only where the GPU's choice is within B of the oracle's minimum:
    D[i, g] - D[i, j*] <= slack * (B[i, g] + B[i, j*]). Returns the mismatch fraction."""
    lab_gpu = np.asarray(lab_gpu)
    lab_ref = np.asarray(lab_ref)
    bad = np.nonzero(lab_gpu != lab_ref)[0]
    if bad.size:
        i = bad
        g, r = lab_gpu[i], lab_ref[i]
        gap = D[i, g] - D[i, r]
        tolr = slack * (B[i, g] + B[i, r])
        ok = (gap <= tolr) | (~np.isfinite(D[i, r]) & ~np.isfinite(D[i, g]))
        assert ok.all(), (f"{(~ok).sum()} inadmissible labels, e.g. row {i[~ok][0]}: "
                          f"gap {gap[~ok][0]:.3e} > tol {tolr[~ok][0]:.3e}")
    return bad.size / max(1, len(lab_ref))


def check_admissible_rows(X, C, lab_gpu, lab_ref, work, dist, guard, slack=2.0):
    """check_labels_admissible for large n: D and B are formed only for the rows whose labels
    differ (each row's distances depend on that row alone). Returns the mismatch fraction."""
    lab_gpu = np.asarray(lab_gpu)
    lab_ref = np.asarray(lab_ref)
    bad = np.nonzero(lab_gpu != lab_ref)[0]
    if bad.size:
        D, B = distances_on_rounded_operands(np.asarray(X)[bad], C, work, dist, guard)
        check_labels_admissible(lab_gpu[bad], lab_ref[bad], D, B, slack)
    return bad.size / max(1, len(lab_ref))
