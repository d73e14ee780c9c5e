"""Pins for oracle O0 (round_to): Table 1 constants, exhaustive code-point / midpoint checks and
cross-checks against library casts that round ONCE (numpy float64->float16/float32, torch
float32->bfloat16/float8_e5m2). SURVEY.md §8c.3 row "O0 rounding"."""
import json
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))


def _sig3(a, b):
    return abs(a - b) <= 0.006 * abs(b)   # "to 3 s.f." as printed in Table 1


@pytest.mark.parametrize("fmt", ["e5m2", "fp16", "fp32", "fp64"])
def test_table1_constants(fmt):
    """Table 1: u = 2^-t, x_min = 2^e_min, x_max = 2^e_max (2 - 2^(1-t))."""
    t, emin, emax = oracle.format_params(fmt)
    g = GOLD[fmt]
    assert (t, emin, emax) == (g["t"], g["e_min"], g["e_max"])
    assert _sig3(2.0 ** -t, g["u"])
    assert _sig3(2.0 ** emin, g["x_min"])
    xmax = 2.0 ** emax * (2 - 2.0 ** (1 - t))
    assert _sig3(xmax, g["x_max"])
    if fmt != "fp64":
        # x_max is representable, and the next binade overflows
        assert oracle.round_to(fmt, [xmax])[0] == xmax


def _all_finite(fmt):
    if fmt == "fp16":
        v = np.arange(1 << 16, dtype=np.uint16).view(np.float16).astype(np.float64)
    elif fmt == "bf16":
        v = (np.arange(1 << 16, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)
    else:  # e5m2: the top byte of an fp16 (same exponent layout, 2 mantissa bits)
        v = (np.arange(256, dtype=np.uint16) << 8).view(np.float16).astype(np.float64)
    v = v[np.isfinite(v)]
    return np.unique(v)


@pytest.mark.parametrize("fmt", ["fp16", "bf16", "e5m2"])
def test_exhaustive_codes_and_midpoints(fmt):
    v = _all_finite(fmt)
    # every code point is a fixed point
    assert np.array_equal(oracle.round_to(fmt, v), v)
    # midpoints between consecutive values go to the neighbour with an even significand
    lo, hi = v[:-1], v[1:]
    mid = (lo + hi) / 2          # exact in fp64
    r = oracle.round_to(fmt, mid)
    t, emin, emax = oracle.format_params(fmt)

    def even(x):
        x = np.abs(x)
        e = np.maximum(np.floor(np.log2(np.where(x > 0, x, 1.0))), emin)
        q = 2.0 ** (e - (t - 1))
        return (np.rint(x / q) % 2) == 0

    want = np.where(even(lo), lo, hi)
    assert np.array_equal(r, want)
    # just off the midpoint goes to the nearer neighbour
    eps = np.abs(mid) * 2.0 ** -45 + 2.0 ** -1070
    assert np.array_equal(oracle.round_to(fmt, mid - eps), lo)
    assert np.array_equal(oracle.round_to(fmt, mid + eps), hi)


def test_fp16_matches_numpy_single_rounding():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(200000) * 10.0 ** rng.integers(-9, 6, 200000),
                        rng.uniform(-7e4, 7e4, 20000)])
    with np.errstate(over="ignore"):
        want = x.astype(np.float16).astype(np.float64)
    assert np.array_equal(oracle.round_to("fp16", x), want)


def test_fp32_matches_numpy_single_rounding():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(200000) * 10.0 ** rng.integers(-40, 38, 200000)
    with np.errstate(over="ignore"):
        want = x.astype(np.float32).astype(np.float64)
    assert np.array_equal(oracle.round_to("fp32", x), want)


@pytest.mark.parametrize("fmt,tdt", [("bf16", torch.bfloat16), ("e5m2", torch.float8_e5m2),
                                     ("fp16", torch.float16)])
def test_matches_torch_from_float32(fmt, tdt):
    """torch casts round once only from float32 inputs."""
    rng = np.random.default_rng(2)
    x = (rng.standard_normal(300000) * 10.0 ** rng.integers(-8, 5, 300000)).astype(np.float32)
    mids = _all_finite(fmt)
    mids = ((mids[:-1] + mids[1:]) / 2).astype(np.float32)   # exact in fp32 for these formats
    x = np.concatenate([x, mids]).astype(np.float32)
    want = torch.from_numpy(x).to(tdt).to(torch.float64).numpy()
    got = oracle.round_to(fmt, x.astype(np.float64))
    if fmt == "e5m2":
        # torch's float8_e5m2 cast saturates nothing but maps overflow to inf as well
        pass
    assert np.array_equal(np.nan_to_num(got, nan=7.0), np.nan_to_num(want, nan=7.0))


def test_overflow_thresholds_and_specials():
    """Reading Z6/Z7: +-inf iff |v| >= 2^e_max (2 - 2^-t); NaN passes; -0 kept."""
    r = oracle.round_to
    assert r("fp16", [65519.99])[0] == 65504.0 and np.isinf(r("fp16", [65520.0])[0])
    assert r("e5m2", [61439.0])[0] == 57344.0 and np.isinf(r("e5m2", [61440.0])[0])
    assert r("e5m2", [-61440.0])[0] == -np.inf
    bmax = 2.0 ** 127 * (2 - 2.0 ** -7)
    assert r("bf16", [2.0 ** 127 * (2 - 2.0 ** -8) * (1 - 2.0 ** -50)])[0] == bmax
    assert np.isinf(r("bf16", [2.0 ** 127 * (2 - 2.0 ** -8)])[0])
    assert np.isnan(r("fp16", [np.nan])[0])
    z = r("fp16", [-2.0 ** -26])[0]
    assert z == 0.0 and np.signbit(z)
    # subnormal boundaries
    assert r("fp16", [2.0 ** -24])[0] == 2.0 ** -24
    assert r("fp16", [2.0 ** -25])[0] == 0.0                  # tie -> even (0)
    assert r("fp16", [1.5 * 2.0 ** -24])[0] == 2.0 ** -23     # tie -> even (2 quanta)
    assert r("e5m2", [2.0 ** -16])[0] == 2.0 ** -16
    assert r("e5m2", [1.5 * 2.0 ** -16])[0] == 2.0 ** -15


def test_single_rounding_not_double():
    """One rounding from fp64 (SURVEY §7 hard part 4): 1.125 + 2^-40 -> E5M2 1.25 (a double
    rounding through fp32 would give 1.0); 1 + 2^-8 + 2^-40 -> bf16 1 + 2^-7."""
    assert oracle.round_to("e5m2", [1.125 + 2.0 ** -40])[0] == 1.25
    assert oracle.round_to("bf16", [1 + 2.0 ** -8 + 2.0 ** -40])[0] == 1 + 2.0 ** -7


def test_relative_error_bound():
    """eq:fpmodel: |fl(x) - x| <= u |x| for normal-range results."""
    rng = np.random.default_rng(3)
    for fmt in ["fp16", "bf16", "e5m2", "fp32"]:
        t, emin, emax = oracle.format_params(fmt)
        x = rng.uniform(1, 2, 100000) * 2.0 ** rng.integers(emin, emax, 100000)
        x = x[np.abs(x) < 2.0 ** emax]
        err = np.abs(oracle.round_to(fmt, x) - x)
        assert np.all(err <= 2.0 ** -t * np.abs(x))
