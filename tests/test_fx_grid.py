"""Host-side model of DESIGN.md reading R9's per-feature grid (k_update.cu `fx_q`): with
2^e > max |x|, c1 = 1.5 * 2^(e+1), c2 = 1.5 * 2^(e-22), the fp32 operations
t1 = RN(x + c1), r = x - (t1 - c1), t2 = RN(r + c2) and the bit-pattern differences
i1 = bits(t1) - bits(c1), i2 = bits(t2) - bits(c2) put x on the grid g = 2^(e-45) as
q = i1 * 2^23 + i2 with |x - q g| <= g / 2 and |i1|, |i2| <= 2^22 (so 256-row piece sums fit in
int32 and cluster totals in int64). Checked here in numpy float32 (IEEE round-to-nearest) against
exact rational arithmetic — the claims the exact-update design rests on. Test infrastructure; no
GPU."""
from fractions import Fraction

import numpy as np
import pytest


def fx_q(x, e):
    x = np.float32(x)
    c1 = np.float32(1.5 * 2.0 ** (e + 1))
    c2 = np.float32(1.5 * 2.0 ** (e - 22))
    with np.errstate(over="ignore"):
        t1 = np.float32(x + c1)
        r = np.float32(x - np.float32(t1 - c1))
        t2 = np.float32(r + c2)
    bits = lambda v: int(np.array(v, np.float32).view(np.int32))
    return bits(t1) - bits(c1), bits(t2) - bits(c2)


def frexp_e(amax):
    return int(np.frexp(np.float64(amax))[1])      # amax < 2^e


@pytest.mark.parametrize("amax", [1.0, 3.7, 1e-3, 6.5e4, 1e-20, 2.0 ** 60])
def test_grid_value_within_half_a_step(amax):
    e = frexp_e(np.float32(amax))
    rng = np.random.default_rng(int(abs(np.log2(amax))) + 7)
    xs = list((rng.uniform(-1, 1, 4000) * amax).astype(np.float32))
    # magnitudes spread down to the subnormals, exact edges and ties
    xs += list((rng.uniform(-1, 1, 2000) * amax * 2.0 ** -rng.integers(0, 60, 2000)).astype(np.float32))
    xs += [np.float32(amax), np.float32(-amax), np.float32(0.0), np.float32(-0.0),
           np.nextafter(np.float32(2.0 ** e), np.float32(0)), np.float32(2.0 ** (e - 23)),
           np.float32(1.5 * 2.0 ** (e - 45)), np.float32(np.finfo(np.float32).smallest_subnormal)]
    g = Fraction(2) ** (e - 45)
    for x in xs:
        if abs(float(x)) >= 2.0 ** e:
            continue
        i1, i2 = fx_q(x, e)
        assert abs(i1) <= 2 ** 22 and abs(i2) <= 2 ** 22, (x, i1, i2)
        q = i1 * 2 ** 23 + i2
        assert abs(Fraction(float(x)) - q * g) <= g / 2, (x, i1, i2)


def test_grid_is_a_function_of_x_only():
    """The integer pair depends on x and the feature's e alone, so sums over any set of rows are
    order- and history-independent: incremental add/subtract reproduces the full sum exactly."""
    rng = np.random.default_rng(3)
    amax = 5.0
    e = frexp_e(np.float32(amax))
    x = (rng.standard_normal(3000) * 1.5).astype(np.float32)
    x = np.clip(x, -4.99, 4.99).astype(np.float32)
    q = np.array([i1 * 2 ** 23 + i2 for i1, i2 in (fx_q(v, e) for v in x)], dtype=object)
    members = rng.random(3000) < 0.5
    full = sum(q[members])
    moved_in = rng.random(3000) < 0.05
    new_members = members ^ moved_in
    incremental = full + sum(q[moved_in & ~members]) - sum(q[moved_in & members])
    assert incremental == sum(q[new_members])
