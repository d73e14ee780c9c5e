"""Pins for O11: Thm 5.3's centre-update precision bound (eq:center-update-prec,
PAPER.md:487-493) recorded per iteration by the oracle's fit, against hand-derived values."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.filterwarnings("ignore")


def test_one_dimension_hand_value():
    """X = {0, 2}, k = 1, c0 = 0.5: mu^ = 1, c^ - mu^ = -0.5: 0.25 / (2 * 0.5 * 1) = 0.25; the
    next iteration does not move (+inf)."""
    r = oracle.fit(np.array([[0.0], [2.0]]), np.array([[0.5]]), work="fp64", dist="fp64",
                   max_iter=2, tol=-1.0)
    assert r["u_bound_t"][0] == 0.25
    assert np.isinf(r["u_bound_t"][1])


@pytest.mark.parametrize("c0,want", [((1.0, 1.0), 0.25), ((3.0, 3.0), 5.0 / 8.0)])
def test_two_dimensions_hand_values(c0, want):
    """X = the corners of [0, 4] x [0, 2], mean (2, 1).
    c0 = (1, 1): diff (-1, 0), num 1, den |-1| * 2 = 2 -> 1 / 4.
    c0 = (3, 3): diff (1, 2), num 5, den 1 * 2 + 2 * 1 = 4 -> 5 / 8."""
    X = np.array([[0.0, 0.0], [4.0, 0.0], [0.0, 2.0], [4.0, 2.0]])
    r = oracle.fit(X, np.array([c0]), work="fp64", dist="fp64", max_iter=1, tol=-1.0)
    assert r["u_bound_t"][0] == want


def test_min_over_clusters():
    """Two far-apart groups, each with its own centre moving by a known vector: the bound is the
    smaller per-cluster value. Group A = {(0,0), (4,0), (0,2), (4,2)} from (1,1) -> 1/4;
    group B = A + (100, 0) from (103, 3): diff (1, 2), den 1 * 102 + 2 * 1 = 104 -> 5 / 208."""
    A = np.array([[0.0, 0.0], [4.0, 0.0], [0.0, 2.0], [4.0, 2.0]])
    X = np.vstack([A, A + [100.0, 0.0]])
    C0 = np.array([[1.0, 1.0], [103.0, 3.0]])
    r = oracle.fit(X, C0, work="fp64", dist="fp64", max_iter=1, tol=-1.0)
    assert r["u_bound_t"][0] == min(0.25, 5.0 / 208.0)


def test_scale_invariance():
    """Numerator and denominator are both quadratic in the data: scaling by 8 (exact) leaves the
    bound unchanged."""
    rng = np.random.default_rng(1)
    X = rng.normal(size=(300, 4))
    C0 = X[:5].copy()
    a = oracle.fit(X, C0, work="fp64", dist="fp64", max_iter=4, tol=-1.0)["u_bound_t"]
    b = oracle.fit(8 * X, 8 * C0, work="fp64", dist="fp64", max_iter=4, tol=-1.0)["u_bound_t"]
    np.testing.assert_array_equal(a, b)
