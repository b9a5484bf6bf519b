"""Pin P1: 1D spline spaces and Gauss rules of the oracle, checked
against closed forms and an independent library (scipy.interpolate.BSpline)."""
import numpy as np
import pytest
from scipy.interpolate import BSpline

from oracle import splines


@pytest.mark.parametrize("p,d,a,b", [(1, 2, 0.0, 1.0), (2, 4, 0.0, 1.0), (3, 8, 0.5, 1.0), (3, 6, 0.25, 0.375)])
def test_partition_of_unity_and_derivative_sum(p, d, a, b):
    t = splines.open_uniform_knots(p, d, a, b)
    assert len(t) - p - 1 == d + p
    rng = np.random.default_rng(1)
    for x in rng.uniform(a, b, 100):
        assert abs(splines.bsplines(t, p, x).sum() - 1.0) <= 1e-13
        assert abs(splines.bspline_derivs(t, p, x).sum()) <= 1e-11 * (d / (b - a))


@pytest.mark.parametrize("p,d", [(1, 2), (2, 4), (3, 8), (3, 3)])
def test_against_scipy_bspline(p, d):
    """B_i and B_i' agree with scipy's BSpline (an independent implementation)."""
    t = splines.open_uniform_knots(p, d, 0.0, 1.0)
    n = d + p
    rng = np.random.default_rng(2)
    xs = rng.uniform(0.0, 1.0, 100)
    for i in range(n):
        c = np.zeros(n)
        c[i] = 1.0
        bs = BSpline(t, c, p)
        dbs = bs.derivative()
        for x in xs:
            assert abs(splines.bsplines(t, p, x)[i] - bs(x)) <= 1e-13
            assert abs(splines.bspline_derivs(t, p, x)[i] - dbs(x)) <= 1e-11 * d


@pytest.mark.parametrize("p,d", [(1, 2), (2, 4), (3, 8)])
def test_dspline_identities(p, d):
    """Curry-Schoenberg: integral D_i = 1 and B_i' = D_{i-1} - D_i (D_{-1} = D_{n-1} = 0)."""
    t = splines.open_uniform_knots(p, d, 0.0, 1.0)
    n = d + p
    integ = np.zeros(n - 1)
    for (_, xs, ws) in splines.element_gauss_points(t, p, p + 1):
        for x, w in zip(xs, ws):
            integ += w * splines.dsplines(t, p, x)
    assert np.max(np.abs(integ - 1.0)) <= 1e-13
    rng = np.random.default_rng(3)
    for x in rng.uniform(0, 1, 100):
        D = np.concatenate([[0.0], splines.dsplines(t, p, x), [0.0]])
        assert np.max(np.abs(splines.bspline_derivs(t, p, x) - (D[:-1] - D[1:]))) <= 1e-12 * d


def test_dsplines_vs_scipy():
    p, d = 3, 5
    t = splines.open_uniform_knots(p, d, 0.0, 2.0)
    n = d + p
    for x in np.linspace(0.01, 1.99, 37):
        for i in range(n - 1):
            c = np.zeros(len(t) - p)
            c[i + 1] = 1.0
            ref = p / (t[i + p + 1] - t[i + 1]) * BSpline(t, c, p - 1)(x)
            assert abs(splines.dsplines(t, p, x)[i] - ref) <= 1e-13


@pytest.mark.parametrize("q", [1, 2, 3, 4, 5])
def test_gauss_exactness(q):
    gp, gw = splines.gauss_rule(q)
    assert abs(gw.sum() - 2.0) <= 1e-14
    for deg in range(2 * q):
        exact = 0.0 if deg % 2 else 2.0 / (deg + 1)
        assert abs(np.sum(gw * gp ** deg) - exact) <= 1e-14
    if q <= 4:
        deg = 2 * q
        assert abs(np.sum(gw * gp ** deg) - 2.0 / (deg + 1)) > 1e-6


def test_spec_examples():
    """SPEC S:L46-79 [TRIVIAL] examples."""
    assert list(splines.open_uniform_knots(1, 2, 0, 1)) == [0, 0, 0.5, 1, 1]
    t = splines.open_uniform_knots(1, 2, 0, 1)
    v = splines.bsplines(t, 1, 0.25)
    assert np.allclose(v, [0.5, 0.5, 0.0], atol=1e-15)
    assert len(splines.open_uniform_knots(3, 8, 0.5, 1.0)) - 4 == 11
    gp, gw = splines.gauss_rule(2)
    assert np.allclose(sorted(gp), [-1 / np.sqrt(3), 1 / np.sqrt(3)]) and np.allclose(gw, [1, 1])
    with pytest.raises(ValueError):
        splines.open_uniform_knots(0, 2, 0, 1)
    with pytest.raises(ValueError):
        splines.gauss_rule(0)
