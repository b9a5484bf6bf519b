"""ORACLE (test infrastructure only) — 1D spline spaces and Gauss rules.

Follows the IGA edge spaces of P:L74-77 (§2.2, "high-order, spline-based,
edge-element basis functions", GeoPDEs/Vazquez_2016aa) with the reading of
DESIGN.md R9 / SURVEY Q9: degree-(p-1) factors are Curry-Schoenberg D-splines
    D_i = p / (t_{i+p+1} - t_{i+1}) * B_{i+1,p-1},   i = 0..n-2,
so that B'_i = D_{i-1} - D_i and the discrete gradient is a +-1 incidence.
"""
from __future__ import annotations

import numpy as np


def open_uniform_knots(p: int, d: int, a: float, b: float) -> np.ndarray:
    """Open knot vector of degree p with d uniform elements on [a,b]:
    end knots repeated p+1 times, interior knots multiplicity 1 (dimension d+p)."""
    if p < 1 or d < 1 or not (a < b):
        raise ValueError("invalid spline space")
    inner = [a + (b - a) * e / d for e in range(1, d)]
    return np.array([a] * (p + 1) + inner + [b] * (p + 1), dtype=np.float64)


def cox_de_boor(t: np.ndarray, i: int, k: int, x: float) -> float:
    """B_{i,k}(x) on knot vector t by the Cox-de Boor recursion (0/0 := 0).
    Half-open support [t_i, t_{i+k+1}); evaluation points are interior."""
    if k == 0:
        return 1.0 if (t[i] <= x < t[i + 1]) else 0.0
    v = 0.0
    den1 = t[i + k] - t[i]
    if den1 > 0.0:
        v += (x - t[i]) / den1 * cox_de_boor(t, i, k - 1, x)
    den2 = t[i + k + 1] - t[i + 1]
    if den2 > 0.0:
        v += (t[i + k + 1] - x) / den2 * cox_de_boor(t, i + 1, k - 1, x)
    return v


def bsplines(t: np.ndarray, p: int, x: float) -> np.ndarray:
    """All n = len(t)-p-1 B-splines of degree p at x."""
    n = len(t) - p - 1
    return np.array([cox_de_boor(t, i, p, x) for i in range(n)])


def dsplines(t: np.ndarray, p: int, x: float) -> np.ndarray:
    """All n-1 Curry-Schoenberg D-splines D_i = p/(t_{i+p+1}-t_{i+1}) B_{i+1,p-1}(x)."""
    n = len(t) - p - 1
    out = np.zeros(n - 1)
    for i in range(n - 1):
        out[i] = p / (t[i + p + 1] - t[i + 1]) * cox_de_boor(t, i + 1, p - 1, x)
    return out


def bspline_derivs(t: np.ndarray, p: int, x: float) -> np.ndarray:
    """B'_i = p/(t_{i+p}-t_i) B_{i,p-1} - p/(t_{i+p+1}-t_{i+1}) B_{i+1,p-1}
    (standard derivative formula; equals D_{i-1} - D_i)."""
    n = len(t) - p - 1
    out = np.zeros(n)
    for i in range(n):
        v = 0.0
        if t[i + p] - t[i] > 0:
            v += p / (t[i + p] - t[i]) * cox_de_boor(t, i, p - 1, x)
        if t[i + p + 1] - t[i + 1] > 0:
            v -= p / (t[i + p + 1] - t[i + 1]) * cox_de_boor(t, i + 1, p - 1, x)
        out[i] = v
    return out


def gauss_rule(q: int):
    """q-point Gauss-Legendre rule on [-1,1] (numpy.polynomial.legendre.leggauss)."""
    if q < 1:
        raise ValueError("q >= 1")
    return np.polynomial.legendre.leggauss(q)


def element_gauss_points(t: np.ndarray, p: int, q: int):
    """Physical Gauss points/weights per element: returns list of (e, xs, ws)."""
    gp, gw = gauss_rule(q)
    brk = np.unique(t)
    out = []
    for e in range(len(brk) - 1):
        a, b = brk[e], brk[e + 1]
        xs = 0.5 * (a + b) + 0.5 * (b - a) * gp
        ws = 0.5 * (b - a) * gw
        out.append((e, xs, ws))
    return out
