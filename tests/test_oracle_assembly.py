"""Pins P2-P4 for the oracle's element-loop assembly.

Independent references used here:
  * de Rham: gradients of vertex scalars (the +-1 edge incidence G built in this
    file) lie in the kernel of the curl-curl stiffness; rank K = #edges - #vertices + 1.
  * Kronecker closed forms of K, M and the load on an affine box,
    built from 1D matrices computed with scipy.interpolate.BSpline, not oracle.splines.
  * e_x is exactly representable, so a^T M a = sigma * volume.
"""
import math

import numpy as np
import pytest
from scipy.interpolate import BSpline

from oracle import assembly


def _space(p, d, lo=(0, 0, 0), hi=(1, 1, 1)):
    return assembly.PatchSpace(p, (d, d, d) if np.isscalar(d) else d, lo, hi)


def _gradient_matrix(n):
    tab = assembly.local_dof_table(n)
    nx, ny, nz = n
    G = np.zeros((len(tab), nx * ny * nz))
    for a, (c, i, j, k) in enumerate(tab):
        h = [i, j, k]
        h[c] += 1
        G[a, i + nx * (j + ny * k)] -= 1.0
        G[a, h[0] + nx * (h[1] + ny * h[2])] += 1.0
    return G


@pytest.mark.parametrize("p,d,nloc", [(1, 1, 12), (2, 2, 144), (1, 2, 54), (3, 8, 3630), (2, 4, 540), (3, 6, 1944)])
def test_counts(p, d, nloc):
    n = d + p
    assert assembly.n_local(n) == nloc == 3 * n * n * (n - 1)


@pytest.mark.parametrize("p,d,rank", [(1, 1, 5), (2, 2, 81), (3, 2, 176)])
def test_de_rham_and_rank(p, d, rank):
    sp = _space(p, d, (0, 0, 0), (0.5, 0.5, 0.5))
    K, M, _ = assembly.assemble_patch(sp, 1.0, 1.0, 0)
    assert np.max(np.abs(K - K.T)) <= 1e-13 * np.max(np.abs(K))
    G = _gradient_matrix(sp.n)
    assert np.max(np.abs(K @ G)) <= 1e-12 * np.max(np.abs(K))
    nv = np.prod(sp.n)
    assert np.linalg.matrix_rank(K, tol=1e-9 * np.max(np.abs(K))) == sp.nloc - nv + 1 == rank
    ev = np.linalg.eigvalsh(M)
    assert ev.min() > 0


def _oned(p, d, a, b):
    """1D matrices Mb, Md, C=[int D_i B_j'], and the source integrals, via scipy BSpline."""
    t = np.array([a] * (p + 1) + [a + (b - a) * e / d for e in range(1, d)] + [b] * (p + 1))
    n = d + p
    Bs = [BSpline(t, np.eye(n)[i], p) for i in range(n)]
    dBs = [B.derivative() for B in Bs]
    cD = np.eye(len(t) - p)
    Ds = [(lambda i: (lambda x: p / (t[i + p + 1] - t[i + 1]) * BSpline(t, cD[i + 1], p - 1)(x)))(i) for i in range(n - 1)]
    gp, gw = np.polynomial.legendre.leggauss(p + 1)
    X, Wt = [], []
    for e in range(d):
        lo, hi = a + (b - a) * e / d, a + (b - a) * (e + 1) / d
        X.append(0.5 * (lo + hi) + 0.5 * (hi - lo) * gp)
        Wt.append(0.5 * (hi - lo) * gw)
    X, Wt = np.concatenate(X), np.concatenate(Wt)
    Bv = np.array([B(X) for B in Bs])
    dBv = np.array([B(X) for B in dBs])
    Dv = np.array([D(X) for D in Ds])
    Mb = (Bv * Wt) @ Bv.T
    Md = (Dv * Wt) @ Dv.T
    Kb = (dBv * Wt) @ dBv.T
    C = (Dv * Wt) @ dBv.T
    pi = math.pi
    sD = (Dv * Wt) @ np.sin(pi * X)
    sB = (Bv * Wt) @ np.sin(pi * X)
    cB = (Bv * Wt) @ np.cos(pi * X)
    return dict(Mb=Mb, Md=Md, Kb=Kb, C=C, sD=sD, sB=sB, cB=cB)


def _k3(ax, ay, az):
    """Matrix with entry [(i,j,k),(i',j',k')] = ax[i,i'] ay[j,j'] az[k,k'] (i fastest)."""
    return np.kron(az, np.kron(ay, ax))


@pytest.mark.parametrize("p,d,lo,hi", [(1, 1, (0, 0, 0), (1, 1, 1)), (2, 2, (0.5, 0, 0.25), (1, 0.5, 0.75)),
                                       (3, 2, (0, 0, 0), (0.5, 0.5, 0.5)), (2, (1, 2, 3), (0, 0, 0), (0.5, 1, 1))])
def test_kronecker_closed_form(p, d, lo, hi):
    """element-loop K, M, j equal the sums of Kronecker products."""
    nu, sigma = 0.7, 3.0
    sp = _space(p, d, lo, hi)
    K, M, jS = assembly.assemble_patch(sp, nu, sigma, 1)
    o = [_oned(p, sp.elems[q], lo[q], hi[q]) for q in range(3)]
    X, Y, Z = o
    Kxx = _k3(X["Md"], Y["Mb"], Z["Kb"]) + _k3(X["Md"], Y["Kb"], Z["Mb"])
    Kyy = _k3(X["Kb"], Y["Md"], Z["Mb"]) + _k3(X["Mb"], Y["Md"], Z["Kb"])
    Kzz = _k3(X["Mb"], Y["Kb"], Z["Md"]) + _k3(X["Kb"], Y["Mb"], Z["Md"])
    Kxy = -_k3(X["C"], Y["C"].T, Z["Mb"])
    Kxz = -_k3(X["C"], Y["Mb"], Z["C"].T)
    Kyz = -_k3(X["Mb"], Y["C"], Z["C"].T)
    Kref = nu * np.block([[Kxx, Kxy, Kxz], [Kxy.T, Kyy, Kyz], [Kxz.T, Kyz.T, Kzz]])
    Mxx = _k3(X["Md"], Y["Mb"], Z["Mb"])
    Myy = _k3(X["Mb"], Y["Md"], Z["Mb"])
    Mzz = _k3(X["Mb"], Y["Mb"], Z["Md"])
    Z0 = np.zeros
    Mref = sigma * np.block([[Mxx, Z0((len(Mxx), len(Myy))), Z0((len(Mxx), len(Mzz)))],
                             [Z0((len(Myy), len(Mxx))), Myy, Z0((len(Myy), len(Mzz)))],
                             [Z0((len(Mzz), len(Mxx))), Z0((len(Mzz), len(Myy))), Mzz]])
    assert np.max(np.abs(K - Kref)) <= 1e-13 * np.max(np.abs(Kref))
    assert np.max(np.abs(M - Mref)) <= 1e-13 * np.max(np.abs(Mref))
    pi = math.pi
    jx = pi * np.kron(Z["sB"], np.kron(Y["cB"], X["sD"]))
    jy = -pi * np.kron(Z["sB"], np.kron(Y["sD"], X["cB"]))
    jz = np.zeros(len(Mzz))
    jref = np.concatenate([jx, jy, jz])
    assert np.max(np.abs(jS - jref)) <= 1e-13 * max(1.0, np.max(np.abs(jref)))


@pytest.mark.parametrize("p,d", [(1, 1), (2, 2), (3, 3)])
def test_mass_quadratic_form_ex(p, d):
    """e_x is representable: a_x[i,j,k] = (t_{i+p+1}-t_{i+1})/p, a_y = a_z = 0;
    then a^T M a = sigma * volume."""
    lo, hi = (0.25, 0.0, 0.5), (0.75, 0.25, 1.0)
    sp = _space(p, d, lo, hi)
    sigma = 2.5
    _, M, _ = assembly.assemble_patch(sp, 1.0, sigma, 0)
    t = sp.knots[0]
    a = np.zeros(sp.nloc)
    for (idx, (c, i, j, k)) in enumerate(assembly.local_dof_table(sp.n)):
        if c == 0:
            a[idx] = (t[i + p + 1] - t[i + 1]) / p
    vol = np.prod(np.array(hi) - np.array(lo))
    assert abs(a @ M @ a - sigma * vol) <= 1e-13


def test_linearity_in_nu_sigma():
    sp = _space(2, 1)
    K1, M1, j1 = assembly.assemble_patch(sp, 1.0, 1.0, 1)
    K2, M2, j2 = assembly.assemble_patch(sp, 2.0, 3.0, 1)
    assert np.allclose(K2, 2 * K1, rtol=0, atol=1e-14 * np.abs(K1).max())
    assert np.allclose(M2, 3 * M1, rtol=0, atol=1e-14 * np.abs(M1).max())
    assert np.array_equal(j1, j2)
    K0, M0, j0 = assembly.assemble_patch(sp, 1.0, 0.0, 0)
    assert not M0.any() and not j0.any()
