"""ORACLE (test infrastructure only) — the paper's own experiment (§4).

P:L158-163 (§4, eq. problem): prescribed solution on Omega = (0,1)^3, t in (0,1),
    A = e^{-t} S(x),  S = (sin x cos y cos z, -2 cos x sin y cos z, cos x cos y sin z),
    B = curl A = e^{-t} (-3 cos x sin y sin z, 0, 3 sin x sin y cos z),
    E_C = -dA/dt = e^{-t} S  (only in Omega_C);
div S = 0 and curl curl S = -Laplace S = 3 S, so the source of eq. formA* is
    J = nu curl curl A + sigma dA/dt = e^{-t} (3 nu - sigma) S.
"From (problem), we derive appropriate homogenized boundary, source and initial terms"
 and "Inhomogeneous boundary conditions can be incorporated by using a classical
homogenization technique": the boundary data is the tangential trace of A. Reading
(R21): the Dirichlet DOFs a_D(t) and the initial coefficients a(0) are those of
the commuting spline projection Pi_h A (interpolation at Greville points
in the B-spline directions, histopolation on the Greville intervals in the D-spline
direction), so a_D(t) = e^{-t} (Pi_h S)_D; a shared DOF gets the same value from every
patch (its value depends only on data on that DOF's own edge line / face).
Errors, with the L2 norms by (p+1)-point Gauss quadrature per element:
    eps_E^2 = dt sum_l || E_C(t_l) + (A_h(t_l) - A_h(t_{l-1}))/dt ||^2_{L2(Omega_C)}
    eps_B^2 = max_l ||B(t_l) - curl A_h(t_l)||^2_{L2(Omega)} + dt sum_l ||B(t_l) - curl A_h(t_l)||^2.
"""
from __future__ import annotations

import math

import numpy as np

from . import assembly, splines

SOURCE_PAPER = 3


def S(x, y, z):
    return (np.sin(x) * np.cos(y) * np.cos(z), -2.0 * np.cos(x) * np.sin(y) * np.cos(z),
            np.cos(x) * np.cos(y) * np.sin(z))


def curlS(x, y, z):
    return (-3.0 * np.cos(x) * np.sin(y) * np.sin(z), 0.0 * x, 3.0 * np.sin(x) * np.sin(y) * np.cos(z))


def greville(t, p):
    """Greville abscissae of the degree-p B-splines on knot vector t."""
    n = len(t) - p - 1
    return np.array([sum(t[i + 1:i + p + 1]) / p for i in range(n)])


def _bsplines_closed(t, p, x):
    """All B-splines at x with the right end point included (B_{n-1}(b) = 1 for open knots)."""
    if x >= t[-1]:
        out = np.zeros(len(t) - p - 1)
        out[-1] = 1.0
        return out
    return splines.bsplines(t, p, x)


def _interval_rule(t, a, b, nq):
    """Gauss points/weights on [a, b], split at the knots inside (exact for piecewise
    polynomials of degree <= 2 nq - 1 on the knot spans)."""
    cuts = [a] + [k for k in np.unique(t) if a < k < b] + [b]
    gp, gw = splines.gauss_rule(nq)
    xs, ws = [], []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        xs.extend(0.5 * (lo + hi) + 0.5 * (hi - lo) * gp)
        ws.extend(0.5 * (hi - lo) * gw)
    return np.array(xs), np.array(ws)


def projection_matrices(t, p, nq):
    """Collocation I[i, j] = B_j(xi_i) at the Greville points xi and histopolation
    H[a, j] = int_{xi_a}^{xi_{a+1}} D_j dx, plus the quadrature of each Greville interval."""
    xi = greville(t, p)
    n = len(xi)
    Icol = np.array([_bsplines_closed(t, p, x) for x in xi])
    rules = [_interval_rule(t, xi[a], xi[a + 1], nq) for a in range(n - 1)]
    H = np.zeros((n - 1, n - 1))
    for a, (xs, ws) in enumerate(rules):
        for x, w in zip(xs, ws):
            H[a] += w * splines.dsplines(t, p, x)
    return xi, Icol, H, rules


def commuting_projection(space, field, nq=None):
    """Local coefficient vector (local order, all n_loc DOFs) of Pi_h g on one box patch:
    component c solves (H_c along c) x (I along the other two directions) C_c = G_c with
    G_c[k, j, i] = int over the Greville interval along c of g_c at the Greville points of the
    other directions (R21)."""
    p = space.p
    nq = p + 3 if nq is None else nq
    mats = [projection_matrices(space.knots[d], p, nq) for d in range(3)]
    out = []
    for c in range(3):
        # per direction: point lists (Greville) or (interval rules) for direction c
        axes = []
        for d in range(3):
            xi, Icol, H, rules = mats[d]
            axes.append(rules if d == c else xi)
        dims = assembly.comp_dims(space.n, c)
        G = np.zeros((dims[2], dims[1], dims[0]))
        for k in range(dims[2]):
            for j in range(dims[1]):
                for i in range(dims[0]):
                    idx = (i, j, k)
                    xs, ws = axes[c][idx[c]]
                    pts = [None, None, None]
                    for d in range(3):
                        pts[d] = xs if d == c else np.full_like(xs, axes[d][idx[d]])
                    G[k, j, i] = float(np.sum(ws * field(*pts)[c]))
        # solve along x (axis 2), y (axis 1), z (axis 0)
        C = G
        for d, ax in ((0, 2), (1, 1), (2, 0)):
            M = mats[d][2] if d == c else mats[d][1]
            C = np.moveaxis(np.linalg.solve(M, np.moveaxis(C, ax, 0).reshape(M.shape[0], -1)).reshape(
                np.moveaxis(C, ax, 0).shape), 0, ax)
        out.append(C.reshape(-1))
    return np.concatenate(out)


class ErrorTracker:
    """Accumulates eps_B, eps_E over the steps of an oracle run."""

    def __init__(self, oracle):
        self.o = oracle
        pr = oracle.prob
        self.sps = [assembly.PatchSpace(pr.p, pr.elems, *oracle.patch_box(s)) for s in range(pr.n_patches)]
        self.B2_max = 0.0
        self.B2_sum = 0.0
        self.E2_sum = 0.0
        self.per_step = []

    def after_step(self, a_old):
        o, pr = self.o, self.o.prob
        t = o.ell * o.dt
        eB = eE = 0.0
        for s, sp in enumerate(self.sps):
            for el in sp.elements():
                ids, val, cur, (X, Y, Z), W = sp.element_values(*el)
                Bh = np.einsum("a,qac->qc", o.a[s][ids], cur)
                Be = math.exp(-t) * np.stack(curlS(X, Y, Z), 1)
                eB += float(np.sum(W[:, None] * (Be - Bh) ** 2))
                if pr.sigma[s] > 0:
                    dA = np.einsum("a,qac->qc", (o.a[s][ids] - a_old[s][ids]) / o.dt, val)
                    Ee = math.exp(-t) * np.stack(S(X, Y, Z), 1)
                    eE += float(np.sum(W[:, None] * (Ee + dA) ** 2))
        self.B2_max = max(self.B2_max, eB)
        self.B2_sum += o.dt * eB
        self.E2_sum += o.dt * eE
        self.per_step.append((eB, eE))

    @property
    def eps_B(self):
        return math.sqrt(self.B2_max + self.B2_sum)

    @property
    def eps_E(self):
        return math.sqrt(self.E2_sum)
