"""ORACLE (test infrastructure only) — element-loop Gauss-quadrature assembly.

Definitions followed (§2.2):
    (K_i)_{jk} = a_i(w_k, w_j) = <nu curl w_k, curl w_j>          (a_i at P:L68)
    (M_C)_{jk} = <sigma w_k, w_j>   (printed <sigma w_k, w_k> at P:L85; read as
                                      <sigma w_k, w_j>, R10 / SURVEY Q10)
    (j_i)_j   = <J_i, w_j>
Quadrature: p+1 Gauss points per direction per element (R8 / SURVEY Q8).
Edge basis:
    x-comp  D_i(x) B_j(y) B_k(z) e_x,  y-comp  B_i D_j B_k e_y,  z-comp  B_i B_j D_k e_z
Local numbering: component-major, then k slowest, j, i fastest.
Geometry: identity map on an axis-aligned box (SPEC design decision S:L104).
"""
from __future__ import annotations

import math
import numpy as np

from . import splines


def _nvec(n):
    return (n, n, n) if np.isscalar(n) else tuple(int(v) for v in n)


def comp_dims(n, c: int):
    """(nx, ny, nz) index ranges of component c: n_d - 1 along direction c, n_d elsewhere
    (n_d = elements_d + p B-splines per direction)."""
    d = list(_nvec(n))
    d[c] -= 1
    return tuple(d)


def n_local(n) -> int:
    return sum(int(np.prod(comp_dims(n, c))) for c in range(3))


def local_index(n, c: int, i: int, j: int, k: int) -> int:
    off = sum(int(np.prod(comp_dims(n, cc))) for cc in range(c))
    dx, dy, _ = comp_dims(n, c)
    return off + i + dx * (j + dy * k)


def local_dof_table(n) -> np.ndarray:
    """(n_loc, 4) array of (component, i, j, k) in local order."""
    rows = []
    for c in range(3):
        dx, dy, dz = comp_dims(n, c)
        for k in range(dz):
            for j in range(dy):
                for i in range(dx):
                    rows.append((c, i, j, k))
    return np.array(rows, dtype=np.int64)


def source_field(kind: int, x, y, z):
    """Spatial part S(x) of J = phi(t) S(x).
    kind 1: S = curl(0,0,psi), psi = sin(pi x) sin(pi y) sin(pi z)   (BJ configs)
    kind 2: S = (sin pi y sin pi z, sin pi x sin pi z, sin pi x sin pi y)  (MMS)
    kind 3: S = (sin x cos y cos z, -2 cos x sin y cos z, cos x cos y sin z)  (the paper's
            prescribed solution A = e^-t S; oracle/paper_mms.py)"""
    pi = math.pi
    if kind == 1:
        return (pi * np.sin(pi * x) * np.cos(pi * y) * np.sin(pi * z),
                -pi * np.cos(pi * x) * np.sin(pi * y) * np.sin(pi * z),
                0.0 * x)
    if kind == 2:
        return (np.sin(pi * y) * np.sin(pi * z), np.sin(pi * x) * np.sin(pi * z), np.sin(pi * x) * np.sin(pi * y))
    if kind == 3:
        return (np.sin(x) * np.cos(y) * np.cos(z), -2.0 * np.cos(x) * np.sin(y) * np.cos(z),
                np.cos(x) * np.cos(y) * np.sin(z))
    return (0.0 * x, 0.0 * x, 0.0 * x)


def sinpi(x: float) -> float:
    """sin(pi x) with exact argument reduction (R19): x mod 2 and the
    reflections r -> r-1, r -> 1-r are exact in binary floating point (Sterbenz), so
    sin(pi x) is exactly 0 at integers and +-1 at half-integers, as the definition is.
    math.sin(math.pi * x) instead rounds pi*x first (sin(2 pi * 1.0) = -2.4e-16)."""
    r = math.fmod(x, 2.0)
    if r < 0.0:
        r += 2.0
    sign = 1.0
    if r >= 1.0:
        r -= 1.0
        sign = -1.0
    if r > 0.5:
        r = 1.0 - r
    return sign * math.sin(math.pi * r)


def source_time_factor(kind: int, t: float, nu: float, sigma: float, params=()) -> float:
    """phi_s(t) with J = phi_s(t) S(x) on patch s (params: an amplitude, and for kind 1 a
    frequency; defaults 1).
    kind 1: amp sin(2 pi freq t) (evaluated as sinpi(2 freq t)).
    kind 2: amp [2 pi^2 nu (1-e^-t) + sigma e^-t] (curl curl S = 2 pi^2 S).
    kind 3: amp e^-t (3 nu - sigma): J = nu curl curl A + sigma dA/dt for A = e^-t S,
            curl curl S = 3 S."""
    amp = params[0] if len(params) >= 1 else 1.0
    if kind == 1:
        freq = params[1] if len(params) >= 2 else 1.0
        return amp * sinpi(2.0 * freq * t)
    if kind == 2:
        return amp * (2.0 * math.pi ** 2 * nu * (1.0 - math.exp(-t)) + sigma * math.exp(-t))
    if kind == 3:
        return amp * math.exp(-t) * (3.0 * nu - sigma)
    return 0.0


class PatchSpace:
    """Curl-conforming spline space on one box patch (degrees (p-1,p,p) cyclic)."""

    def __init__(self, p: int, elems, lo, hi, nq: int | None = None):
        self.p = p
        self.elems = tuple(int(e) for e in elems)
        self.lo = tuple(float(v) for v in lo)
        self.hi = tuple(float(v) for v in hi)
        self.n = tuple(e + p for e in self.elems)
        self.nloc = n_local(self.n)
        self.nq = p + 1 if nq is None else nq
        self.knots = [splines.open_uniform_knots(p, self.elems[d], self.lo[d], self.hi[d]) for d in range(3)]
        # per direction, per element: (xs, ws, B[q,:], D[q,:], dB[q,:])
        self.tab = []
        for d in range(3):
            t = self.knots[d]
            per_el = []
            for (e, xs, ws) in splines.element_gauss_points(t, p, self.nq):
                B = np.array([splines.bsplines(t, p, x) for x in xs])
                D = np.array([splines.dsplines(t, p, x) for x in xs])
                dB = np.array([splines.bspline_derivs(t, p, x) for x in xs])
                per_el.append((xs, ws, B, D, dB))
            self.tab.append(per_el)

    def element_values(self, ex, ey, ez):
        """Active local DOFs of element (ex,ey,ez), basis values val[q,a,3] and curls
        cur[q,a,3] at the tensor Gauss points, physical points (X,Y,Z) and weights W."""
        p, n = self.p, self.n
        tx, ty, tz = self.tab[0][ex], self.tab[1][ey], self.tab[2][ez]
        nq = self.nq
        # 3D point ordering: qx fastest
        X = np.tile(tx[0], nq * nq)
        Y = np.tile(np.repeat(ty[0], nq), nq)
        Z = np.repeat(tz[0], nq * nq)
        W = np.tile(tx[1], nq * nq) * np.tile(np.repeat(ty[1], nq), nq) * np.repeat(tz[1], nq * nq)
        Bx, Dx, dBx = tx[2], tx[3], tx[4]
        By, Dy, dBy = ty[2], ty[3], ty[4]
        Bz, Dz, dBz = tz[2], tz[3], tz[4]
        e3 = (ex, ey, ez)
        ids, vals, curls = [], [], []
        for c in range(3):
            rng = []
            for d in range(3):
                if d == c:
                    rng.append(range(e3[d], e3[d] + p))        # D-spline actives
                else:
                    rng.append(range(e3[d], e3[d] + p + 1))    # B-spline actives
            for k in rng[2]:
                for j in rng[1]:
                    for i in rng[0]:
                        ids.append(local_index(n, c, i, j, k))
                        v = np.zeros((nq ** 3, 3))
                        cu = np.zeros((nq ** 3, 3))
                        if c == 0:
                            fx, fy, fz = Dx[:, i], By[:, j], Bz[:, k]
                            gy, gz = dBy[:, j], dBz[:, k]
                            v[:, 0] = _t3(fx, fy, fz)
                            cu[:, 1] = _t3(fx, fy, gz)           # d/dz of w_x
                            cu[:, 2] = -_t3(fx, gy, fz)          # -d/dy of w_x
                        elif c == 1:
                            fx, fy, fz = Bx[:, i], Dy[:, j], Bz[:, k]
                            gx, gz = dBx[:, i], dBz[:, k]
                            v[:, 1] = _t3(fx, fy, fz)
                            cu[:, 0] = -_t3(fx, fy, gz)          # -d/dz of w_y
                            cu[:, 2] = _t3(gx, fy, fz)           # d/dx of w_y
                        else:
                            fx, fy, fz = Bx[:, i], By[:, j], Dz[:, k]
                            gx, gy = dBx[:, i], dBy[:, j]
                            v[:, 2] = _t3(fx, fy, fz)
                            cu[:, 0] = _t3(fx, gy, fz)           # d/dy of w_z
                            cu[:, 1] = -_t3(gx, fy, fz)          # -d/dx of w_z
                        vals.append(v)
                        curls.append(cu)
        val = np.stack(vals, axis=1)
        cur = np.stack(curls, axis=1)
        return np.array(ids), val, cur, (X, Y, Z), W

    def elements(self):
        for ez in range(self.elems[2]):
            for ey in range(self.elems[1]):
                for ex in range(self.elems[0]):
                    yield ex, ey, ez


def _t3(fx, fy, fz):
    """Tensor product over the (qx fastest) 3D Gauss grid of three 1D value columns."""
    nq = len(fx)
    return (np.tile(fx, nq * nq) * np.tile(np.repeat(fy, nq), nq) * np.repeat(fz, nq * nq))


def assemble_patch(space: PatchSpace, nu: float, sigma: float, source_kind: int):
    """Element loop: K = nu <curl w_k, curl w_j>, M = sigma <w_k, w_j>, jS = <S, w_j>."""
    N = space.nloc
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    jS = np.zeros(N)
    for (ex, ey, ez) in space.elements():
        ids, val, cur, (X, Y, Z), W = space.element_values(ex, ey, ez)
        Ke = np.einsum("q,qac,qbc->ab", W, cur, cur)
        Me = np.einsum("q,qac,qbc->ab", W, val, val)
        Sx, Sy, Sz = source_field(source_kind, X, Y, Z)
        S = np.stack([Sx, Sy, Sz], axis=1)
        je = np.einsum("q,qc,qac->a", W, S, val)
        K[np.ix_(ids, ids)] += nu * Ke
        M[np.ix_(ids, ids)] += sigma * Me
        jS[ids] += je
    return K, M, jS
