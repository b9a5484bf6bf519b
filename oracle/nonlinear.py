"""ORACLE (test infrastructure only) — nonlinear reluctivity nu(|B|) with Newton's method
(SURVEY §8(f) f4). Only tests/, __graft_entry__.smoke() and bench.py's cpu legs may import it.

Paper: "we focus on linear material, but note that nonlinear behavior can be modeled as a
simple extension of the approaches discussed in this treatise" (§2). The paper gives
no material law and no linearisation; the readings used here are DESIGN.md R25:

  * material law (Brauer): nu(|B|) = k1 exp(k2 |B|^2) + k3 per nonlinear patch (k1, k2 >= 0,
    k3 > 0), so nu > 0 and the magnetic field H = nu(|B|) B is strictly monotone in B;
    patches with (k1, k2, k3) = 0 keep their constant nu_s.
  * weak form of curl(nu(|curl A|) curl A) (P:L42 eq. formA* with nu = nu(|B|)) per patch:
        R_s(a) = K_s(a) a + (sigma_s/dt) M_s (a - a^l) - j_s^(l+1),
        K_s(a)_jk = <nu(|B|) curl w_k, curl w_j>,  B = curl A_h = sum_k a_k curl w_k
    (the implicit-Euler step of P:L133 with K evaluated at the new level).
  * Jacobian (Gateaux derivative of K(a) a):
        J_s(a) = Kt_s(a) + (sigma_s/dt) M_s,
        Kt_s(a)_jk = < (nu I + 2 nu'(|B|^2) B B^T) curl w_k, curl w_j >,  nu' = d nu / d(|B|^2)
    which is SPD on the gauged space because nu + 2 nu' |B|^2 >= nu > 0 (monotone H(B)).
  * Newton per time step from a_0 = a^l, written for the IETI-DP solve as
        J(a_k) a_{k+1} = J(a_k) a_k - R(a_k) = (Kt(a_k) - K(a_k)) a_k + (sigma/dt) M a^l + j^(l+1)
    (the same Newton iterate, a_{k+1} = a_k - J^-1 R(a_k), with the right-hand side expanded;
    the patches' torn residuals sum to the glued one), each linear solve the
    linear method of oracle/ietidp.py with W^_s := J_s(a_k) (gauge, partition, primal
    set, preconditioner and rho weights from J's diagonal all as in the linear case).
    Stop when ||a_{k+1} - a_k||_2 <= newton_tol ||a_{k+1}||_2 (per-patch local vectors
    concatenated); more than newton_max iterations -> NoConvergence.
Quadrature: the linear assembly's p+1 Gauss points per direction per element (R8).
"""
from __future__ import annotations

import numpy as np

from . import assembly
from .ietidp import Oracle, NoConvergence, patch_box, local_operators


def brauer(b2, k):
    """nu(b2) and dnu/d(b2) of the Brauer law nu = k1 exp(k2 b2) + k3 (b2 = |B|^2)."""
    k1, k2, k3 = (float(v) for v in k)
    e = np.exp(k2 * b2)
    return k1 * e + k3, k1 * k2 * e


def is_nonlinear(k) -> bool:
    return any(float(v) != 0.0 for v in k)


def patch_space(prob, s):
    lo, hi = patch_box(prob, s)
    return assembly.PatchSpace(prob.p, prob.elems, lo, hi)


def field_B(space, a):
    """B = curl A_h at every Gauss point of every element: list of (ids, cur, B, W)."""
    out = []
    for (ex, ey, ez) in space.elements():
        ids, val, cur, _, W = space.element_values(ex, ey, ez)
        B = np.einsum("a,qac->qc", a[ids], cur)
        out.append((ids, cur, B, W))
    return out


def patch_nonlinear_matrices(space, a, k):
    """Element loop: the secant matrix K(a) (nu(|B|) at each Gauss point) and the tangent
    matrix Kt(a) (nu I + 2 nu' B B^T) of one patch at its local coefficients a."""
    N = space.nloc
    Ks = np.zeros((N, N))
    Kt = np.zeros((N, N))
    for ids, cur, B, W in field_B(space, a):
        b2 = np.einsum("qc,qc->q", B, B)
        nu, dnu = brauer(b2, k)
        Ke = np.einsum("q,qac,qbc->ab", W * nu, cur, cur)
        cb = np.einsum("qac,qc->qa", cur, B)              # B . curl w_a at each point
        Kp = np.einsum("q,qa,qb->ab", W * 2.0 * dnu, cb, cb)
        Ks[np.ix_(ids, ids)] += Ke
        Kt[np.ix_(ids, ids)] += Ke + Kp
    return Ks, Kt


class NewtonOracle(Oracle):
    """The linear IETI-DP oracle with Newton's method around every implicit-Euler step for
    the patches with Brauer parameters prob.nl[s] != 0 (R25). Per step records the
    Newton iterations (newton_iters), and per linear solve its PCG iterations (solve_iters)
    and the relative increment (increments)."""

    def __init__(self, prob, **kw):
        nl = getattr(prob, "nl", None)
        self.nl = np.asarray(np.zeros((prob.n_patches, 3)) if nl is None else nl, dtype=float).reshape(-1, 3)
        self.nl_patches = [s for s in range(prob.n_patches) if is_nonlinear(self.nl[s])]
        self.newton_tol = float(getattr(prob, "newton_tol", 1e-8))
        self.newton_max = int(getattr(prob, "newton_max", 20))
        super().__init__(prob, **kw)
        self.spaces = {s: patch_space(prob, s) for s in self.nl_patches}
        self.newton_iters, self.solve_iters, self.increments = [], [], []

    def _nl_operators(self, a_k):
        """Re-factor the nonlinear patches with W^_s := Kt_s(a_k) + (sigma_s/dt) M_s and return
        g_s = (Kt_s(a_k) - K_s(a_k)) a_k for them (zero vectors elsewhere)."""
        pt = self.part
        g = [np.zeros_like(a_k[s]) for s in range(self.prob.n_patches)]
        for s in self.nl_patches:
            Ks, Kt = patch_nonlinear_matrices(self.spaces[s], a_k[s], self.nl[s])
            g[s] = Kt @ a_k[s] - Ks @ a_k[s]
            loc = local_operators(self.prob, s, pt.r_order(s), pt.p_loc[s], len(pt.r_i[s]), self.dt,
                                  False, self.d_loc[s], K_override=Kt)
            for n in self._local_names:
                getattr(self, n)[s] = loc[n]
            self.Ss[s] = loc["Ss"]
        self._coarse_and_weights()
        return g

    def step(self, load=None):
        if not self.nl_patches:
            k = super().step(load)
            self.newton_iters.append(1)
            self.solve_iters.append(k)
            self.increments.append(0.0)
            return k
        P = self.prob.n_patches
        t = (self.ell + 1) * self.dt
        a_prev = self.a
        a_k = [v.copy() for v in a_prev]
        total = 0
        for it in range(1, self.newton_max + 1):
            g = self._nl_operators(a_k)
            f = []
            for s in range(P):
                js = load[s] if load is not None else self.source_factor(s, t) * self.jS[s]
                f.append(self.Ma(s, a_prev[s]) / self.dt + js + g[s])
            a_new, k, hist = self.solve_rhs(f, t)
            total += k
            num = np.sqrt(sum(float(np.sum((a_new[s] - a_k[s]) ** 2)) for s in range(P)))
            den = np.sqrt(sum(float(np.sum(a_new[s] ** 2)) for s in range(P)))
            inc = num / den if den > 0 else 0.0
            self.solve_iters.append(k)
            self.increments.append(inc)
            self.hist.append(hist)
            a_k = a_new
            if inc <= self.newton_tol:
                break
        else:
            raise NoConvergence(f"step {self.ell}: Newton did not converge in {self.newton_max} iterations "
                                f"(increment {inc})")
        self.a = a_k
        self.ell += 1
        self.iters.append(total)
        self.newton_iters.append(it)
        return total


class MonolithicNewton:
    """Pin for NewtonOracle (R25, pin P22): textbook Newton on the glued conforming
    system with the same eliminated set E (the linear pin P11's system, R15):
    J(u_k) delta = -R(u_k), u_{k+1} = u_k + delta, with J and R summed from the patches'
    element-loop matrices and solved by a sparse direct solver (no IETI-DP, no rearranged
    right-hand side). Stops when ||delta|| <= newton_tol ||u_{k+1}|| (glued vector)."""

    def __init__(self, orc):
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla
        from .gauge import CLS_P, CLS_R
        self._sp, self._spla = sp, spla
        self.o = orc
        topo, pt = orc.topo, orc.part
        self.keep = np.nonzero((pt.part == CLS_R) | (pt.part == CLS_P))[0]
        self.gid = -np.ones(topo.nedges, dtype=np.int64)
        self.gid[self.keep] = np.arange(len(self.keep))
        self.nl = np.asarray(orc.prob.nl if orc.prob.nl is not None else np.zeros((orc.prob.n_patches, 3))).reshape(-1, 3)
        self.spaces = {s: patch_space(orc.prob, s) for s in range(orc.prob.n_patches) if is_nonlinear(self.nl[s])}
        self.Klin = {s: orc.K[s].copy() for s in range(orc.prob.n_patches) if s not in self.spaces}
        self.u = np.zeros(len(self.keep))
        self.ell = 0
        self.newton_iters = []

    def local(self, s, u):
        g = self.gid[self.o.topo.l2g[s]]
        a = np.zeros(len(g))
        a[g >= 0] = u[g[g >= 0]]
        return a

    def step(self):
        o = self.o
        pr = o.prob
        t = (self.ell + 1) * o.dt
        n = len(self.keep)
        u_prev = self.u.copy()
        u = u_prev.copy()
        for it in range(1, int(pr.newton_max) + 1):
            rows, cols, vals = [], [], []
            R = np.zeros(n)
            for s in range(pr.n_patches):
                a, ap = self.local(s, u), self.local(s, u_prev)
                if s in self.spaces:
                    Ks, Kt = patch_nonlinear_matrices(self.spaces[s], a, self.nl[s])
                else:
                    Ks = Kt = self.Klin[s]
                Js = Kt + o.M[s] / o.dt
                Rs = Ks @ a + o.M[s] @ (a - ap) / o.dt - o.source_factor(s, t) * o.jS[s]
                g = self.gid[o.topo.l2g[s]]
                loc = np.nonzero(g >= 0)[0]
                rr, cc = np.meshgrid(g[loc], g[loc], indexing="ij")
                rows.append(rr.ravel())
                cols.append(cc.ravel())
                vals.append(Js[np.ix_(loc, loc)].ravel())
                np.add.at(R, g[loc], Rs[loc])
            J = self._sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                    shape=(n, n)).tocsc()
            delta = self._spla.spsolve(J, -R)
            u = u + delta
            if np.linalg.norm(delta) <= pr.newton_tol * np.linalg.norm(u):
                break
        self.u = u
        self.ell += 1
        self.newton_iters.append(it)
        return u

    def coefficients(self):
        out = np.zeros(self.o.topo.nedges)
        out[self.keep] = self.u
        return out
