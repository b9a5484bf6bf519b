"""ORACLE (test infrastructure only) — plain CPU tree-cotree IETI-DP implicit Euler.

Paper passages followed, in order:
  P:L122-135 (§2.2, eq. (euler)): W = M + dt K, f = M a^(l) + dt j^(l+1).  Used in the
      scaled form W^ = W/dt = K + M/dt, f^ = M a^(l)/dt + j^(l+1) (same a; the
      multipliers are rescaled; R7 / SURVEY Q7).
  P:L78-82, L116 (§2.2): coupling by signed Boolean restrictions, B = [R_C, -R_I];
      for many patches one multiplier per b-edge, +1 at the lower patch id,
      -1 at the higher (R4).
  P:L138-153 (§3): a = (a_e, a_p = N p, a_r); the 3x3 block system.
  P:L154 (§3): "two sequential Schur complements" (Farhat_2001aa): the primal
      Schur complement S_pp = sum_s N_s^T (W_pp - W_pr W_rr^-1 W_rp) N_s and the
      dual operator F = B W_rr^-1 B^T + B Phi N S_pp^-1 N^T Phi^T B^T, Phi = W_rr^-1 W_rp.
  P:L170 (§4): PCG with the Dirichlet preconditioner M^-1 = sum_s B_D S_bb B_D^T
      (scaling none as in the paper, or rho-scaling, R5).
PCG recurrences, stopping rule and iteration count: DESIGN.md R6 / SURVEY Appendix C.
Every solve uses LAPACK Cholesky (scipy.linalg.cho_factor / cho_solve) on the
full-storage local matrices; S_bb is applied by its definition
W_bb - W_bi W_ii^-1 W_ib (interior solves), not by any condensed factor.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import assembly, topology, gauge


class NotSPD(RuntimeError):
    pass


class NoConvergence(RuntimeError):
    pass


def _chol(A, what):
    if A.shape[0] == 0:
        return None
    try:
        return sla.cho_factor(A, lower=True, check_finite=True)
    except np.linalg.LinAlgError as exc:
        raise NotSPD(f"{what}: {exc}") from exc


def _solve(cf, b):
    if cf is None:
        return np.zeros_like(b)
    return sla.cho_solve(cf, b, check_finite=False)


def chol_skip_solve(G, b, tol=1e-12):
    """Solve G c = b for a small symmetric G by Cholesky in index order, skipping (c_j = 0)
    every column whose pivot is <= tol * max_i G_ii (numerically dependent directions).
    Used by the warm start (R20), written out so the GPU's copy can follow it."""
    k = len(b)
    L = np.zeros((k, k))
    act = [False] * k
    gmax = max((G[i, i] for i in range(k)), default=0.0)
    for j in range(k):
        s = G[j, j] - sum(L[j, q] * L[j, q] for q in range(j) if act[q])
        if not (s > tol * gmax):
            continue
        act[j] = True
        L[j, j] = np.sqrt(s)
        for i in range(j + 1, k):
            L[i, j] = (G[i, j] - sum(L[i, q] * L[j, q] for q in range(j) if act[q])) / L[j, j]
    y = np.zeros(k)
    for j in range(k):
        if act[j]:
            y[j] = (b[j] - sum(L[j, q] * y[q] for q in range(j) if act[q])) / L[j, j]
    c = np.zeros(k)
    for j in reversed(range(k)):
        if act[j]:
            c[j] = (y[j] - sum(L[q, j] * c[q] for q in range(j + 1, k) if act[q])) / L[j, j]
    return c


class Oracle:
    def __init__(self, prob, assemble=True):
        self.prob = prob
        P = prob.n_patches
        self.topo = topology.Topology(prob.npatch, prob.p, prob.elems, prob.sigma)
        self.tree = gauge.build_tree(self.topo, prob.tree_order)
        self.part = gauge.Partition(self.topo, self.tree)
        self.dt = prob.T / prob.n_steps
        if assemble:
            self._assemble()
            self._factor()
        self.a = [np.zeros(self.topo.l2g.shape[1]) for _ in range(P)]
        self.ell = 0
        self.iters = []
        self.hist = []
        self.warm_W, self.warm_FW = [], []  # previous solutions and F times them (R20)

    # ---- setup -------------------------------------------------------------------
    def patch_box(self, s):
        pr = self.prob
        ix = s % pr.npatch[0]
        iy = (s // pr.npatch[0]) % pr.npatch[1]
        iz = s // (pr.npatch[0] * pr.npatch[1])
        idx = (ix, iy, iz)
        lo = [pr.lo[d] + (pr.hi[d] - pr.lo[d]) * idx[d] / pr.npatch[d] for d in range(3)]
        hi = [pr.lo[d] + (pr.hi[d] - pr.lo[d]) * (idx[d] + 1) / pr.npatch[d] for d in range(3)]
        return lo, hi

    def _assemble(self):
        pr = self.prob
        self.K, self.M, self.jS = [], [], []
        for s in range(pr.n_patches):
            lo, hi = self.patch_box(s)
            sp = assembly.PatchSpace(pr.p, pr.elems, lo, hi)
            K, M, jS = assembly.assemble_patch(sp, pr.nu[s], pr.sigma[s], pr.source)
            self.K.append(K)
            self.M.append(M)
            self.jS.append(jS)

    def W(self, s):
        """W^_s = nu_s K_s + (sigma_s/dt) M_s (K, M carry nu, sigma)."""
        return self.K[s] + self.M[s] / self.dt

    def _factor(self):
        pt = self.part
        P = self.prob.n_patches
        self.Wrr_cf, self.Wii_cf, self.Wrp, self.Wpp, self.Phi, self.Wbb, self.Wbi, self.Wfull = [], [], [], [], [], [], [], []
        nc = pt.nc
        Spp = np.zeros((nc, nc))
        for s in range(P):
            W = self.W(s)
            r = pt.r_order(s)
            pl = pt.p_loc[s]
            Wrr = W[np.ix_(r, r)]
            cf = _chol(Wrr, f"W_rr patch {s}")
            Wrp = W[np.ix_(r, pl)]
            Wpp = W[np.ix_(pl, pl)]
            Phi = _solve(cf, Wrp) if cf is not None else np.zeros_like(Wrp)
            Ss = Wpp - Wrp.T @ Phi
            g = pt.p_grp[s]
            Spp[np.ix_(g, g)] += Ss
            ni = len(pt.r_i[s])
            Wii = Wrr[:ni, :ni]
            self.Wii_cf.append(_chol(Wii, f"W_ii patch {s}"))
            self.Wbb.append(Wrr[ni:, ni:])
            self.Wbi.append(Wrr[ni:, :ni])
            self.Wrr_cf.append(cf)
            self.Wrp.append(Wrp)
            self.Wpp.append(Wpp)
            self.Phi.append(Phi)
            self.Wfull.append(W)
        self.Spp = Spp
        self.Spp_cf = _chol(Spp, "coarse S_pp")
        # rho-scaling weights (R5): rho_s = W^_s diagonal at the b-DOF
        m = pt.m
        self.wplus = np.ones(m)
        self.wminus = np.ones(m)
        if self.prob.scaling == 1 and m > 0:
            for k in range(m):
                sp, ap = pt.lam_plus[k]
                sm, am = pt.lam_minus[k]
                lp = pt.r_order(sp)[ap]
                lm = pt.r_order(sm)[am]
                rp = self.Wfull[sp][lp, lp]
                rm = self.Wfull[sm][lm, lm]
                self.wplus[k] = rm / (rp + rm)
                self.wminus[k] = rp / (rp + rm)

    # ---- operators ---------------------------------------------------------------
    def nr(self, s):
        return len(self.part.r_i[s]) + len(self.part.r_b[s])

    def Bt(self, lam, wp=None, wm=None):
        """Per-patch v_s = B_s^T lam (optionally weighted: B_D^(s)T)."""
        pt = self.part
        v = [np.zeros(self.nr(s)) for s in range(self.prob.n_patches)]
        for k in range(pt.m):
            sp, ap = pt.lam_plus[k]
            sm, am = pt.lam_minus[k]
            v[sp][ap] += lam[k] * (1.0 if wp is None else wp[k])
            v[sm][am] -= lam[k] * (1.0 if wm is None else wm[k])
        return v

    def Bj(self, y, wp=None, wm=None):
        """(B y)_k = y_{s+}[a+] - y_{s-}[a-] (optionally weighted)."""
        pt = self.part
        out = np.zeros(pt.m)
        for k in range(pt.m):
            sp, ap = pt.lam_plus[k]
            sm, am = pt.lam_minus[k]
            out[k] = y[sp][ap] * (1.0 if wp is None else wp[k]) - y[sm][am] * (1.0 if wm is None else wm[k])
        return out

    def NT(self, vecs):
        """sum_s N_s^T v_s (v_s indexed by the patch's primal DOFs)."""
        g = np.zeros(self.part.nc)
        for s in range(self.prob.n_patches):
            np.add.at(g, self.part.p_grp[s], vecs[s])
        return g

    def F(self, lam):
        """F lam = B W_rr^-1 B^T lam + B Phi N S_pp^-1 N^T Phi^T B^T lam."""
        P = self.prob.n_patches
        v = self.Bt(lam)
        u = [_solve(self.Wrr_cf[s], v[s]) for s in range(P)]
        g = self.NT([self.Phi[s].T @ v[s] for s in range(P)])
        pc = _solve(self.Spp_cf, g)
        y = [u[s] + self.Phi[s] @ pc[self.part.p_grp[s]] for s in range(P)]
        return self.Bj(y)

    def Sbb_apply(self, s, vb):
        """S_bb v = W_bb v - W_bi W_ii^-1 W_ib v (Dirichlet problem on patch s)."""
        out = self.Wbb[s] @ vb
        if self.Wii_cf[s] is not None:
            out = out - self.Wbi[s] @ _solve(self.Wii_cf[s], self.Wbi[s].T @ vb)
        return out

    def precond(self, r):
        """z = sum_s B_D^(s) S_bb^(s) B_D^(s)T r."""
        pt = self.part
        P = self.prob.n_patches
        v = self.Bt(r, self.wplus, self.wminus)
        w = []
        for s in range(P):
            ni = len(pt.r_i[s])
            ws = np.zeros(self.nr(s))
            ws[ni:] = self.Sbb_apply(s, v[s][ni:])
            w.append(ws)
        return self.Bj(w, self.wplus, self.wminus)

    # ---- time step ---------------------------------------------------------------
    def source_factor(self, s, t):
        pr = self.prob
        return assembly.source_time_factor(pr.source, t, pr.nu[s], pr.sigma[s])

    def pcg(self, d, W=None, FW=None):
        """Classical Hestenes-Stiefel PCG from lam0 = 0 (R6), or, warm start
        (R20), from the Galerkin projection of the solution on
        the span of previous solutions W_j: lam0 = sum_j c_j W_j with
        G c = W^T d, G_ij = (W_i^T FW_j + W_j^T FW_i)/2, FW_j = F W_j taken as d_j - r_j
        (the step's right-hand side minus its final recurrence residual), solved by
        chol_skip_solve; r0 = d - sum_j c_j FW_j. The stopping reference is
        sqrt(d^T M^-1 d) in both cases (the cold r0^T z0). Returns (lam, iterations,
        relres history, final recurrence residual)."""
        pr = self.prob
        z = self.precond(d)
        rho = rho0 = float(d @ z)
        if rho0 == 0.0 or len(d) == 0:
            return np.zeros_like(d), 0, [1.0], np.zeros_like(d)
        if not W:
            lam = np.zeros_like(d)
            r = d.copy()
            hist = [1.0]
        else:
            k = len(W)
            G = np.zeros((k, k))
            for i in range(k):
                for j in range(k):
                    G[i, j] = 0.5 * (float(W[i] @ FW[j]) + float(W[j] @ FW[i]))
            c = chol_skip_solve(G, np.array([float(w @ d) for w in W]))
            lam = sum(c[j] * W[j] for j in range(k))
            r = d - sum(c[j] * FW[j] for j in range(k))
            z = self.precond(r)
            rho = float(r @ z)
            rel = np.sqrt(max(rho, 0.0) / rho0)
            hist = [rel]
            if rel <= pr.rtol:
                return lam, 0, hist, r
        pk = z.copy()
        k = 0
        while True:
            q = self.F(pk)
            k += 1
            alpha = rho / float(pk @ q)
            lam += alpha * pk
            r -= alpha * q
            z = self.precond(r)
            rhon = float(r @ z)
            rel = np.sqrt(max(rhon, 0.0) / rho0)
            hist.append(rel)
            if rel <= pr.rtol:
                return lam, k, hist, r
            if k >= pr.max_iter:
                raise NoConvergence(f"step {self.ell}: {k} iterations, relres {rel}")
            beta = rhon / rho
            rho = rhon
            pk = z + beta * pk

    def step(self, load=None):
        """One implicit-Euler step l -> l+1 (t = (l+1) dt). `load`, if given, is a list
        of per-patch load vectors j^(l+1) replacing phi_s(t) jS_s (pin P15)."""
        pt = self.part
        P = self.prob.n_patches
        t = (self.ell + 1) * self.dt
        f = []
        for s in range(P):
            js = load[s] if load is not None else self.source_factor(s, t) * self.jS[s]
            f.append(self.M[s] @ self.a[s] / self.dt + js)
        fr = [f[s][pt.r_order(s)] for s in range(P)]
        fp = [f[s][pt.p_loc[s]] for s in range(P)]
        x1 = [_solve(self.Wrr_cf[s], fr[s]) for s in range(P)]
        h = [self.Wrp[s].T @ x1[s] for s in range(P)]
        fpg = self.NT(fp)
        p0 = _solve(self.Spp_cf, fpg - self.NT(h))
        d = self.Bj([x1[s] - self.Phi[s] @ p0[pt.p_grp[s]] for s in range(P)])
        kw = int(getattr(self.prob, "warm_start", 0))
        if self.ell == 0:
            self.warm_W, self.warm_FW = [], []
        lam, k, hist, r = self.pcg(d, self.warm_W[-kw:] if kw else None, self.warm_FW[-kw:] if kw else None)
        if kw:
            self.warm_W = (self.warm_W + [lam.copy()])[-kw:]
            self.warm_FW = (self.warm_FW + [d - r])[-kw:]
        v = self.Bt(lam)
        pc = _solve(self.Spp_cf, fpg - self.NT([h[s] - self.Phi[s].T @ v[s] for s in range(P)]))
        for s in range(P):
            ar = _solve(self.Wrr_cf[s], fr[s] - v[s] - self.Wrp[s] @ pc[pt.p_grp[s]])
            a = np.zeros(self.topo.l2g.shape[1])
            a[pt.r_order(s)] = ar
            a[pt.p_loc[s]] = pc[pt.p_grp[s]]
            self.a[s] = a
        self.lam = lam
        self.pc = pc
        self.ell += 1
        self.iters.append(k)
        self.hist.append(hist)
        return k

    def run(self, n=None):
        n = self.prob.n_steps - self.ell if n is None else n
        for _ in range(n):
            self.step()
        return self

    # ---- readout -----------------------------------------------------------------
    def coefficients(self, layout=1):
        """layout 0: per-patch local vectors concatenated; layout 1: one value per
        glued edge, taken from the lowest-id owner (E edges = 0)."""
        if layout == 0:
            return np.concatenate(self.a)
        out = np.zeros(self.topo.nedges)
        done = np.zeros(self.topo.nedges, dtype=bool)
        for s in range(self.prob.n_patches):
            g = self.topo.l2g[s]
            new = ~done[g]
            out[g[new]] = self.a[s][new]
            done[g] = True
        return out

    def dense_F(self):
        m = self.part.m
        return np.column_stack([self.F(e) for e in np.eye(m)]) if m else np.zeros((0, 0))

    def dense_precond(self):
        m = self.part.m
        return np.column_stack([self.precond(e) for e in np.eye(m)]) if m else np.zeros((0, 0))
