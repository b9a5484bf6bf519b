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

import math

import numpy as np
import scipy.linalg as sla

from . import assembly, topology, gauge, paper_mms


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


def patch_box(prob, s):
    """Axis-aligned box of patch s = ix + Px (iy + Py iz) in the uniform patch grid."""
    ix = s % prob.npatch[0]
    iy = (s // prob.npatch[0]) % prob.npatch[1]
    iz = s // (prob.npatch[0] * prob.npatch[1])
    idx = (ix, iy, iz)
    lo = [prob.lo[d] + (prob.hi[d] - prob.lo[d]) * idx[d] / prob.npatch[d] for d in range(3)]
    hi = [prob.lo[d] + (prob.hi[d] - prob.lo[d]) * (idx[d] + 1) / prob.npatch[d] for d in range(3)]
    return lo, hi


def local_operators(prob, s, r, pl, ni, dt, lean=False, dl=None, K_override=None):
    """Per-patch setup (P:L83-87 assembly, P:L133 W^ = K + M/dt, P:L154 local Schur
    complement): element-loop K, M, j_S of patch s; W^ = nu K + (sigma/dt) M restricted to
    r = [i; b] (local ids `r`) and to the primal DOFs `pl`; Cholesky of W_rr and W_ii;
    Phi = W_rr^-1 W_rp; S^s = W_pp - W_pr Phi. lean=True keeps only what the time stepping
    needs (no K / full W; the blocks of W that are only multiplied with, and M, in sparse
    storage; M dropped for insulators, where it is zero) -- storage only, same operators.
    K_override replaces nu K (the Newton step of oracle/nonlinear.py: the tangent matrix).
    Module-level so that a process pool can run it patch by patch."""
    lo, hi = patch_box(prob, s)
    sp = assembly.PatchSpace(prob.p, prob.elems, lo, hi)
    K, M, jS = assembly.assemble_patch(sp, prob.nu[s], prob.sigma[s], prob.source)
    if K_override is not None:
        K = K_override
    W = K + M / dt
    Wrr = W[np.ix_(r, r)]
    cf = _chol(Wrr, f"W_rr patch {s}")
    Wrp = W[np.ix_(r, pl)]
    Wpp = W[np.ix_(pl, pl)]
    Phi = _solve(cf, Wrp) if cf is not None else np.zeros_like(Wrp)
    Ss = Wpp - Wrp.T @ Phi
    Wii_cf = _chol(Wrr[:ni, :ni], f"W_ii patch {s}")
    out = dict(Wrr_cf=cf, Wii_cf=Wii_cf, Wrp=Wrp, Wpp=Wpp, Phi=Phi, Ss=Ss, Wbb=Wrr[ni:, ni:], Wbi=Wrr[ni:, :ni],
               Wdiag=np.diag(W).copy(), jS=jS, K=K, M=M, Wfull=W, Pi=None, hr=None, hp=None)
    if prob.source == paper_mms.SOURCE_PAPER:
        # the paper's experiment: a(0) = Pi_h S and the Dirichlet lifting
        # a_D(t) = e^-t (Pi_h S)_D (R21); its right-hand-side terms W_rD a_D, W_pD a_D
        Pi = paper_mms.commuting_projection(sp, paper_mms.S)
        dl = np.zeros(0, dtype=np.int64) if dl is None else dl
        out.update(Pi=Pi, hr=W[np.ix_(r, dl)] @ Pi[dl], hp=W[np.ix_(pl, dl)] @ Pi[dl])
    if lean:
        import scipy.sparse as sps
        out.update(K=None, Wfull=None, Wpp=None, M=sps.csr_matrix(M) if prob.sigma[s] > 0 else None,
                   Wrp=sps.csr_matrix(Wrp), Wbb=sps.csr_matrix(out["Wbb"]), Wbi=sps.csr_matrix(out["Wbi"]))
    return out


def _local_job(args):
    return local_operators(*args)


class Oracle:
    """workers > 1 runs the per-patch work (assembly + local factorisations in a process
    pool, the local solves of every F / preconditioner / step in a thread pool; LAPACK
    releases the GIL) and lean=True drops storage the stepping never reads (see
    local_operators). Neither changes the operators; sums over patches keep patch order."""

    def __init__(self, prob, assemble=True, workers=1, lean=False):
        self.prob = prob
        P = prob.n_patches
        self.workers = max(1, int(workers))
        self.lean = lean
        self._tp = None
        self.topo = topology.Topology(prob.npatch, prob.p, prob.elems, prob.sigma)
        self.tree = gauge.build_tree(self.topo, prob.tree_order)
        self.part = gauge.Partition(self.topo, self.tree)
        self.dt = prob.T / prob.n_steps
        self._index_tables()
        # local Dirichlet DOFs (class D edges) of every patch
        self.d_loc = [np.array([a for a in self.part.e_loc[s] if self.part.part[self.topo.l2g[s][a]] == gauge.CLS_D],
                               dtype=np.int64) for s in range(P)]
        self.lifting = prob.source == paper_mms.SOURCE_PAPER
        if assemble:
            self._setup_locals()
        self.a = [np.zeros(self.topo.l2g.shape[1]) for _ in range(P)]
        if self.lifting and assemble:  # A(0) = Pi_h A_0 (R21)
            self.a = [self.Pi[s].copy() for s in range(P)]
        self.errors = paper_mms.ErrorTracker(self) if (self.lifting and getattr(prob, "track_errors", False)) else None
        self.ell = 0
        self.iters = []
        self.hist = []
        self.warm_W, self.warm_FW = [], []  # previous solutions and F times them (R20)

    # ---- setup -------------------------------------------------------------------
    def patch_box(self, s):
        return patch_box(self.prob, s)

    def _map(self, fn, items):
        """[fn(x) for x in items], on the thread pool when workers > 1 (results in order)."""
        if self.workers == 1:
            return [fn(x) for x in items]
        if self._tp is None:
            from concurrent.futures import ThreadPoolExecutor
            self._tp = ThreadPoolExecutor(self.workers)
        return list(self._tp.map(fn, items))

    def _index_tables(self):
        """Flat positions of the two local copies of every multiplier (B_s entries)
        in the concatenation of the patches' r vectors."""
        pt = self.part
        P = self.prob.n_patches
        self.r_off = np.zeros(P + 1, dtype=np.int64)
        for s in range(P):
            self.r_off[s + 1] = self.r_off[s] + len(pt.r_i[s]) + len(pt.r_b[s])
        if pt.m:
            self.pos_plus = self.r_off[pt.lam_plus[:, 0]] + pt.lam_plus[:, 1]
            self.pos_minus = self.r_off[pt.lam_minus[:, 0]] + pt.lam_minus[:, 1]
        else:
            self.pos_plus = self.pos_minus = np.zeros(0, dtype=np.int64)

    _local_names = ("Wrr_cf", "Wii_cf", "Wrp", "Wpp", "Phi", "Wbb", "Wbi", "Wdiag", "jS", "K", "M", "Wfull", "Pi",
                    "hr", "hp")

    def _setup_locals(self):
        pr = self.prob
        pt = self.part
        P = pr.n_patches
        jobs = [(pr, s, pt.r_order(s), pt.p_loc[s], len(pt.r_i[s]), self.dt, self.lean, self.d_loc[s]) for s in range(P)]
        names = self._local_names
        for n in names:
            setattr(self, n, [])
        self.Ss = []
        if self.workers == 1:
            results = map(_local_job, jobs)
            pool = None
        else:
            import multiprocessing as mp
            from threadpoolctl import threadpool_limits
            self._limits = threadpool_limits(1)   # one BLAS thread per pool worker
            pool = mp.get_context("fork").Pool(self.workers)
            results = pool.imap(_local_job, jobs, chunksize=1)
        for s, loc in enumerate(results):
            self.Ss.append(loc["Ss"])
            for n in names:
                getattr(self, n).append(loc[n])
        if pool is not None:
            pool.close()
            pool.join()
        self._coarse_and_weights()

    def _coarse_and_weights(self):
        """S_pp = sum_s N_s^T S^s N_s (patch order: the sums are ordered), its Cholesky factor,
        and the rho-scaling weights from the local matrices' diagonals."""
        pt = self.part
        nc = pt.nc
        Spp = np.zeros((nc, nc))
        for s in range(self.prob.n_patches):
            g = pt.p_grp[s]
            Spp[np.ix_(g, g)] += self.Ss[s]
        self.Spp = Spp
        if self.workers > 1:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(self.workers):
                self.Spp_cf = _chol(Spp, "coarse S_pp")
        else:
            self.Spp_cf = _chol(Spp, "coarse S_pp")
        if self.lean:
            self.Spp = None
            self.Ss = [None] * len(self.Ss)
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
                rp = self.Wdiag[sp][lp]
                rm = self.Wdiag[sm][lm]
                self.wplus[k] = rm / (rp + rm)
                self.wminus[k] = rp / (rp + rm)

    def W(self, s):
        """W^_s = nu_s K_s + (sigma_s/dt) M_s (K, M carry nu, sigma)."""
        return self.K[s] + self.M[s] / self.dt

    def Ma(self, s, a):
        """M_s a (zero for an insulator whose M is not stored, lean mode)."""
        M = self.M[s]
        return np.zeros_like(a) if M is None else M @ a

    # ---- operators ---------------------------------------------------------------
    def nr(self, s):
        return len(self.part.r_i[s]) + len(self.part.r_b[s])

    def Bt(self, lam, wp=None, wm=None):
        """Per-patch v_s = B_s^T lam (optionally weighted: B_D^(s)T): the multiplier k adds
        +lam_k at its lower patch's copy and -lam_k at the other (R4)."""
        flat = np.zeros(self.r_off[-1])
        np.add.at(flat, self.pos_plus, lam * (1.0 if wp is None else wp))
        np.add.at(flat, self.pos_minus, -(lam * (1.0 if wm is None else wm)))
        return [flat[self.r_off[s]:self.r_off[s + 1]] for s in range(self.prob.n_patches)]

    def Bj(self, y, wp=None, wm=None):
        """(B y)_k = y_{s+}[a+] - y_{s-}[a-] (optionally weighted)."""
        if self.part.m == 0:
            return np.zeros(0)
        flat = np.concatenate(y)
        return flat[self.pos_plus] * (1.0 if wp is None else wp) - flat[self.pos_minus] * (1.0 if wm is None else wm)

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
        u = self._map(lambda s: _solve(self.Wrr_cf[s], v[s]), range(P))
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

        def one(s):
            ni = len(pt.r_i[s])
            ws = np.zeros(self.nr(s))
            ws[ni:] = self.Sbb_apply(s, v[s][ni:])
            return ws
        w = self._map(one, range(P))
        return self.Bj(w, self.wplus, self.wminus)

    # ---- time step ---------------------------------------------------------------
    def source_factor(self, s, t):
        pr = self.prob
        return assembly.source_time_factor(pr.source, t, pr.nu[s], pr.sigma[s], getattr(pr, "source_params", ()))

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
        P = self.prob.n_patches
        t = (self.ell + 1) * self.dt
        f = []
        for s in range(P):
            js = load[s] if load is not None else self.source_factor(s, t) * self.jS[s]
            f.append(self.Ma(s, self.a[s]) / self.dt + js)
        a_old = self.a
        self.a, k, hist = self.solve_rhs(f, t)
        self.ell += 1
        self.iters.append(k)
        self.hist.append(hist)
        if self.errors is not None:
            self.errors.after_step(a_old)
        return k

    def solve_rhs(self, f, t):
        """The 3x3 block system of P:L139-153 for the per-patch (torn) right-hand sides f_s at
        time t: dual rhs d, PCG for lambda, recovery of a = (a_e = 0, a_p = N p, a_r).
        Returns (per-patch local vectors, PCG iterations, relres history)."""
        pt = self.part
        P = self.prob.n_patches
        fr = [f[s][pt.r_order(s)] for s in range(P)]
        fp = [f[s][pt.p_loc[s]] for s in range(P)]
        if self.lifting:  # f_r - W_rD a_D(t), f_p - W_pD a_D(t), a_D(t) = e^-t (Pi_h S)_D
            eD = math.exp(-t)
            fr = [fr[s] - eD * self.hr[s] for s in range(P)]
            fp = [fp[s] - eD * self.hp[s] for s in range(P)]
        x1 = self._map(lambda s: _solve(self.Wrr_cf[s], fr[s]), range(P))
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

        def recover(s):
            ar = _solve(self.Wrr_cf[s], fr[s] - v[s] - self.Wrp[s] @ pc[pt.p_grp[s]])
            a = np.zeros(self.topo.l2g.shape[1])
            a[pt.r_order(s)] = ar
            a[pt.p_loc[s]] = pc[pt.p_grp[s]]
            if self.lifting:
                dl = self.d_loc[s]
                a[dl] = math.exp(-t) * self.Pi[s][dl]
            return a
        a_new = self._map(recover, range(P))
        self.lam = lam
        self.pc = pc
        return a_new, k, hist

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
