"""ORACLE (test infrastructure only) — monolithic glued direct solve (pin P11).

The conforming glued system of P:L122-135 with the same eliminated set E as the
IETI-DP oracle: unknowns are the non-E glued edges; the glued matrix and load are
sums of the patch contributions (B a = 0 is exactly continuity). Solved
with a sparse direct solver (scipy.sparse.linalg.splu). This is the plain
definition the IETI-DP iteration must reach at convergence (R15).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .gauge import CLS_P, CLS_R


class Monolithic:
    def __init__(self, orc):
        """`orc` is an oracle.ietidp.Oracle (its assembly and partition are reused)."""
        self.o = orc
        topo, pt = orc.topo, orc.part
        keep = np.nonzero((pt.part == CLS_R) | (pt.part == CLS_P))[0]
        self.keep = keep
        self.gid = -np.ones(topo.nedges, dtype=np.int64)
        self.gid[keep] = np.arange(len(keep))
        rows, cols, vals = [], [], []
        for s in range(orc.prob.n_patches):
            W = orc.W(s)
            g = self.gid[topo.l2g[s]]
            loc = np.nonzero(g >= 0)[0]
            Ws = W[np.ix_(loc, loc)]
            rr, cc = np.meshgrid(g[loc], g[loc], indexing="ij")
            rows.append(rr.ravel())
            cols.append(cc.ravel())
            vals.append(Ws.ravel())
        n = len(keep)
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsc()
        self.A = A
        self.lu = spla.splu(A)
        self.u = np.zeros(n)     # glued coefficient vector (non-E edges)
        self.ell = 0

    def local(self, s, u=None):
        u = self.u if u is None else u
        g = self.gid[self.o.topo.l2g[s]]
        a = np.zeros(len(g))
        a[g >= 0] = u[g[g >= 0]]
        return a

    def step(self, load=None):
        o = self.o
        t = (self.ell + 1) * o.dt
        n = len(self.keep)
        f = np.zeros(n)
        for s in range(o.prob.n_patches):
            js = load[s] if load is not None else o.source_factor(s, t) * o.jS[s]
            fs = o.M[s] @ self.local(s) / o.dt + js
            g = self.gid[o.topo.l2g[s]]
            np.add.at(f, g[g >= 0], fs[g >= 0])
        self.u = self.lu.solve(f)
        self.ell += 1
        return self.u

    def coefficients(self):
        out = np.zeros(self.o.topo.nedges)
        out[self.keep] = self.u
        return out
