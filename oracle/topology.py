"""ORACLE (test infrastructure only) — glued control grid of a box multipatch domain.

Follows P:L78 (§2.2: conforming spaces, "pairwise matching basis functions" on
interfaces) and the control-mesh view of P:L154 (§3: "construct a tree on the
underlying (control) mesh"). With Curry-Schoenberg D-splines every local DOF is
an edge of the patch's n x n x n control grid; neighbouring patches share their
boundary control layer, so the glued grid has N_c = P_c (n_c-1) + 1 vertices per
direction and a shared DOF is one glued edge (R3/R4).

Edge classes (R3 / SURVEY Q3, §8(c) step 3):
  D  tangential on the domain boundary (a transverse index in {0, N-1})
  WB both transverse indices are interior patch-boundary layers (wirebasket curves)
  F  exactly one transverse index is an interior patch-boundary layer
  I  otherwise
Region: C-owned if any owning patch has sigma > 0, else I-only.
"""
from __future__ import annotations

import numpy as np

from .assembly import local_dof_table

D, WB, F, I = 0, 1, 2, 3


class Topology:
    def __init__(self, npatch, p, elems, sigma):
        self.npatch = tuple(int(v) for v in npatch)
        self.n = tuple(int(e) + p for e in elems)
        n = self.n
        self.N = tuple(P * (nd - 1) + 1 for P, nd in zip(self.npatch, n))
        Nx, Ny, Nz = self.N
        self.nverts = Nx * Ny * Nz
        # global edge numbering: component-major, i fastest, then j, then k
        self.edims = []
        self.eoff = []
        off = 0
        for c in range(3):
            d = list(self.N)
            d[c] -= 1
            self.edims.append(tuple(d))
            self.eoff.append(off)
            off += d[0] * d[1] * d[2]
        self.nedges = off
        self.n_patches = int(np.prod(self.npatch))
        self.sigma = np.asarray(sigma, dtype=np.float64)

        # local -> global edge maps by brute force over every patch's local DOFs
        tab = local_dof_table(n)
        self.l2g = np.zeros((self.n_patches, len(tab)), dtype=np.int64)
        for s in range(self.n_patches):
            ix = s % self.npatch[0]
            iy = (s // self.npatch[0]) % self.npatch[1]
            iz = s // (self.npatch[0] * self.npatch[1])
            for a, (c, i, j, k) in enumerate(tab):
                self.l2g[s, a] = self.edge_id(c, ix * (n[0] - 1) + i, iy * (n[1] - 1) + j, iz * (n[2] - 1) + k)
        owners = [[] for _ in range(self.nedges)]
        for s in range(self.n_patches):
            for a in range(len(tab)):
                owners[self.l2g[s, a]].append(s)
        self.owners = owners
        # every glued edge has at least one owner
        assert all(len(o) > 0 for o in owners)

        self.cls = np.zeros(self.nedges, dtype=np.int64)
        self.c_owned = np.zeros(self.nedges, dtype=bool)
        self.i_owned = np.zeros(self.nedges, dtype=bool)
        for e in range(self.nedges):
            c, i, j, k = self.edge_coords(e)
            idx = (i, j, k)
            trans = [d for d in range(3) if d != c]
            bnd = any(idx[d] == 0 or idx[d] == self.N[d] - 1 for d in trans)
            if bnd:
                self.cls[e] = D
            else:
                nlay = sum(1 for d in trans if idx[d] % (n[d] - 1) == 0)
                self.cls[e] = WB if nlay == 2 else (F if nlay == 1 else I)
            sig = [self.sigma[s] > 0 for s in owners[e]]
            self.c_owned[e] = any(sig)
            self.i_owned[e] = not all(sig)

    def edge_id(self, c, i, j, k) -> int:
        dx, dy, _ = self.edims[c]
        return self.eoff[c] + i + dx * (j + dy * k)

    def edge_coords(self, e):
        c = 0 if e < self.eoff[1] else (1 if e < self.eoff[2] else 2)
        r = e - self.eoff[c]
        dx, dy, _ = self.edims[c]
        return c, r % dx, (r // dx) % dy, r // (dx * dy)

    def vertex_id(self, i, j, k) -> int:
        return i + self.N[0] * (j + self.N[1] * k)

    def edge_vertices(self, e):
        """(tail, head): head = tail + unit step along the edge's direction."""
        c, i, j, k = self.edge_coords(e)
        a = self.vertex_id(i, j, k)
        h = [i, j, k]
        h[c] += 1
        return a, self.vertex_id(*h)
