r"""ORACLE (test infrastructure only) — tree-cotree gauge and e/p/r DOF splitting.

Paper passages:
  P:L138 (§3)  split a into eliminated e (gauge or Dirichlet), primal p (coupled
               strongly, one value p_k per coupled group via N), remaining r.
  P:L154 (§3)  tree built globally on the control mesh, "on the wirebasket first,
               before it is extended into the subdomain faces and at last into
               the subdomain interiors"; tree DOFs in Omega_I eliminated; tree DOFs
               on Gamma primal; Dirichlet DOFs eliminated; rest remaining.
Readings (R1/R2), needed for more than two subdomains:
  tree = ranked Kruskal over (rank, id): 0 D, 1 C-owned WB, 2 C-owned F,
         3 C-owned I, 4 I-only WB, 5 I-only F, 6 I-only I; edge added iff its two
         endpoints are in different union-find sets. tree_order=1 visits ids
         descending within each rank (gauge-invariance pin P13).
  E = D u (T n I-only);  P = (WB \ E) u (T n Gamma-closure \ D);  r = rest,
  where Gamma-closure edges have both a C and an I owner.
"""
from __future__ import annotations

import numpy as np

from .topology import D, WB, F, I

GAUGE_E, CLS_P, CLS_R, CLS_D = 0, 1, 2, 3   # partition codes: eliminated-gauge, primal, remaining, Dirichlet


class UnionFind:
    def __init__(self, n):
        self.parent = list(range(n))

    def find(self, a):
        root = a
        while self.parent[root] != root:
            root = self.parent[root]
        while self.parent[a] != root:
            self.parent[a], a = root, self.parent[a]
        return root

    def union(self, a, b) -> bool:
        ra, rb = self.find(a), self.find(b)
        if ra == rb:
            return False
        self.parent[max(ra, rb)] = min(ra, rb)
        return True


def edge_rank(topo, e) -> int:
    c = topo.cls[e]
    if c == D:
        return 0
    base = 1 if topo.c_owned[e] else 4
    return base + {WB: 0, F: 1, I: 2}[int(c)]


def build_tree(topo, tree_order: int = 0) -> np.ndarray:
    """Boolean mask of tree edges (ranked Kruskal)."""
    ranks = np.array([edge_rank(topo, e) for e in range(topo.nedges)])
    ids = np.arange(topo.nedges)
    key_id = ids if tree_order == 0 else -ids
    order = np.lexsort((key_id, ranks))
    uf = UnionFind(topo.nverts)
    in_tree = np.zeros(topo.nedges, dtype=bool)
    for e in order:
        a, b = topo.edge_vertices(int(e))
        if uf.union(a, b):
            in_tree[e] = True
    return in_tree


class Partition:
    """Global classification and per-patch index sets.

    part[e] in {CLS_D, GAUGE_E, CLS_P, CLS_R}. For each patch s:
      r_i[s]  local ids of r-DOFs with one owner (interior, i)
      r_b[s]  local ids of r-DOFs with two owners (interface, b)
      p_loc[s], p_grp[s]  local ids of primal DOFs and their global primal group
    lam_edges: glued ids of b-edges, ascending = multiplier order; each lambda k
    has (s_plus, a_plus) at the lower patch id (+1) and (s_minus, a_minus) (-1).
    """

    def __init__(self, topo, in_tree):
        self.topo = topo
        self.in_tree = in_tree
        ne = topo.nedges
        part = np.full(ne, CLS_R, dtype=np.int64)
        for e in range(ne):
            if topo.cls[e] == D:
                part[e] = CLS_D
            elif in_tree[e] and not topo.c_owned[e]:
                part[e] = GAUGE_E
            elif topo.cls[e] == WB or (in_tree[e] and topo.c_owned[e] and topo.i_owned[e]):
                part[e] = CLS_P
        self.part = part
        self.primal_edges = np.nonzero(part == CLS_P)[0]
        self.group_of_edge = -np.ones(ne, dtype=np.int64)
        self.group_of_edge[self.primal_edges] = np.arange(len(self.primal_edges))
        r_edges = np.nonzero(part == CLS_R)[0]
        nown = np.array([len(topo.owners[e]) for e in range(ne)])
        assert np.all(nown[r_edges] <= 2), "an r-DOF with more than two owners"
        self.lam_edges = r_edges[nown[r_edges] == 2]
        self.m = len(self.lam_edges)
        self.nc = len(self.primal_edges)

        P = topo.n_patches
        self.r_i, self.r_b, self.p_loc, self.p_grp, self.e_loc = [], [], [], [], []
        lam_of_edge = -np.ones(ne, dtype=np.int64)
        lam_of_edge[self.lam_edges] = np.arange(self.m)
        self.lam_plus = np.zeros((self.m, 2), dtype=np.int64)   # (patch, local index into r ordering)
        self.lam_minus = np.zeros((self.m, 2), dtype=np.int64)
        for s in range(P):
            g = topo.l2g[s]
            cl = part[g]
            ri = [a for a in range(len(g)) if cl[a] == CLS_R and nown[g[a]] == 1]
            rb = [a for a in range(len(g)) if cl[a] == CLS_R and nown[g[a]] == 2]
            # b-DOFs ordered by their multiplier index (ascending glued id)
            rb.sort(key=lambda a: lam_of_edge[g[a]])
            pl = [a for a in range(len(g)) if cl[a] == CLS_P]
            el = [a for a in range(len(g)) if cl[a] in (CLS_D, GAUGE_E)]
            self.r_i.append(np.array(ri, dtype=np.int64))
            self.r_b.append(np.array(rb, dtype=np.int64))
            self.p_loc.append(np.array(pl, dtype=np.int64))
            self.p_grp.append(self.group_of_edge[g[pl]] if pl else np.zeros(0, dtype=np.int64))
            self.e_loc.append(np.array(el, dtype=np.int64))
            for pos, a in enumerate(rb):
                k = lam_of_edge[g[a]]
                owners = topo.owners[g[a]]
                if s == min(owners):
                    self.lam_plus[k] = (s, len(ri) + pos)
                else:
                    self.lam_minus[k] = (s, len(ri) + pos)

    def r_order(self, s):
        """Local ids of patch s's remaining DOFs in [i; b] order."""
        return np.concatenate([self.r_i[s], self.r_b[s]])

    def counts(self):
        return dict(E=int(np.sum((self.part == CLS_D) | (self.part == GAUGE_E))),
                    D=int(np.sum(self.part == CLS_D)), GAUGE=int(np.sum(self.part == GAUGE_E)),
                    P=int(self.nc), R=int(np.sum(self.part == CLS_R)), m=int(self.m))
