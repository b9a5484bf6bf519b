"""Pins P5, P6, P8 for the oracle's topology, tree and partition.

References: graph theory (spanning tree, gradient-kernel dimension), brute-force
enumeration, SPEC S:L377 (single insulator patch: (E,R,P) = (49,5,0)), the paper's
Fig. 1(g) primal counts for its 2-subdomain cube (slope label 1.7 between
divs 4 and 8 for p=3; counts (divs+p-2)^2 derived in SURVEY §8(c) P6), and the
exact cfg1/cfg2 counts derived by hand in SURVEY Appendix A.
"""
import math

import numpy as np
import pytest
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components

import workloads
from oracle import topology, gauge
from oracle.gauge import CLS_D, CLS_P, CLS_R, GAUGE_E


def _build(pr):
    topo = topology.Topology(pr.npatch, pr.p, pr.elems, pr.sigma)
    tree = gauge.build_tree(topo, pr.tree_order)
    return topo, tree, gauge.Partition(topo, tree)


def _edges_graph(topo, mask):
    ids = np.nonzero(mask)[0]
    ab = np.array([topo.edge_vertices(int(e)) for e in ids]).reshape(-1, 2)
    g = coo_matrix((np.ones(len(ids)), (ab[:, 0], ab[:, 1])), shape=(topo.nverts, topo.nverts))
    return g


def _conductor_vertex_info(topo, pr):
    """Vertices in the closure of some conductor patch, and the number of floating
    conductor components (components of the conductor closure not touching the boundary)."""
    n = topo.n
    Nx, Ny, Nz = topo.N
    inC = np.zeros(topo.nverts, dtype=bool)
    bnd = np.zeros(topo.nverts, dtype=bool)
    for k in range(Nz):
        for j in range(Ny):
            for i in range(Nx):
                if i in (0, Nx - 1) or j in (0, Ny - 1) or k in (0, Nz - 1):
                    bnd[topo.vertex_id(i, j, k)] = True
    for s in range(topo.n_patches):
        if pr.sigma[s] <= 0:
            continue
        ix, iy, iz = workloads.patch_coords(s, pr.npatch)
        for k in range(iz * (n[2] - 1), (iz + 1) * (n[2] - 1) + 1):
            for j in range(iy * (n[1] - 1), (iy + 1) * (n[1] - 1) + 1):
                for i in range(ix * (n[0] - 1), (ix + 1) * (n[0] - 1) + 1):
                    inC[topo.vertex_id(i, j, k)] = True
    g = _edges_graph(topo, topo.c_owned)
    ncomp, lab = connected_components(g, directed=False)
    floating = 0
    for c in np.unique(lab[inC]):
        members = (lab == c) & inC
        if not np.any(bnd[members]):
            floating += 1
    return inC, bnd, floating


CASES = [
    workloads.cfg1(),
    workloads.custom((1, 1, 1), 1, (2, 2, 2), [0.0], [1.0], name="single-insulator"),
    workloads.custom((2, 2, 2), 2, (2, 2, 2), [0, 0, 0, 0, 0, 0, 0, 1.0], [1.0], name="corner-conductor"),
    workloads.custom((3, 3, 3), 1, (2, 2, 2), [1.0 if s == 13 else 0.0 for s in range(27)], [1.0], name="floating-centre"),
    workloads.custom((3, 2, 2), 2, (1, 2, 1), [1.0 if s % 3 == 0 else 0.0 for s in range(12)], [1.0], name="aniso"),
]


@pytest.mark.parametrize("pr", CASES, ids=lambda p: p.name)
@pytest.mark.parametrize("order", [0, 1])
def test_tree_spanning_and_gauge_dimension(pr, order):
    pr.tree_order = order
    topo, tree, part = _build(pr)
    assert tree.sum() == topo.nverts - 1
    ncomp, _ = connected_components(_edges_graph(topo, tree), directed=False)
    assert ncomp == 1                      # connected with |V|-1 edges => spanning tree (acyclic)
    inC, bnd, floating = _conductor_vertex_info(topo, pr)
    strict = int(np.sum(~inC & ~bnd))
    assert part.counts()["GAUGE"] == strict + floating
    # every Dirichlet edge is eliminated; every r-DOF has at most 2 owners
    assert np.all(part.part[topo.cls == topology.D] == CLS_D)


@pytest.mark.parametrize("pr", CASES, ids=lambda p: p.name)
def test_patch_closures_connected_by_fixed_edges(pr):
    """Each patch's closure vertices are connected through its non-r edges (E u P):
    the condition for a nonsingular gauged W_rr on insulator patches (R1)."""
    topo, tree, part = _build(pr)
    for s in range(topo.n_patches):
        if pr.sigma[s] > 0:
            continue
        g = topo.l2g[s]
        fixed = g[part.part[g] != CLS_R]
        uf = gauge.UnionFind(topo.nverts)
        verts = set()
        for e in g:
            a, b = topo.edge_vertices(int(e))
            verts.update((a, b))
        for e in fixed:
            a, b = topo.edge_vertices(int(e))
            uf.union(a, b)
        roots = {uf.find(v) for v in verts}
        assert len(roots) == 1


def test_single_insulator_patch_counts():
    """single insulator patch, p=1, d=2, full Dirichlet -> (|E|,|R|,|P|) = (49,5,0)."""
    pr = workloads.custom((1, 1, 1), 1, (2, 2, 2), [0.0], [1.0])
    _, _, part = _build(pr)
    c = part.counts()
    assert (c["E"], c["R"], c["P"], c["m"]) == (49, 5, 0, 0)


def test_cfg1_exact_counts():
    """n_r C/I = 68/52, n_b 32/24, m = 112, n_c = 32, GAUGE = 50,
    glued unknowns 400 = sum n_r + n_c - m."""
    pr = workloads.cfg1()
    topo, _, part = _build(pr)
    c = part.counts()
    assert (c["m"], c["P"], c["GAUGE"]) == (112, 32, 50)
    for s in range(8):
        nr = len(part.r_i[s]) + len(part.r_b[s])
        assert (nr, len(part.r_b[s])) == ((68, 32) if pr.sigma[s] > 0 else (52, 24))
    assert c["R"] + c["P"] == 400
    assert sum(len(part.r_i[s]) + len(part.r_b[s]) for s in range(8)) + c["P"] - c["m"] == 400


def test_cfg2_counts():
    """cfg2 m = 3648, n_c = 707 (Appendix A formula with one floating conductor)."""
    _, _, part = _build(workloads.cfg2())
    assert (part.m, part.nc) == (3648, 707)


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("divs", [2, 4, 8])
def test_paper_two_subdomain_primal_count(p, divs):
    """Paper experiment: Omega=(0,1)^3 split at x=0.5 into C (x<0.5) and I.
    All Gamma tree DOFs are primal; count (divs+p-2)^2."""
    pr = workloads.custom((2, 1, 1), p, (divs // 2, divs, divs), [1.0, 0.0], [1.0, 1.0])
    _, _, part = _build(pr)
    assert part.nc == (divs + p - 2) ** 2


def test_paper_primal_slope_label():
    """Fig. 1(g) prints slope 1.7 for the primal count vs h; for p=3 between
    divs 4 and 8: log2(81/25) = 1.70."""
    counts = {}
    for divs in (4, 8):
        pr = workloads.custom((2, 1, 1), 3, (divs // 2, divs, divs), [1.0, 0.0], [1.0, 1.0])
        counts[divs] = _build(pr)[2].nc
    assert round(math.log2(counts[8] / counts[4]), 1) == 1.7


@pytest.mark.parametrize("pr", CASES, ids=lambda p: p.name)
def test_coupling_structure(pr):
    """P8: each multiplier row has one +1 (lower patch id) and one -1 on the same glued
    edge; each primal group appears in every owner of its edge."""
    topo, _, part = _build(pr)
    for k in range(part.m):
        sp, ap = part.lam_plus[k]
        sm, am = part.lam_minus[k]
        assert sp < sm
        ep = topo.l2g[sp][part.r_order(sp)[ap]]
        em = topo.l2g[sm][part.r_order(sm)[am]]
        assert ep == em == part.lam_edges[k]
        assert sorted(topo.owners[ep]) == [sp, sm]
    for gidx, e in enumerate(part.primal_edges):
        for s in topo.owners[e]:
            loc = np.nonzero(topo.l2g[s][part.p_loc[s]] == e)[0]
            assert len(loc) == 1 and part.p_grp[s][loc[0]] == gidx
