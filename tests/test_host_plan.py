"""CPU tests of the C-ABI library (no GPU, no compute calls): it loads, exports every
symbol include/tcg_ietidp.h declares, validates arguments, and its host planning
(topology, ranked-Kruskal tree, e/p/r partition, multiplier/primal numbering; C++) is
identical to the oracle's independent Python implementation."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import workloads
from oracle import topology, gauge

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcg_ietidp.h")


@pytest.fixture(scope="module")
def tcg():
    from paper_2510_23446_b200 import build
    build.build()
    import paper_2510_23446_b200 as pkg
    return pkg


def test_exports_match_header(tcg):
    decl = set(re.findall(r"\b(tcg_[a-z_]+)\s*\(", open(HEADER).read()))
    L = tcg.lib()
    for name in decl:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", tcg.LIBPATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(tcg_[a-z_]+)\b", out))
    assert decl <= exported
    assert set(tcg.EXPORTS) == decl


def test_argument_validation(tcg):
    s = tcg.Solver()
    with pytest.raises(tcg.TcgError) as e:
        s.set_patches((0, 1, 1), (0, 0, 0), (1, 1, 1), 2, (1, 1, 1))
    assert e.value.status == tcg.TCG_EINVAL
    with pytest.raises(tcg.TcgError):
        s.set_patches((1, 1, 1), (0, 0, 0), (1, 1, 1), 0, (1, 1, 1))
    s.set_patches((2, 1, 1), (0, 0, 0), (1, 1, 1), 2, (1, 1, 1))
    with pytest.raises(tcg.TcgError):
        s.set_materials([1.0], [1.0])            # wrong length
    with pytest.raises(tcg.TcgError):
        s.set_materials([1.0, -1.0], [1.0, 1.0])  # sigma < 0
    with pytest.raises(tcg.TcgError):
        s.set_materials([1.0, 0.0], [1.0, 0.0])   # nu <= 0
    with pytest.raises(tcg.TcgError) as e:
        s.plan()                                   # materials/time missing
    assert e.value.status == tcg.TCG_ESTATE
    for k in (-1, 5):                              # warm-start subspace 0..4 (R20)
        with pytest.raises(tcg.TcgError) as e:
            s.set_warm_start(k)
        assert e.value.status == tcg.TCG_EINVAL
    s.set_warm_start(4)
    s.set_warm_start(0)
    # nonlinear reluctivity (R25): one Brauer triple per patch
    for bad in ([[0.1, 4.0, 0.9]], [[0.1, 4.0, 0.0], [0, 0, 0]], [[-0.1, 4.0, 0.9], [0, 0, 0]],
                [[0.1, -1.0, 0.9], [0, 0, 0]], [[np.nan, 1.0, 1.0], [0, 0, 0]]):
        with pytest.raises(tcg.TcgError) as e:
            s.set_nonlinear(np.array(bad, dtype=float))
        assert e.value.status == tcg.TCG_EINVAL
    for tol, mx in ((0.0, 20), (1e-8, 0)):
        with pytest.raises(tcg.TcgError) as e:
            s.set_nonlinear(np.array([[0.1, 4.0, 0.9], [0, 0, 0]]), tol, mx)
        assert e.value.status == tcg.TCG_EINVAL
    s.set_nonlinear(np.array([[0.1, 4.0, 0.9], [0, 0, 0]]))
    with pytest.raises(tcg.TcgError) as e:
        s.set_warm_start(2)                        # not with nonlinear patches
    assert e.value.status == tcg.TCG_EINVAL
    s.set_nonlinear(np.zeros((2, 3)))              # all-zero triples: linear again
    s.set_warm_start(2)
    with pytest.raises(tcg.TcgError) as e:
        s.set_nonlinear(np.array([[0.1, 4.0, 0.9], [0, 0, 0]]))
    assert e.value.status == tcg.TCG_EINVAL        # ... nor with a warm start set
    s.set_warm_start(0)
    s.set_materials([1.0, 0.0], [1.0, 1.0])
    s.set_time(1.0, 4)
    s.plan()
    with pytest.raises(tcg.TcgError) as e:
        s.set_solver(1e-10, 10, 1, 0)              # after plan
    assert e.value.status == tcg.TCG_ESTATE
    with pytest.raises(tcg.TcgError) as e:
        s.step(1)                                   # before setup
    assert e.value.status == tcg.TCG_ESTATE
    s.close()


CASES = [
    workloads.cfg1(),
    workloads.custom((1, 1, 1), 1, (2, 2, 2), [0.0], [1.0], name="single-insulator"),
    workloads.custom((3, 3, 3), 1, (2, 2, 2), [1.0 if s == 13 else 0.0 for s in range(27)], [1.0], name="floating"),
    workloads.custom((3, 2, 2), 2, (1, 2, 1), [1.0 if s % 3 == 0 else 0.0 for s in range(12)], [1.0], name="aniso"),
    workloads.cfg2(),
]


# BASELINE.json configs[2..4] at full size (tree order 0, the one every run uses)
BIG = [(workloads.cfg3, 0), (workloads.cfg4, 0), (workloads.cfg5, 0)]


@pytest.mark.parametrize("make,order", [(lambda p=p: p, o) for p in CASES for o in (0, 1)] + BIG,
                         ids=[f"{p.name}-{o}" for p in CASES for o in (0, 1)] + ["cfg3-0", "cfg4-0", "cfg5-0"])
def test_plan_matches_oracle(tcg, make, order):
    pr = make()
    pr.tree_order = order
    topo = topology.Topology(pr.npatch, pr.p, pr.elems, pr.sigma)
    tree = gauge.build_tree(topo, order)
    part = gauge.Partition(topo, tree)
    s = tcg.Solver().configure(pr)
    s.plan()
    inf = s.info()
    assert (inf["n_edges"], inf["n_verts"], inf["m"], inf["n_c"]) == (topo.nedges, topo.nverts, part.m, part.nc)
    assert np.array_equal(s.plan_array(tcg.PLAN_EDGE_CLASS, topo.nedges), topo.cls)
    reg = s.plan_array(tcg.PLAN_EDGE_REGION, topo.nedges)
    assert np.array_equal(reg & 1 > 0, topo.c_owned) and np.array_equal(reg & 2 > 0, topo.i_owned)
    assert np.array_equal(s.plan_array(tcg.PLAN_TREE, topo.nedges).astype(bool), tree)
    # partition codes: library 0 GAUGE, 1 P, 2 R, 3 D  == oracle GAUGE_E, CLS_P, CLS_R, CLS_D
    assert np.array_equal(s.plan_array(tcg.PLAN_PART, topo.nedges), part.part)
    lam = s.plan_array(tcg.PLAN_LAMBDA, 3 * part.m).reshape(-1, 3)
    assert np.array_equal(lam[:, 0], part.lam_edges)
    assert np.array_equal(lam[:, 1], part.lam_plus[:, 0]) and np.array_equal(lam[:, 2], part.lam_minus[:, 0])
    assert np.array_equal(s.plan_array(tcg.PLAN_PRIMAL, part.nc), part.primal_edges)
    cnt = s.plan_array(tcg.PLAN_PATCH_COUNTS, 3 * pr.n_patches).reshape(-1, 3)
    for p_ in range(pr.n_patches):
        assert tuple(cnt[p_]) == (len(part.r_i[p_]), len(part.r_b[p_]), len(part.p_loc[p_]))
    s.close()


def test_sharding_x_slabs_virtual(tcg):
    """Patch -> rank map: contiguous x-slabs (each rank has <= 2 neighbouring ranks)."""
    pr = workloads.cfg2()
    for world in (1, 2, 4):
        s = tcg.Solver()
        s.set_virtual_ranks(world)
        s.configure(pr)
        s.plan()
        r = s.plan_array(tcg.PLAN_RANK_OF_PATCH, pr.n_patches)
        ix = np.arange(pr.n_patches) % pr.npatch[0]
        assert np.array_equal(r, (ix * world) // pr.npatch[0])
        assert set(np.unique(r)) == set(range(min(world, pr.npatch[0])))
        s.close()
