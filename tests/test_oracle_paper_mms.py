"""Pins of the oracle's version of the paper's own experiment (§4; SURVEY §8(f) f3;
oracle/paper_mms.py): the prescribed field and its closed forms, the commuting spline
projection that supplies the inhomogeneous Dirichlet lifting and the initial condition
(R21), and the convergence rates the paper states and plots:
eps_E = O(h^p + n_t^-1), eps_B = O(h^p + n_t^-1) (Fig. 1(a)-(d)), plus the primal
count of Fig. 1(g)."""
import math

import numpy as np
import pytest

import workloads
from oracle import assembly, paper_mms, splines
from oracle.ietidp import Oracle


def _fd_curl(F, x, y, z, h=1e-5):
    def d(c, ax):
        e = [0.0, 0.0, 0.0]
        e[ax] = h
        return (F(x + e[0], y + e[1], z + e[2])[c] - F(x - e[0], y - e[1], z - e[2])[c]) / (2 * h)
    return (d(2, 1) - d(1, 2), d(0, 2) - d(2, 0), d(1, 0) - d(0, 1))


def test_prescribed_field_identities():
    """div S = 0, curl S = the closed form used for B, curl curl S = 3 S (so J = e^-t (3 nu -
    sigma) S), checked by central differences at random points."""
    rng = np.random.default_rng(0)
    x, y, z = rng.uniform(0, 1, (3, 20))
    h = 1e-5
    div = sum((paper_mms.S(*(np.array([x, y, z]) + h * np.eye(3)[c][:, None]))[c]
               - paper_mms.S(*(np.array([x, y, z]) - h * np.eye(3)[c][:, None]))[c]) / (2 * h) for c in range(3))
    assert np.max(np.abs(div)) <= 1e-8
    cs = _fd_curl(paper_mms.S, x, y, z)
    ce = paper_mms.curlS(x, y, z)
    for c in range(3):
        assert np.max(np.abs(cs[c] - ce[c])) <= 1e-8
    ccs = _fd_curl(paper_mms.curlS, x, y, z, 1e-4)
    se = paper_mms.S(x, y, z)
    for c in range(3):
        assert np.max(np.abs(ccs[c] - 3 * se[c])) <= 1e-6
    assert assembly.source_time_factor(3, 0.5, 2.0, 1.0) == pytest.approx(math.exp(-0.5) * (6.0 - 1.0), rel=1e-15)


def _eval_field(space, coef):
    """The discrete field sum_a coef_a w_a as a callable (pointwise spline evaluation)."""
    n = space.n
    p = space.p

    def F(X, Y, Z):
        out = []
        off = 0
        for c in range(3):
            dims = assembly.comp_dims(n, c)
            C = coef[off:off + int(np.prod(dims))].reshape(dims[2], dims[1], dims[0])
            off += int(np.prod(dims))
            vals = np.zeros(np.shape(X))
            for q, (x, y, z) in enumerate(zip(np.ravel(X), np.ravel(Y), np.ravel(Z))):
                bx = [paper_mms._bsplines_closed(space.knots[0], p, x), splines.dsplines(space.knots[0], p, min(x, space.hi[0] - 1e-15))]
                by = [paper_mms._bsplines_closed(space.knots[1], p, y), splines.dsplines(space.knots[1], p, min(y, space.hi[1] - 1e-15))]
                bz = [paper_mms._bsplines_closed(space.knots[2], p, z), splines.dsplines(space.knots[2], p, min(z, space.hi[2] - 1e-15))]
                fx = bx[1] if c == 0 else bx[0]
                fy = by[1] if c == 1 else by[0]
                fz = bz[1] if c == 2 else bz[0]
                vals.flat[q] = np.einsum("kji,k,j,i->", C, fz, fy, fx)
            out.append(vals)
        return tuple(out)
    return F


@pytest.mark.parametrize("p", [1, 2])
def test_commuting_projection_reproduces_discrete_fields(p):
    """Pi_h is a projector: applied to a field of the discrete space it returns that field's
    coefficients (interpolation / histopolation identities)."""
    sp = assembly.PatchSpace(p, (2, 1, 2), (0.0, 0.5, 0.25), (0.5, 1.0, 0.75))
    c = np.random.default_rng(p).standard_normal(sp.nloc)
    got = paper_mms.commuting_projection(sp, _eval_field(sp, c))
    assert np.max(np.abs(got - c)) <= 1e-10 * np.max(np.abs(c))


def test_commuting_projection_p1_line_integrals():
    """p = 1 (lowest order): with unit-integral D-splines an edge DOF is the line integral of
    the field's component along that edge."""
    sp = assembly.PatchSpace(1, (2, 2, 2), (0, 0, 0), (0.5, 0.5, 0.5))
    coef = paper_mms.commuting_projection(sp, paper_mms.S)
    gp, gw = splines.gauss_rule(10)
    n = sp.n
    for (c, i, j, k) in [(0, 0, 0, 0), (0, 1, 2, 1), (1, 2, 1, 0), (2, 1, 1, 1)]:
        nodes = [np.linspace(sp.lo[d], sp.hi[d], n[d]) for d in range(3)]
        idx = (i, j, k)
        a, b = nodes[c][idx[c]], nodes[c][idx[c] + 1]
        xs = 0.5 * (a + b) + 0.5 * (b - a) * gp
        pts = [xs if d == c else np.full_like(xs, nodes[d][idx[d]]) for d in range(3)]
        ref = float(np.sum(0.5 * (b - a) * gw * paper_mms.S(*pts)[c]))
        assert coef[assembly.local_index(n, c, i, j, k)] == pytest.approx(ref, rel=1e-12, abs=1e-14)


def test_projection_values_agree_across_an_interface():
    """A DOF shared by two patches gets the same value from either patch (the lifting and the
    initial condition are continuous), here on the paper's x = 1/2 interface."""
    pr = workloads.paper(2, 4, 1)
    o = Oracle(pr)
    top = o.topo
    first = {}
    for s in range(pr.n_patches):
        for a, g in enumerate(top.l2g[s]):
            if g in first:
                assert abs(first[g] - o.Pi[s][a]) <= 1e-13
            else:
                first[g] = o.Pi[s][a]


@pytest.mark.parametrize("p", [1, 2])
def test_paper_space_rate(p):
    """eps_B = O(h^p) (Fig. 1(b)): divs 2 -> 4 with many time steps; observed order
    within 0.25 of p. Also the primal count of Fig. 1(g): (divs + p - 2)^2."""
    errs = []
    for d in (2, 4):
        o = Oracle(workloads.paper(p, d, 32)).run()
        errs.append(o.errors.eps_B)
        assert o.part.nc == (d + p - 2) ** 2
    rate = math.log2(errs[0] / errs[1])
    assert abs(rate - p) <= 0.25, (errs, rate)


def test_paper_time_rate():
    """eps_E = O(n_t^-1) (Fig. 1(c)): p = 3, divs 2 (space error far below), n_t 4 -> 8
    -> 16; observed order within 0.15 of 1."""
    errs = []
    for nt in (4, 8, 16):
        errs.append(Oracle(workloads.paper(3, 2, nt)).run().errors.eps_E)
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert abs(rates[-1] - 1.0) <= 0.15, (errs, rates)
