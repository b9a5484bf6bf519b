"""Pins of the nonlinear oracle (oracle/nonlinear.py, R25 / P22).

P:L41 ("nonlinear behavior can be modeled as a simple extension") fixes no material law; the
Brauer law and Newton's method are the readings of R25. What pins the oracle here, other than
itself:
  * closed forms for a field with constant B (representable exactly): a^T K(a) a =
    nu(b^2) b^2 vol, a^T Kt(a) a = (nu + 2 nu' b^2) b^2 vol, for two directions of B;
  * the tangent matrix is the derivative of a -> K(a) a (central finite differences);
  * a constant law (k2 = 0) reduces to the linear assembly with nu = k1 + k3 (itself pinned
    by the Kronecker closed forms, P2-P4) and the Newton oracle to the linear oracle;
  * the IETI-DP Newton oracle (rearranged right-hand side) equals textbook Newton on the glued
    conforming system with sparse direct solves (MonolithicNewton);
  * quadratic convergence of the Newton increments.
"""
import copy

import numpy as np
import pytest

import workloads
from oracle import assembly
from oracle import nonlinear as nl
from oracle.ietidp import Oracle, NoConvergence

K_LAW = (0.1, 4.0, 0.9)


def _space(p=2, el=(2, 2, 2), lo=(0.0, 0.0, 0.0), hi=(0.5, 0.5, 0.5)):
    return assembly.PatchSpace(p, el, lo, hi)


def test_brauer_derivative():
    b2 = np.linspace(0.0, 1.5, 7)
    nu, dnu = nl.brauer(b2, K_LAW)
    h = 1e-6
    fd = (nl.brauer(b2 + h, K_LAW)[0] - nl.brauer(b2 - h, K_LAW)[0]) / (2 * h)
    assert np.allclose(dnu, fd, rtol=1e-8)
    assert np.allclose(nu, 0.1 * np.exp(4.0 * b2) + 0.9)


@pytest.mark.parametrize("which", ["z", "y"])
@pytest.mark.parametrize("p", [1, 2])
def test_constant_field_closed_forms(which, p):
    """A = b(-y/2, x/2, 0) gives B = (0, 0, b); A = (0, 0, b x) gives B = (0, -b, 0). Both are
    in the spline space (the commuting projection reproduces them), so every Gauss point sees
    |B| = b and the energies have closed forms."""
    b = 0.7
    sp = _space(p=p, el=(2, 3, 2), lo=(0.1, 0.0, 0.2), hi=(0.6, 0.75, 0.5))
    vol = 0.5 * 0.75 * 0.3
    if which == "z":
        field = lambda x, y, z: (-0.5 * b * y, 0.5 * b * x, 0.0 * x)
        Bex = np.array([0.0, 0.0, b])
    else:
        field = lambda x, y, z: (0.0 * x, 0.0 * x, b * x)
        Bex = np.array([0.0, -b, 0.0])
    from oracle import paper_mms
    a = paper_mms.commuting_projection(sp, field)
    for _, _, B, _ in nl.field_B(sp, a):
        assert np.allclose(B, Bex[None, :], atol=1e-12)
    Ks, Kt = nl.patch_nonlinear_matrices(sp, a, K_LAW)
    nu, dnu = nl.brauer(b * b, K_LAW)
    assert a @ Ks @ a == pytest.approx(nu * b * b * vol, rel=1e-12)
    assert a @ Kt @ a == pytest.approx((nu + 2 * dnu * b * b) * b * b * vol, rel=1e-12)
    assert a @ (Kt - Ks) @ a == pytest.approx(2 * dnu * b ** 4 * vol, rel=1e-11)


def test_tangent_is_derivative_of_residual():
    sp = _space(p=2, el=(2, 2, 2))
    rng = np.random.default_rng(3)
    a = rng.standard_normal(sp.nloc)
    bmax = max(np.sqrt((B * B).sum(1)).max() for _, _, B, _ in nl.field_B(sp, a))
    a *= 0.8 / bmax                              # |B| <= 0.8: nu varies by a factor ~10
    v = rng.standard_normal(sp.nloc) * 0.8 / bmax
    Ks, Kt = nl.patch_nonlinear_matrices(sp, a, K_LAW)
    eps = 1e-5
    Kp, _ = nl.patch_nonlinear_matrices(sp, a + eps * v, K_LAW)
    Km, _ = nl.patch_nonlinear_matrices(sp, a - eps * v, K_LAW)
    fd = (Kp @ (a + eps * v) - Km @ (a - eps * v)) / (2 * eps)
    jv = Kt @ v
    assert np.linalg.norm(fd - jv) <= 1e-7 * np.linalg.norm(jv)
    # symmetric, and the 2 nu' B B^T term is what makes Kt differ from Ks
    assert np.allclose(Kt, Kt.T, atol=1e-13 * np.abs(Kt).max())
    assert np.linalg.norm(Kt - Ks) > 1e-3 * np.linalg.norm(Ks)


def test_constant_law_equals_linear_assembly():
    sp = _space(p=2, el=(2, 2, 3))
    a = np.random.default_rng(1).standard_normal(sp.nloc)
    k = (0.25, 0.0, 0.5)
    Ks, Kt = nl.patch_nonlinear_matrices(sp, a, k)
    K, _, _ = assembly.assemble_patch(sp, 0.75, 0.0, 0)
    assert np.allclose(Ks, K, rtol=0, atol=1e-13 * np.abs(K).max())
    assert np.allclose(Kt, K, rtol=0, atol=1e-13 * np.abs(K).max())


def test_constant_law_newton_equals_linear_oracle():
    prob = workloads.cfg1()
    prob.n_steps = 10
    cond = [s for s in range(8) if prob.sigma[s] > 0]
    pn = workloads.nonlinear(copy.deepcopy(prob), cond, k=(0.2, 0.0, 0.3))
    o = nl.NewtonOracle(pn)
    o.run(3)
    lin = copy.deepcopy(prob)
    lin.nu = lin.nu.copy()
    lin.nu[cond] = 0.5
    ol = Oracle(lin).run(3)
    ref = ol.coefficients(1)
    assert np.linalg.norm(o.coefficients(1) - ref) <= 1e-10 * np.linalg.norm(ref)
    assert o.newton_iters == [2, 2, 2]          # the second solve only confirms the first
    assert max(o.increments[1::2]) < 1e-9


@pytest.fixture(scope="module")
def nl_small():
    prob = workloads.custom((2, 2, 1), 2, (2, 2, 2), [1.0, 0.0, 1.0, 0.0], 1.0, hi=(1.0, 1.0, 0.5),
                            n_steps=8, name="nl-small")
    prob = workloads.nonlinear(prob, [0, 1], amp=4.0)
    o = nl.NewtonOracle(copy.deepcopy(prob))
    o.run(4)
    return prob, o


def test_newton_oracle_equals_monolithic_newton(nl_small):
    prob, o = nl_small
    base = nl.NewtonOracle(copy.deepcopy(prob))
    mono = nl.MonolithicNewton(base)
    for _ in range(4):
        mono.step()
    ref = mono.coefficients()
    err = np.linalg.norm(o.coefficients(1) - ref) / np.linalg.norm(ref)
    assert err <= 1e-9, err
    assert max(o.newton_iters) >= 3              # the case is really nonlinear
    assert all(abs(a - b) <= 1 for a, b in zip(o.newton_iters, mono.newton_iters))


def test_newton_quadratic_convergence(nl_small):
    _, o = nl_small
    # increments of the first step's solves: each at most ~ C times the square of the previous
    incs = o.increments[: o.newton_iters[0]]
    big = [x for x in incs if x > 1e-9]
    assert len(big) >= 3
    for x0, x1 in zip(big[1:], big[2:]):
        assert x1 <= 50.0 * x0 * x0, incs


def test_newton_max_iter_raises():
    prob = workloads.custom((2, 2, 1), 2, (2, 2, 2), [1.0, 0.0, 1.0, 0.0], 1.0, hi=(1.0, 1.0, 0.5), n_steps=8)
    prob = workloads.nonlinear(prob, [0, 1], amp=4.0, newton_max=1)
    with pytest.raises(NoConvergence):
        nl.NewtonOracle(prob).run(1)
