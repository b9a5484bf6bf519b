"""GPU parity of the nonlinear extension (R25): Brauer reluctivity
with Newton's method per implicit-Euler step, CUDA path (C ABI: nonlinear.cu + the stepper's
Newton right-hand side) against the Newton oracle (oracle/nonlinear.py, pinned in
tests/test_oracle_nonlinear.py) on the same seeded inputs. Bar as the linear path: relative l2
of the final coefficients <= 1e-8; Newton iterations per step identical; PCG iterations per
linear solve within +-1."""
import copy

import numpy as np
import pytest

import workloads
from oracle import nonlinear as onl
from oracle.ietidp import Oracle

pytestmark = pytest.mark.gpu

TOL = 1e-8


@pytest.fixture(scope="module")
def tcg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2510_23446_b200 import build
    build.build()
    import paper_2510_23446_b200 as pkg
    return pkg


def run_gpu(tcg, pr, steps, vranks=1):
    s = tcg.Solver()
    if vranks > 1:
        s.set_virtual_ranks(vranks)
    s.configure(pr)
    s.setup()
    s.step(steps)
    out = dict(a1=s.coefficients(1), a0=s.coefficients(0), hist=s.history(), newton=s.newton(), info=s.info())
    s.close()
    return out


def small():
    pr = workloads.custom((2, 2, 1), 2, (2, 2, 2), [1.0, 0.0, 1.0, 0.0], 1.0, hi=(1.0, 1.0, 0.5),
                          n_steps=8, name="nl-small")
    return workloads.nonlinear(pr, [0, 1], amp=4.0)


def compare(tcg, pr, steps, vranks=1):
    o = onl.NewtonOracle(copy.deepcopy(pr))
    o.run(steps)
    g = run_gpu(tcg, pr, steps, vranks)
    ref1, ref0 = o.coefficients(1), o.coefficients(0)
    err = np.linalg.norm(g["a1"] - ref1) / np.linalg.norm(ref1)
    err0 = np.linalg.norm(g["a0"] - ref0) / np.linalg.norm(ref0)
    ni, si, inc = g["newton"]
    assert err <= TOL and err0 <= TOL, (err, err0)
    assert list(ni) == o.newton_iters, (list(ni), o.newton_iters)
    assert len(si) == len(o.solve_iters)
    assert np.all(np.abs(si - np.array(o.solve_iters)) <= 1), (list(si), o.solve_iters)
    it, fr, hist = g["hist"]
    assert list(it) == [int(v) for v in np.add.reduceat(si, np.concatenate([[0], np.cumsum(ni)[:-1]]))]
    assert len(hist) == g["info"]["hist_len"] == int(np.sum(si + 1))
    assert g["info"]["newton_iters"] == int(np.sum(ni)) and g["info"]["n_nonlinear"] == int(np.sum(np.any(pr.nl != 0, 1)))
    return err, o, g


def test_small_nonlinear_matches_oracle(tcg):
    err, o, g = compare(tcg, small(), 4)
    assert max(o.newton_iters) >= 3     # really nonlinear
    # the Newton increments agree with the oracle's (quadratic convergence on both sides)
    inc = g["newton"][2]
    big = np.array(o.increments) > 1e-6
    assert np.allclose(inc[big], np.array(o.increments)[big], rtol=1e-5)


def test_nl1_matches_oracle(tcg):
    """cfg1 with its conductor patches nonlinear (workloads.nl1), all 10 steps."""
    compare(tcg, workloads.nl1(), 10)


def test_nonlinear_insulator_and_scaling_none(tcg):
    """nonlinear insulator patches (no mass term; the rhs path of the conductors) and the
    paper's unscaled preconditioner."""
    pr = workloads.custom((2, 2, 2), 2, (2, 2, 2), [1.0, 1.0, 1.0, 1.0, 0, 0, 0, 0], 1.0, n_steps=6, scaling=0)
    pr = workloads.nonlinear(pr, [4, 5, 6, 7], k=(0.05, 3.0, 0.5), amp=3.0)
    compare(tcg, pr, 3)


def test_nonlinear_p3(tcg):
    pr = workloads.custom((2, 1, 2), 3, (2, 2, 2), [1.0, 1.0, 0, 0], [1.0, 0.5, 1.0, 2.0], n_steps=5)
    pr = workloads.nonlinear(pr, [0, 2], amp=3.0)
    compare(tcg, pr, 2)


def test_nonlinear_virtual_ranks(tcg):
    compare(tcg, small(), 3, vranks=2)


@pytest.mark.parametrize("group", [0, 1])
def test_nonlinear_with_explicit_sbb_inverse(tcg, monkeypatch, group):
    """Newton iterates re-form S_bb^-1 for the nonlinear patches (k_sbbinv over their list);
    forced on for the small case, with row items and with whole-patch items."""
    monkeypatch.setenv("TCG_SBBINV", "1")
    monkeypatch.setenv("TCG_GROUP", str(group))
    compare(tcg, workloads.nl1(), 4)


def test_constant_law_equals_linear(tcg):
    """k2 = 0: nu = k1 + k3 everywhere on the patch; the first Newton solve is the linear
    step and the second confirms it."""
    base = workloads.cfg1()
    cond = [s for s in range(8) if base.sigma[s] > 0]
    pr = workloads.nonlinear(copy.deepcopy(base), cond, k=(0.2, 0.0, 0.3))
    g = run_gpu(tcg, pr, 4)
    lin = copy.deepcopy(base)
    lin.nu = lin.nu.copy()
    lin.nu[cond] = 0.5
    s = tcg.Solver().configure(lin)
    s.setup()
    s.step(4)
    ref = s.coefficients(1)
    s.close()
    assert np.linalg.norm(g["a1"] - ref) <= 1e-10 * np.linalg.norm(ref)
    assert list(g["newton"][0]) == [2, 2, 2, 2]


def test_newton_max_iter_fails_with_enoconv(tcg):
    pr = small()
    pr.newton_max = 1
    s = tcg.Solver().configure(pr)
    s.setup()
    with pytest.raises(tcg.TcgError) as ei:
        s.step(1)
    assert ei.value.status == tcg.TCG_ENOCONV and "Newton" in str(ei.value)
    s.close()


def test_refactor_restarts_newton(tcg):
    pr = small()
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(2)
    a = s.coefficients(1)
    ni = list(s.newton()[0])
    s.refactor()
    assert s.info()["linear_solves"] == 0
    s.step(2)
    assert np.array_equal(a, s.coefficients(1)) and list(s.newton()[0]) == ni
    s.close()


def test_nl2_golden(tcg):
    """cfg2-size nonlinear workload (workloads.nl2: 32 nonlinear patches), first 5 steps, against
    the oracle's golden file (tools/make_golden.py nl2 --steps 5, oracle only), in the bench's
    launch configuration (library defaults)."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nl2_s5.npz")
    gd = np.load(path)
    meta = json.loads(str(gd["meta"]))
    pr = workloads.nl2()
    g = run_gpu(tcg, pr, meta["steps"])
    ref = gd["a1"]
    err = np.linalg.norm(g["a1"] - ref) / np.linalg.norm(ref)
    assert err <= TOL, err
    assert np.max(np.abs(g["a1"] - ref)) <= TOL * np.max(np.abs(ref))
    ni, si, inc = g["newton"]
    assert list(ni) == list(gd["newton_iters"]), (list(ni), list(gd["newton_iters"]))
    assert np.all(np.abs(si - gd["solve_iters"]) <= 1), (list(si), list(gd["solve_iters"]))
