"""The paper's own experiment on the GPU: the two-patch cube with
the prescribed A = e^-t S, inhomogeneous Dirichlet lifting and A(0) from the commuting spline
projection (R21), against the oracle (oracle/paper_mms.py: same definitions, plain
numpy), and the convergence rates the paper states: eps_B, eps_E = O(h^p + n_t^-1)."""
import copy
import math

import numpy as np
import pytest

import workloads
from oracle.ietidp import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tcg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2510_23446_b200 import build
    build.build()
    import paper_2510_23446_b200 as pkg
    return pkg


def run_gpu(tcg, pr):
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(pr.n_steps)
    a1 = s.coefficients(1)
    it = s.history()[0]
    eb, ee, per = s.errors(per_step=True)
    nc = s.info()["n_c"]
    s.close()
    return a1, list(map(int, it)), eb, ee, per, nc


@pytest.mark.parametrize("p,divs,nt", [(1, 4, 6), (2, 4, 5), (3, 2, 4), (2, 6, 3)])
def test_paper_problem_matches_oracle(tcg, p, divs, nt):
    """Coefficients (layout 1: glued, Dirichlet DOFs = the lifting), iterations and the
    per-step error norms against the oracle at the parity tolerance (PCG rtol 1e-10)."""
    pr = workloads.paper(p, divs, nt)
    pr.rtol = 1e-10
    a1, it, eb, ee, per, nc = run_gpu(tcg, copy.deepcopy(pr))
    o = Oracle(copy.deepcopy(pr)).run()
    ref = o.coefficients(1)
    err = np.linalg.norm(a1 - ref) / np.linalg.norm(ref)
    assert err <= 1e-8, (err, it, o.iters)
    assert all(abs(x - y) <= 1 for x, y in zip(it, o.iters)), (it, o.iters)
    ops = np.array(o.errors.per_step)
    assert np.allclose(per, ops, rtol=1e-6, atol=1e-14 * ops.max()), (per, ops)
    assert abs(eb - o.errors.eps_B) <= 1e-6 * o.errors.eps_B and abs(ee - o.errors.eps_E) <= 1e-6 * o.errors.eps_E
    assert nc == (divs + p - 2) ** 2  # Fig. 1(g) primal count


def test_paper_tolerance_errors_match_oracle(tcg):
    """At the paper's own PCG tolerance 1e-6 and without scaling the error
    norms still agree with the oracle's (same iterates)."""
    pr = workloads.paper(2, 4, 8)
    _, it, eb, ee, _, _ = run_gpu(tcg, copy.deepcopy(pr))
    o = Oracle(copy.deepcopy(pr)).run()
    assert it == o.iters
    assert abs(eb - o.errors.eps_B) <= 1e-8 * o.errors.eps_B and abs(ee - o.errors.eps_E) <= 1e-8 * o.errors.eps_E


@pytest.mark.parametrize("p", [1, 2])
def test_paper_space_rate_gpu(tcg, p):
    """eps_B = O(h^p) (Fig. 1(b)): divs 4 -> 8, n_t = 512 (time error well below the
    space error); observed order within 0.3 of p."""
    errs = []
    for d in (4, 8):
        _, _, eb, _, _, _ = run_gpu(tcg, workloads.paper(p, d, 512))
        errs.append(eb)
    rate = math.log2(errs[0] / errs[1])
    assert abs(rate - p) <= 0.3, (errs, rate)


def test_paper_time_rate_gpu(tcg):
    """eps_E = O(n_t^-1) (Fig. 1(c)): p = 3, divs 4, n_t 16 -> 32 -> 64; observed order
    within 0.1 of 1."""
    errs = [run_gpu(tcg, workloads.paper(3, 4, nt))[3] for nt in (16, 32, 64)]
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert abs(rates[-1] - 1.0) <= 0.1, (errs, rates)
