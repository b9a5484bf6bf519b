"""Failure paths and API details of the C ABI on the GPU (include/tcg_ietidp.h):
TCG_ENOCONV when PCG reaches max_iter, TCG_ENOTSPD when a pivot is not
positive (a gauging bug; forced with the TCG_DEBUG_NOTSPD test hook), the handle state
after each, source parameters against the oracle, the warm-start history restart against an
oracle whose history is cleared at the same step, and the release of device memory."""
import copy
import re

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


def test_enoconv_reports_step_iterations_relres(tcg):
    pr = workloads.cfg1()
    pr.max_iter = 3
    s = tcg.Solver().configure(pr)
    s.setup()
    with pytest.raises(tcg.TcgError) as e:
        s.step(2)
    assert e.value.status == tcg.TCG_ENOCONV
    msg = str(e.value)
    m = re.search(r"step (\d+), iterations (\d+), relres ([0-9.eE+-]+)", msg)
    assert m, msg
    assert int(m.group(1)) == 1 and int(m.group(2)) == 3
    o = Oracle(copy.deepcopy(workloads.cfg1()))
    o.step()
    # the oracle's relres after 3 iterations of the same PCG
    assert abs(float(m.group(3)) - o.hist[0][3]) <= 1e-6 * o.hist[0][3], (m.group(3), o.hist[0][3])
    with pytest.raises(tcg.TcgError) as e2:   # failed handle: only get_* / destroy
        s.step(1)
    assert e2.value.status == tcg.TCG_ESTATE
    assert s.info()["n_patches"] == 8
    s.close()


@pytest.mark.parametrize("patch", [0, 5])
def test_enotspd_reports_patch_and_pivot(tcg, monkeypatch, patch):
    monkeypatch.setenv("TCG_DEBUG_NOTSPD", str(patch))
    s = tcg.Solver().configure(workloads.cfg1())
    with pytest.raises(tcg.TcgError) as e:
        s.setup()
    assert e.value.status == tcg.TCG_ENOTSPD
    msg = str(e.value)
    assert f"patch {patch}" in msg and "pivot 0" in msg and "value -" in msg, msg
    for call in (lambda: s.step(1), lambda: s.refactor()):
        with pytest.raises(tcg.TcgError) as e2:
            call()
        assert e2.value.status == tcg.TCG_ESTATE
    assert s.info()["m"] == 112
    s.close()


def test_source_params_match_oracle(tcg):
    """tcg_set_source params (amplitude 2.5, frequency 1.5) against the oracle's phi_s(t)."""
    pr = workloads.cfg1()
    pr.source_params = (2.5, 1.5)
    pr.n_steps = 6
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(6)
    a = s.coefficients(1)
    it = s.history()[0]
    s.close()
    o = Oracle(copy.deepcopy(pr)).run()
    ref = o.coefficients(1)
    assert np.linalg.norm(a - ref) <= 1e-8 * np.linalg.norm(ref)
    assert all(abs(int(x) - y) <= 1 for x, y in zip(it, o.iters))
    with pytest.raises(tcg.TcgError) as e:
        tcg.Solver().set_source(2, (1.0, 2.0))
    assert e.value.status == tcg.TCG_EINVAL


def test_warm_k_change_matches_oracle_with_cleared_history(tcg):
    """k = 4 for steps 1-3, then k = 2: the GPU restarts its history; the oracle does the same
    by clearing warm_W / warm_FW at that step. Iterations per step within +-1, and the
    solution after each part matches."""
    pr = copy.deepcopy(workloads.cfg1())
    pr.warm_start = 4
    o = Oracle(copy.deepcopy(pr))
    o.run(3)
    o.prob.warm_start = 2
    o.warm_W, o.warm_FW = [], []
    o.run(3)
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(3)
    s.set_warm_start(2)
    s.step(3)
    it = list(map(int, s.history()[0]))
    a = s.coefficients(1)
    s.close()
    assert all(abs(x - y) <= 1 for x, y in zip(it, o.iters)), (it, o.iters)
    assert it[3] >= it[4], it   # step 3 starts cold, step 4 from a 1-vector history
    ref = o.coefficients(1)
    assert np.linalg.norm(a - ref) <= 1e-8 * np.linalg.norm(ref)


def test_destroy_returns_device_memory(tcg):
    """The library allocates from its own pool and trims it when the last handle is released,
    so the memory is usable by other allocators (e.g. PyTorch's) afterwards."""
    import torch
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    s = tcg.Solver().configure(workloads.cfg3())
    s.setup()
    used = s.info()["device_bytes"]
    s.close()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert used > 1e9
    assert free1 >= free0 - 64 * 2**20, (free0, free1, used)
    x = torch.empty(int(used) // 8, dtype=torch.float64, device="cuda")  # the memory is reusable
    del x
