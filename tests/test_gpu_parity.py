"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded
inputs. Bar (BASELINE.json north_star): relative l2 error of the final coefficient vector
<= 1e-8 at PCG rtol 1e-10, PCG iteration counts within +-1 per step."""
import copy

import numpy as np
import pytest

import workloads
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


def run_gpu(tcg, pr, steps=None):
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(pr.n_steps if steps is None else steps)
    a1 = s.coefficients(1)
    a0 = s.coefficients(0)
    it, fr, hist = s.history()
    inf = s.info()
    s.close()
    return a1, a0, it, hist, inf


def compare(tcg, pr, steps=None, tol=TOL):
    pr_o = copy.deepcopy(pr)
    o = Oracle(pr_o)
    n = pr.n_steps if steps is None else steps
    o.run(n)
    a1, a0, it, hist, inf = run_gpu(tcg, pr, n)
    ref1 = o.coefficients(1)
    err = np.linalg.norm(a1 - ref1) / np.linalg.norm(ref1)
    err0 = np.linalg.norm(a0 - o.coefficients(0)) / np.linalg.norm(o.coefficients(0))
    assert err <= tol, (err, list(it), o.iters)
    assert err0 <= tol, err0
    assert np.all(np.abs(np.array(it) - np.array(o.iters)) <= 1), (list(it), o.iters)
    return err, it, o


def test_cfg1_full(tcg):
    """BJ configs[0], all 10 steps."""
    err, it, o = compare(tcg, workloads.cfg1())
    assert len(it) == 10


def test_cfg1_unscaled_paper_preconditioner(tcg):
    pr = workloads.cfg1()
    pr.scaling = 0
    compare(tcg, pr)


SMALL = [
    workloads.custom((2, 2, 2), 2, (2, 2, 2), [0, 0, 0, 0, 0, 0, 0, 10.0], [1, 2, 3, 4, 5, 6, 7, 8], n_steps=3,
                     name="corner-conductor"),
    workloads.custom((3, 3, 3), 1, (2, 2, 2), [1.0 if s == 13 else 0.0 for s in range(27)],
                     np.linspace(0.5, 1.5, 27), n_steps=3, name="floating-centre"),
    workloads.custom((3, 2, 2), 2, (1, 2, 1), [1e3 if s % 3 == 0 else 0.0 for s in range(12)], [1.0], n_steps=3,
                     name="aniso"),
    workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast"),
    workloads.custom((2, 1, 1), 2, (2, 4, 4), [1.0, 0.0], [1.0, 1.0], n_steps=4, source=workloads.SOURCE_MMS,
                     name="paper-2subdomain-mms"),
    workloads.custom((3, 3, 2), 3, (3, 3, 3), [1e6 if s < 9 else 0.0 for s in range(18)],
                     10.0 ** np.random.default_rng(0).uniform(-3, 0, 18), n_steps=3, name="p3-ragged-tiles"),
]


@pytest.mark.parametrize("pr", SMALL, ids=lambda p: p.name)
def test_small_cases(tcg, pr):
    compare(tcg, pr)


def test_single_conductor_patch_zero_iterations(tcg):
    pr = workloads.custom((1, 1, 1), 2, (2, 2, 2), [5.0], [0.5], n_steps=3)
    err, it, o = compare(tcg, pr)
    assert list(it) == [0, 0, 0]


def test_zero_source(tcg):
    pr = workloads.cfg1()
    pr.n_steps = 2
    pr.source = workloads.SOURCE_NONE
    a1, a0, it, hist, inf = run_gpu(tcg, pr)
    assert not a1.any() and list(it) == [0, 0]


def test_cfg2_steps(tcg):
    """BJ configs[1] (the bench workload): first 4 steps vs the oracle."""
    compare(tcg, workloads.cfg2(), steps=4)


def test_history_and_determinism(tcg):
    pr = workloads.cfg1()
    a, _, it1, h1, _ = run_gpu(tcg, pr, 4)
    b, _, it2, h2, _ = run_gpu(tcg, pr, 4)
    assert np.array_equal(a, b) and np.array_equal(it1, it2) and np.array_equal(h1, h2)
    o = Oracle(workloads.cfg1()).run(4)
    ref = np.concatenate([np.array(h) for h in o.hist])
    assert list(it1) == o.iters and len(ref) == len(h1)   # cfg1: identical counts, so the histories align
    big = ref > 1e-6
    assert np.all(np.abs(h1[big] - ref[big]) <= 1e-4 * ref[big])
    assert h1[0] == 1.0


def test_step_splitting_is_invariant(tcg):
    """tcg_step(n) once == tcg_step(1) n times (the persistent stepper recovers insulator
    coefficients only at the last step of a launch; nothing else may change)."""
    pr = workloads.cfg1()
    s1 = tcg.Solver().configure(pr)
    s1.setup()
    s1.step(4)
    s2 = tcg.Solver().configure(pr)
    s2.setup()
    for _ in range(4):
        s2.step(1)
    a1, a2 = s1.coefficients(0), s2.coefficients(0)
    assert np.array_equal(a1, a2)
    assert np.array_equal(s1.history()[0], s2.history()[0])
    s1.close()
    s2.close()


def test_refactor_resets(tcg):
    """tcg_refactor re-runs assembly + factorisation and restarts at t=0: identical results."""
    pr = workloads.cfg1()
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(3)
    a = s.coefficients(1)
    s.refactor()
    s.step(3)
    b = s.coefficients(1)
    assert np.array_equal(a, b)
    s.close()


def _glued_ids(pr, s):
    """Glued edge id of every local DOF of patch s (structured indexing, independent of both
    the oracle's brute-force topology and the library's plan)."""
    n = [e + pr.p for e in pr.elems]
    N = [P * (nd - 1) + 1 for P, nd in zip(pr.npatch, n)]
    ix, iy, iz = s % pr.npatch[0], (s // pr.npatch[0]) % pr.npatch[1], s // (pr.npatch[0] * pr.npatch[1])
    off, out = 0, []
    for c in range(3):
        dims = [nd - (1 if d == c else 0) for d, nd in enumerate(n)]
        edims = [Nd - (1 if d == c else 0) for d, Nd in enumerate(N)]
        k, j, i = np.meshgrid(np.arange(dims[2]), np.arange(dims[1]), np.arange(dims[0]), indexing="ij")
        gi, gj, gk = i + ix * (n[0] - 1), j + iy * (n[1] - 1), k + iz * (n[2] - 1)
        out.append(off + (gi + edims[0] * (gj + edims[1] * gk)).ravel())
        off += edims[0] * edims[1] * edims[2]
    return np.concatenate(out)


@pytest.mark.parametrize("name,samples", [("cfg3", 3), ("cfg4", 3), ("cfg5", 2)])
def test_full_size_properties(tcg, name, samples):
    """BASELINE.json configs[2..4] at full size in the bench launch configuration, two steps,
    checked by properties that hold at any size: (a) PCG reached rtol every step; (b) the two
    local copies of every interface DOF agree (the jump B a_r = 0 the multipliers enforce, up to
    the PCG tolerance); (c) on sampled patches, assembled independently by the oracle's element
    loop, the interior rows of the step-2 equation W^ a2 = M a1/dt + phi(t2) j_S hold (no
    multiplier or primal term acts there)."""
    from oracle import assembly
    pr = workloads.get(name)
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(1)
    a1 = s.coefficients(0)
    s.step(1)
    a2 = s.coefficients(0)
    it, fr, _ = s.history()
    part = s.plan_array(tcg.PLAN_PART, s.info()["n_edges"])
    s.close()
    assert np.all(fr <= pr.rtol)
    P = pr.n_patches
    nloc = len(a2) // P
    gids = [_glued_ids(pr, p) for p in range(P)]
    allg = np.concatenate(gids)
    nown = np.bincount(allg, minlength=len(part))
    # (b) interface continuity: max over b-edges of |copy_1 - copy_2| relative to max |a|
    first = np.full(len(part), np.nan)
    worst = 0.0
    for p in range(P):
        g = gids[p]
        vals = a2[p * nloc:(p + 1) * nloc]
        m = (part[g] == 2) & (nown[g] == 2)
        seen = ~np.isnan(first[g]) & m
        if seen.any():
            worst = max(worst, float(np.max(np.abs(first[g][seen] - vals[seen]))))
        newm = m & np.isnan(first[g])
        first[g[newm]] = vals[newm]
    assert worst <= 1e-6 * np.max(np.abs(a2)), worst
    # (c) interior equations on sampled patches
    rng = np.random.default_rng(1)
    picks = list(rng.choice(np.nonzero(pr.sigma > 0)[0], 1)) + list(rng.choice(np.nonzero(pr.sigma == 0)[0], samples - 1))
    t2 = 2 * pr.dt
    for p in picks:
        idx = (p % pr.npatch[0], (p // pr.npatch[0]) % pr.npatch[1], p // (pr.npatch[0] * pr.npatch[1]))
        lo = [pr.lo[d] + (pr.hi[d] - pr.lo[d]) * idx[d] / pr.npatch[d] for d in range(3)]
        hi = [pr.lo[d] + (pr.hi[d] - pr.lo[d]) * (idx[d] + 1) / pr.npatch[d] for d in range(3)]
        sp = assembly.PatchSpace(pr.p, pr.elems, lo, hi)
        K, M, jS = assembly.assemble_patch(sp, pr.nu[p], pr.sigma[p], pr.source)
        x1, x2 = a1[p * nloc:(p + 1) * nloc], a2[p * nloc:(p + 1) * nloc]
        f = M @ x1 / pr.dt + assembly.source_time_factor(pr.source, t2, pr.nu[p], pr.sigma[p]) * jS
        lhs = (K + M / pr.dt) @ x2
        g = gids[p]
        rows = (part[g] == 2) & (nown[g] == 1)
        scale = max(np.max(np.abs(f)), np.max(np.abs(lhs)))
        assert np.max(np.abs((lhs - f)[rows])) <= 1e-7 * scale, (p, np.max(np.abs((lhs - f)[rows])), scale)


@pytest.mark.parametrize("name", ["cfg3"])
def test_full_size_local_equations(tcg, name):
    """BASELINE.json configs[2] at full size, first step, checked by properties the oracle can
    evaluate patch by patch: with the oracle's own element-loop assembly of sampled patches,
    (a) interior rows of W^_s a_s = f_s (no multiplier acts there), (b) across a sampled interface
    edge the two copies agree and the summed rows balance, (c) PCG reached rtol."""
    from oracle import assembly
    pr = workloads.get(name)
    s = tcg.Solver().configure(pr)
    s.setup()
    s.step(1)
    a0 = s.coefficients(0)
    it, fr, hist = s.history()
    assert fr[0] <= pr.rtol
    nloc = len(a0) // pr.n_patches
    import copy
    from oracle.ietidp import Oracle
    o = Oracle(copy.deepcopy(pr), assemble=False)   # topology + partition only
    rng = np.random.default_rng(0)
    t = pr.dt
    for sidx in rng.choice(pr.n_patches, 3, replace=False):
        lo, hi = o.patch_box(int(sidx))
        sp = assembly.PatchSpace(pr.p, pr.elems, lo, hi)
        K, M, jS = assembly.assemble_patch(sp, pr.nu[sidx], pr.sigma[sidx], pr.source)
        W = K + M / pr.dt
        a = a0[sidx * nloc:(sidx + 1) * nloc]
        f = assembly.source_time_factor(pr.source, t, pr.nu[sidx], pr.sigma[sidx]) * jS  # a(0) = 0
        ri = o.part.r_i[sidx]
        res = (W @ a - f)[ri]
        assert np.max(np.abs(res)) <= 1e-7 * max(np.max(np.abs(f)), np.max(np.abs(W @ a)))
    s.close()


@pytest.mark.parametrize("vranks", [2, 3, 4])
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_virtual_ranks_match_single_rank(tcg, name, vranks):
    """The sharded dataflow (patches owned by ranks, remote reads through per-rank pointer
    tables, two-level barrier with fused fixed-order reductions) emulated as `vranks` ranks in
    one cooperative grid equals the single-rank solve (reduction order differs -> rounding)."""
    pr = workloads.get(name)
    steps = 3
    a1, a0, it1, h1, _ = run_gpu(tcg, pr, steps)
    s = tcg.Solver()
    s.set_virtual_ranks(vranks)
    s.configure(pr)
    s.setup()
    s.step(steps)
    b1 = s.coefficients(1)
    it2, _, _ = s.history()
    inf = s.info()
    s.close()
    assert inf["world"] == vranks
    assert np.linalg.norm(b1 - a1) <= 1e-11 * np.linalg.norm(a1)
    assert np.all(np.abs(np.array(it2) - np.array(it1)) <= 1)


@pytest.mark.parametrize("name,vranks", [("cfg1", 1), ("cfg2", 1), ("cfg2", 3), ("contrast", 1)])
def test_apply_F_matches_oracle(tcg, name, vranks):
    """The dual operator alone (tcg_fapply, the persistent kernel's F-apply mode) against the
    oracle's F = B W~^-1 B^T (full-storage solves, no shared code) on a seeded lambda."""
    pr = next(p for p in SMALL if p.name == name) if name == "contrast" else workloads.get(name)
    o = Oracle(copy.deepcopy(pr))
    lam = np.random.default_rng(7).standard_normal(o.part.m)
    ref = o.F(lam)
    s = tcg.Solver().configure(pr)
    if vranks > 1:
        s.set_virtual_ranks(vranks)
    s.setup()
    q = s.apply_F(lam)
    ms = s.bench_fapply(3)
    q2 = s.apply_F(lam)
    s.close()
    err = np.linalg.norm(q - ref) / np.linalg.norm(ref)
    assert err <= 1e-11, err
    assert np.array_equal(q, q2) and ms > 0.0


@pytest.fixture
def sparse_coarse(monkeypatch):
    """Force the nested-dissection multifrontal coarse solver for small cases."""
    monkeypatch.setenv("TCG_COARSE", "sparse")
    yield


@pytest.mark.parametrize("name", ["cfg1", "corner-conductor", "floating-centre", "contrast", "p3-ragged-tiles"])
def test_sparse_coarse_matches_oracle(tcg, sparse_coarse, name):
    """The sparse coarse path (nested dissection, multifrontal factor, per-level forward /
    backward solves in the persistent kernel) against the oracle's dense coarse Cholesky."""
    pr = workloads.cfg1() if name == "cfg1" else next(p for p in SMALL if p.name == name)
    compare(tcg, pr)


def test_sparse_coarse_cfg2_steps_and_F(tcg, sparse_coarse):
    compare(tcg, workloads.cfg2(), steps=3)
    o = Oracle(workloads.cfg2())
    lam = np.random.default_rng(3).standard_normal(o.part.m)
    s = tcg.Solver().configure(workloads.cfg2())
    s.setup()
    q = s.apply_F(lam)
    s.close()
    ref = o.F(lam)
    assert np.linalg.norm(q - ref) / np.linalg.norm(ref) <= 1e-11


@pytest.mark.parametrize("group", [0, 1])
def test_overlap_side_items_small_cases_and_F(tcg, sparse_coarse, monkeypatch, group):
    """The S_bb^-1 items as side work of the sparse coarse solve (PH_P1B, TCG_OVERLAP=1) with the
    explicit S_bb^-1 forced on: small cases end to end and the isolated F-apply against the oracle."""
    monkeypatch.setenv("TCG_SBBINV", "1")
    monkeypatch.setenv("TCG_OVERLAP", "1")
    monkeypatch.setenv("TCG_GROUP", str(group))
    compare(tcg, workloads.cfg1())
    for name in ("contrast", "p3-ragged-tiles"):
        compare(tcg, next(p for p in SMALL if p.name == name))
    o = Oracle(workloads.cfg2())
    lam = np.random.default_rng(5).standard_normal(o.part.m)
    s = tcg.Solver().configure(workloads.cfg2())
    s.setup()
    q = s.apply_F(lam)
    q2 = s.apply_F(lam)
    s.close()
    ref = o.F(lam)
    assert np.linalg.norm(q - ref) / np.linalg.norm(ref) <= 1e-11
    assert np.array_equal(q, q2)


def test_sparse_vs_dense_coarse_cfg4(tcg, monkeypatch):
    """cfg4 (n_c ~ 15.7k, sparse by default) against the dense S_pp^-1 path, first 2 steps."""
    pr = workloads.cfg4()
    res = {}
    for mode in ("sparse", "dense"):
        monkeypatch.setenv("TCG_COARSE", mode)
        a1, a0, it, hist, inf = run_gpu(tcg, pr, 2)
        res[mode] = (a1, list(it))
    a, b = res["sparse"][0], res["dense"][0]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-9
    assert all(abs(x - y) <= 1 for x, y in zip(res["sparse"][1], res["dense"][1]))


def test_back_to_back_reductions_no_race(tcg, monkeypatch):
    """Regression: P5 and P7 end in reducing barriers back to back; blocks without items run
    ahead and write the next round's partial while slow blocks still sum the previous round
    (the partials are double-buffered by round parity). Small cases leave most of the 296
    blocks idle, the sparse coarse and no shared-memory caches widen the window."""
    monkeypatch.setenv("TCG_COARSE", "sparse")
    monkeypatch.setenv("TCG_NO_SMEM_CACHE", "1")
    cc = next(p for p in SMALL if p.name == "corner-conductor")
    fc = next(p for p in SMALL if p.name == "floating-centre")
    o_it = {}
    for pr in (cc, fc):
        o = Oracle(copy.deepcopy(pr))
        o.run(pr.n_steps)
        o_it[pr.name] = (o.iters, o.coefficients(1))
    for rep in range(3):
        for pr in (cc, fc):
            a1, _, it, _, _ = run_gpu(tcg, pr)
            its, ref = o_it[pr.name]
            assert list(it) == its, (rep, pr.name, list(it), its)
            assert np.linalg.norm(a1 - ref) / np.linalg.norm(ref) <= TOL


@pytest.mark.parametrize("name,steps,vranks,k,knobs", [("cfg1", 10, 1, 4, ""), ("cfg1", 10, 1, 1, ""),
                                                       ("contrast", 6, 1, 4, ""), ("cfg2", 8, 1, 4, ""),
                                                       ("cfg2", 6, 3, 4, ""), ("insulators", 7, 1, 3, ""),
                                                       ("cfg2", 8, 1, 4, "si-group")])
def test_warm_start_matches_oracle(tcg, monkeypatch, name, steps, vranks, k, knobs):
    """Warm start (R20): the GPU's Galerkin projection on the
    previous k solutions (ring buffers, d - r products, skip-Cholesky in thread 0) against
    the oracle's warm PCG, every step; on cfg2 it saves PCG iterations against the cold start.
    'insulators' has exact starts (0 iterations after step 0), a d = 0 step (t = 1/2) and a
    rank-1 subspace; it stops at t = 7/8 (at t = 1 the solution is exactly 0). 'si-group'
    runs the item kinds of cfg5 (explicit S_bb^-1, whole-patch items) on cfg2."""
    if knobs == "si-group":
        monkeypatch.setenv("TCG_SBBINV", "1")
        monkeypatch.setenv("TCG_GROUP", "1")
    if name == "insulators":
        pr = workloads.custom((2, 2, 1), 1, (2, 2, 2), [0.0] * 4, [1.0, 2.0, 1.0, 3.0], name="insulators")
        pr.n_steps = 8
    else:
        pr = next(p for p in SMALL if p.name == name) if name == "contrast" else workloads.get(name)
    pr = copy.deepcopy(pr)
    pr.warm_start = k
    steps = min(steps, pr.n_steps)
    o = Oracle(copy.deepcopy(pr))
    o.run(steps)
    s = tcg.Solver().configure(pr)
    if vranks > 1:
        s.set_virtual_ranks(vranks)
    s.setup()
    s.step(steps)
    a1 = s.coefficients(1)
    it, _, hist = s.history()
    s.close()
    ref = o.coefficients(1)
    tol = TOL
    err = np.linalg.norm(a1 - ref) / np.linalg.norm(ref)
    print(f"warm {name} k={k}: rel err {err:.3e}")
    assert err <= tol, (err, list(it), o.iters)
    assert np.all(np.abs(np.array(it) - np.array(o.iters)) <= 1), (list(it), o.iters)
    if name == "insulators":
        assert all(i == 0 for i in it[1:]), list(it)
    if name == "cfg2":
        cold = copy.deepcopy(pr)
        cold.warm_start = 0
        c = tcg.Solver().configure(cold)
        c.setup()
        c.step(steps)
        itc = c.history()[0]
        c.close()
        assert sum(it[1:]) < sum(itc[1:]), (list(it), list(itc))


def test_sparse_coarse_dataflow_equals_level_sync(tcg, sparse_coarse, monkeypatch):
    """The dataflow ordering of the sparse coarse levels (per-node counters) changes only the
    synchronisation, not the arithmetic: bit-identical to one grid barrier per level."""
    pr = workloads.cfg2()
    out = {}
    for sync in ("0", "1"):
        monkeypatch.setenv("TCG_CF_LEVELSYNC", sync)
        a1, a0, it, hist, inf = run_gpu(tcg, pr, 3)
        out[sync] = (a1, list(it), hist)
    assert np.array_equal(out["0"][0], out["1"][0]) and out["0"][1] == out["1"][1]
    assert np.array_equal(out["0"][2], out["1"][2])


def test_warm_start_with_sparse_coarse(tcg, sparse_coarse):
    """Warm start (R20) on the sparse coarse path against the oracle's warm PCG."""
    pr = copy.deepcopy(workloads.cfg2())
    pr.warm_start = 4
    compare(tcg, pr, steps=5)


def test_warm_start_k_change_restarts_history(tcg):
    """Changing the warm-start subspace mid-run restarts the history. Against an oracle run
    whose stored solutions are cleared at the change (k = 4 for 3 steps, then k = 2 from an
    empty history): every step's iteration count within +-1 and the same final relative
    residuals, so a wrong ring slot or a history that was not reset shows up as a different
    count on the steps after the change; the first step after it equals a cold step."""
    pr = copy.deepcopy(workloads.cfg1())
    cold = Oracle(copy.deepcopy(pr))
    cold.run(6)
    pw = copy.deepcopy(pr)
    pw.warm_start = 4
    o = Oracle(pw)
    o.run(3)
    o.warm_W, o.warm_FW = [], []  # the restart the ABI documents for a change of k
    o.prob.warm_start = 2
    o.run(3)
    s = tcg.Solver().configure(pr)
    s.setup()
    s.set_warm_start(4)
    s.step(3)
    s.set_warm_start(2)
    s.step(3)
    it, rel, _ = s.history()
    it = list(map(int, it))
    a1 = s.coefficients(1)
    s.close()
    assert np.all(np.abs(np.array(it) - np.array(o.iters[:6])) <= 1), (it, o.iters)
    assert abs(it[3] - cold.iters[3]) <= 1, (it, cold.iters)  # step 3 is cold again
    assert it[4] < cold.iters[4] or it[5] < cold.iters[5], (it, cold.iters)
    ref = o.coefficients(1)
    assert np.linalg.norm(a1 - ref) / np.linalg.norm(ref) <= TOL
    refc = cold.coefficients(1)
    assert np.linalg.norm(a1 - refc) / np.linalg.norm(refc) <= TOL
