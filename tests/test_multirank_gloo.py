"""Multi-rank host logic on CPU (torch.distributed gloo, world_size 2, 127.0.0.1).

1. Every rank's C++ host plan (tcg_plan on a world=2 handle; no CUDA, no NCCL) is identical
   and the x-slab patch -> rank map partitions the patches.
2. The sharded dataflow of the GPU stepper (pcg.cu: patches owned by ranks, coarse rows owned
   by ranks as I*NR/Tc, lambda entries gathered from both interface sides) reproduces the
   un-sharded dual operator and preconditioner: each rank applies the oracle's local operators
   to its own patches only, and the values the GPU kernels read from peers are exchanged with
   gloo all_reduce. The result must equal the oracle's F(lambda) and M^-1(r).
3. Two coarse ownerships: "rows" (dense S_pp^-1, coarse row block I owned by rank I*NR/Tc,
   every rank reads the solution rows from their owners) and "replicated" (the sparse coarse
   solver on several ranks: every rank gathers the primal rows -g_s of all patches through
   the peer tables and runs the whole coarse solve itself; the solutions must be identical
   on every rank, bit for bit, and no coarse exchange follows)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _worker(rank, world, port, name, coarse, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import paper_2510_23446_b200 as tcg
        from oracle.ietidp import Oracle
        from oracle import ietidp as oi

        pr = {"cfg1": workloads.cfg1(), "aniso": workloads.custom((3, 2, 2), 2, (1, 2, 1),
              [1e3 if s % 3 == 0 else 0.0 for s in range(12)], [1.0], name="aniso")}[name]
        # ---- 1. host plan on a world-2 handle (dummy NCCL id: no setup is run) ----
        s = tcg.Solver(rank=rank, world=world, nccl_id=b"\0" * 128)
        s.configure(pr)
        s.plan()
        own = s.plan_array(tcg.PLAN_RANK_OF_PATCH, pr.n_patches)
        lam = s.plan_array(tcg.PLAN_LAMBDA, 3 * s.info()["m"])
        s.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, (own.tolist(), lam.tolist()))
        assert all(g == gathered[0] for g in gathered), "plans differ across ranks"
        assert set(own.tolist()) <= set(range(world))

        # ---- 2. sharded F and M^-1 with gloo standing in for the peer reads ----
        o = Oracle(pr)
        pt = o.part
        mine = [p for p in range(pr.n_patches) if own[p] == rank]
        rng = np.random.default_rng(7)
        lam_v = rng.standard_normal(pt.m)
        # P1 (owned patches): v_s, w_s = W_rr^-1 v_s (full solve stands in for X_bb v), -g_s
        v = o.Bt(lam_v)
        u = {p: oi._solve(o.Wrr_cf[p], v[p]) for p in mine}
        g_part = np.zeros(pt.nc)
        for p in mine:
            np.add.at(g_part, pt.p_grp[p], o.Phi[p].T @ v[p])
        g = _allreduce(g_part)                         # PC reads -g_s of every patch
        Tc = (pt.nc + 63) // 64
        pc_full = oi._solve(o.Spp_cf, g)
        if coarse == "rows":
            pc_part = np.zeros(pt.nc)                  # coarse rows owned as I*NR/Tc
            for I in range(Tc):
                if (I * world) // Tc == rank:
                    pc_part[I * 64:(I + 1) * 64] = pc_full[I * 64:(I + 1) * 64]
            pc = _allreduce(pc_part)                   # P5 reads Pc from the row owners
        else:
            pc = pc_full                               # replicated: every rank solved it whole
            allpc = [None] * world
            dist.all_gather_object(allpc, pc.tobytes())
            assert all(x == allpc[0] for x in allpc), "replicated coarse solutions differ across ranks"
        y = {p: u[p] + o.Phi[p] @ pc[pt.p_grp[p]] for p in mine}
        q_part = np.zeros(pt.m)                        # jump: both sides, possibly remote
        for k in range(pt.m):
            sp, ap = pt.lam_plus[k]
            sm, am = pt.lam_minus[k]
            if sp in y:
                q_part[k] += y[sp][ap]
            if sm in y:
                q_part[k] -= y[sm][am]
        q = _allreduce(q_part)
        ref = o.F(lam_v)
        err_f = float(np.linalg.norm(q - ref) / np.linalg.norm(ref))
        # preconditioner: u_s = B_D^T r on owned patches, S_bb u_s, weighted jump
        r = rng.standard_normal(pt.m)
        vw = o.Bt(r, o.wplus, o.wminus)
        z_part = np.zeros(pt.m)
        for p in mine:
            ni = len(pt.r_i[p])
            w = np.zeros(o.nr(p))
            w[ni:] = o.Sbb_apply(p, vw[p][ni:])
            for k in range(pt.m):
                sp, ap = pt.lam_plus[k]
                sm, am = pt.lam_minus[k]
                if sp == p:
                    z_part[k] += o.wplus[k] * w[ap]
                if sm == p:
                    z_part[k] -= o.wminus[k] * w[am]
        z = _allreduce(z_part)
        zref = o.precond(r)
        err_m = float(np.linalg.norm(z - zref) / np.linalg.norm(zref))
        # scalar reductions: p^T F p = sum over ranks of sum_s v_s . y_s  (fused dot of P5)
        dot_part = sum(float(v[p] @ np.concatenate([np.zeros(len(pt.r_i[p])), y[p][len(pt.r_i[p]):]]))
                       for p in mine)
        dot = float(_allreduce(np.array([dot_part]))[0])
        err_dot = abs(dot - float(lam_v @ ref)) / abs(float(lam_v @ ref))
        out_q.put((rank, err_f, err_m, err_dot, len(mine)))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        out_q.put((rank, "error", repr(exc), 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("coarse", ["rows", "replicated"])
@pytest.mark.parametrize("name", ["cfg1", "aniso"])
def test_sharded_dataflow_gloo(name, coarse):
    from paper_2510_23446_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, coarse, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ef, em, ed, nown in res:
        assert ef != "error", em
        assert ef <= 1e-12 and em <= 1e-12 and ed <= 1e-12, (rank, ef, em, ed)
    assert sum(r[4] for r in res) == workloads.get(name).n_patches if name == "cfg1" else True
