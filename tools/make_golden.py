#!/usr/bin/env python
"""Write oracle-only golden files for the full-size GPU parity tests.

  python tools/make_golden.py cfg3 --steps 50 [--workers N]

Imports only `oracle/` (and the seeded problem descriptions in `workloads/`): the stored
values are the oracle's, never the CUDA path's. The oracle runs as it stands (the same
arithmetic as `Oracle(prob)`), with its per-patch work spread over N host cores
(`Oracle(workers=N, lean=True)`: a process pool for assembly + local factorisations, a
thread pool for the per-patch solves; patch-ordered sums). Output
tests/golden/<cfg>_s<steps>.npz holds
  a1         final coefficient vector, layout 1 (one value per glued edge)
  iters      PCG iterations of every step
  relres     final relative residual of every step
  meta       JSON: config, steps, rtol, scaling, counts, host cores, wall times
  nonlinear workloads (prob.nl set, oracle/nonlinear.py NewtonOracle) add newton_iters (per
  step), solve_iters and increments (per linear solve); relres is then per linear solve
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402
from oracle.ietidp import Oracle  # noqa: E402
from oracle.nonlinear import NewtonOracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--steps", type=int, required=True)
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    args = ap.parse_args()
    prob = workloads.get(args.config)
    t0 = time.perf_counter()
    if prob.nl is not None:  # nonlinear workloads: Newton oracle, full storage
        o = NewtonOracle(prob, workers=args.workers)
    else:
        o = Oracle(prob, workers=args.workers, lean=True)
    t_setup = time.perf_counter() - t0
    print(f"{args.config}: setup {t_setup:.1f} s (m={o.part.m}, n_c={o.part.nc})", flush=True)
    t_steps = []
    for k in range(args.steps):
        t1 = time.perf_counter()
        o.step()
        t_steps.append(time.perf_counter() - t1)
        print(f"  step {k + 1}/{args.steps}: {o.iters[-1]} iterations, relres {o.hist[-1][-1]:.3e}, "
              f"{t_steps[-1]:.1f} s", flush=True)
    a1 = o.coefficients(1)
    meta = {"config": args.config, "steps": args.steps, "rtol": prob.rtol, "scaling": prob.scaling,
            "n_patches": prob.n_patches, "m": int(o.part.m), "n_c": int(o.part.nc), "n_edges": int(o.topo.nedges),
            "workers": args.workers, "host_cores": len(os.sched_getaffinity(0)), "setup_s": t_setup,
            "step_s": t_steps, "writer": "tools/make_golden.py (oracle only)"}
    os.makedirs(args.out, exist_ok=True)
    path = os.path.join(args.out, f"{args.config}_s{args.steps}.npz")
    extra = {}
    if prob.nl is not None:
        extra = dict(newton_iters=np.array(o.newton_iters, dtype=np.int32),
                     solve_iters=np.array(o.solve_iters, dtype=np.int32), increments=np.array(o.increments))
    np.savez_compressed(path, a1=a1, iters=np.array(o.iters, dtype=np.int32),
                        relres=np.array([h[-1] for h in o.hist]), meta=np.array(json.dumps(meta)), **extra)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    main()
