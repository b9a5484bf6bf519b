#!/usr/bin/env python
"""bench.py — implicit-Euler steps/s of the tree-cotree IETI-DP hot path on B200.

One bench "step" = one pass of the whole hot path over one batch of synthetic input
(SURVEY §8(a) rows a2, b1, b2, c1-c3): assembly of W^_s, batched Cholesky + coarse
factorisation (tcg_refactor) and all n_t implicit-Euler steps (tcg_step(n_t)) of the
configuration BASELINE.json's metric is quoted on (configs[1] = cfg2 by default).
value = implicit-Euler steps per second of that whole pass (setup amortised over n_t),
timed with CUDA events on the library's stream, L2 flushed (256 MiB write) between
timed steps outside the event pairs, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl reference]
Under torchrun (N>1) the patches of ONE solve are sharded over the N GPUs (x-slabs; ranks
read interface/coarse/lambda values from peer memory over NVLink inside one persistent
kernel per rank; NCCL only bootstraps), value = n_t * K / max_rank_time, scaling "strong".
TCG_BENCH_REPLICAS=1 runs N independent replicas instead (scaling "weak").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

KERNELS = {7: "k_steps"}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_desc(prob):
    return (f"{prob.name}: {prob.npatch[0]}x{prob.npatch[1]}x{prob.npatch[2]} patches, p={prob.p}, "
            f"{prob.elems[0]} el/patch/dir, n_t={prob.n_steps}, T={prob.T}, rtol={prob.rtol}, "
            f"scaling={'rho' if prob.scaling else 'none'}")


# ---------------------------------------------------------------------------------------
# oracle (CPU) legs: cpu_baseline and --impl reference
# ---------------------------------------------------------------------------------------
def oracle_sample(prob, n_euler):
    """Time the oracle as it stands: setup once + n_euler implicit-Euler steps, single
    thread. Returns (setup_s, [step_s...])."""
    import copy
    from threadpoolctl import threadpool_limits
    from oracle.ietidp import Oracle
    with threadpool_limits(1):
        t0 = time.perf_counter()
        o = Oracle(copy.deepcopy(prob))
        t_setup = time.perf_counter() - t0
        ts = []
        for _ in range(n_euler):
            t1 = time.perf_counter()
            o.step()
            ts.append(time.perf_counter() - t1)
    return t_setup, ts


def oracle_rate(prob, t_setup, ts):
    """Whole-run steps/s extrapolated from the sample: n_t / (setup + n_t * mean step)."""
    return prob.n_steps / (t_setup + prob.n_steps * float(np.mean(ts)))


def run_reference(args, prob, world, rank):
    if rank != 0:
        return 0
    W, K = args.warmup, args.steps
    t_setup, ts = oracle_sample(prob, W + K)
    ts = ts[W:]
    value = oracle_rate(prob, t_setup, ts)
    ms_per_step = 1000.0 * (t_setup / prob.n_steps + float(np.mean(ts)))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": config_desc(prob)},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle setup once ({t_setup:.1f} s) + {W}+{K} implicit-Euler steps of "
                                   f"{prob.name}, each timed step = one Euler step + setup/n_t"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "implicit-Euler steps/s (whole pass: assembly + factorisation + n_t steps)"


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    world, rank, local = dist_init()
    prob = workloads.get(args.config)
    if args.impl == "reference":
        return run_reference(args, prob, world, rank)

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2510_23446_b200 as tcg
    stream = torch.cuda.Stream()
    sharded = world > 1 and os.environ.get("TCG_BENCH_REPLICAS", "0") != "1"

    def make_solver(strm):
        if not sharded:
            return tcg.Solver(device=local, stream=strm)
        obj = [tcg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return tcg.Solver(device=local, rank=rank, world=world, nccl_id=obj[0], stream=strm)

    s = make_solver(stream.cuda_stream)
    s.configure(prob)
    s.setup()
    n_t = prob.n_steps
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def one_pass():
        s.refactor()
        s.step(n_t)

    for _ in range(args.warmup):
        one_pass()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = s.info()["kernel_launches"]
    clk = ClockSampler(local)
    clk.start()
    total_ms = 0.0
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)  # L2 flush outside the event pair
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_pass()
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    clocks = clk.stop()
    launches = s.info()["kernel_launches"] - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    max_ms = float(t.item())
    # sharded: one solve over all GPUs (strong scaling); replicas: one solve per GPU
    value = (1 if sharded else world) * n_t * args.steps / (max_ms / 1000.0)
    inf = s.info()

    # ---- roofline of the dominant kernel (separate instrumented passes) ----
    roof = None
    shares = {}
    if not args.no_roofline:
        peak, peak_kind = peaks()
        best = None
        for kid in KERNELS:
            s.set_profile(kid)
            one_pass()
            i2 = s.info()
            if i2["prof_launches"] > 0:
                bpl = i2["prof_bytes_per_launch"]
                if kid == 7:
                    # persistent stepper (one launch = n_t steps): per step it*(B_F+B_M) for the PCG
                    # + bytes_step_fixed (conductor forward/backward, p0/d/recovery GEMVs, z0)
                    it, _, _ = s.history()
                    bpl = float(sum(k * (i2["bytes_fapply"] + i2["bytes_precond"]) + i2["bytes_step_fixed"]
                                    for k in it))
                shares[KERNELS[kid]] = {"ms_per_pass": i2["prof_ms"], "launches": i2["prof_launches"],
                                        "us_per_launch": 1000 * i2["prof_ms"] / i2["prof_launches"],
                                        "bytes_per_launch": bpl}
                if best is None or i2["prof_ms"] > shares[KERNELS[best]]["ms_per_pass"]:
                    best = kid
        s.set_profile(0)
        if best is not None:
            b = shares[KERNELS[best]]
            achieved = b["bytes_per_launch"] / (b["us_per_launch"] * 1e-6) / 1e9
            traffic = None
            try:  # DRAM bytes of this kernel from the committed ncu --set full capture (profiles/)
                with open(os.path.join(ROOT, "profiles", "round1_ncu_k_steps.json")) as f:
                    nc = json.load(f).get(prob.name)
                if nc and KERNELS[best] == nc["kernel"]:
                    traffic = nc["dram_bytes_read"] + nc["dram_bytes_write"]
            except Exception:
                traffic = None
            roof = {"kernel": KERNELS[best], "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                    "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                    "share_of_pass": b["ms_per_pass"] / (max_ms / args.steps),
                    "note": "achieved = algorithmic bytes per launch (one launch = all n_t steps) / event-timed "
                            "launch duration; traffic = ncu DRAM bytes of that launch (profiles/round1_ncu_k_steps.json); "
                            "cfg1/cfg2 are L2-resident (effective bandwidth, latency/barrier bound)"}

    # ---- F-apply (BASELINE metric's second half): the dual operator alone, isolated loop ----
    fap = None
    if world == 1 and not args.no_roofline:
        peak, peak_kind = peaks()
        lam = np.random.default_rng(0).standard_normal(inf["m"])
        s.apply_F(lam)
        est = s.bench_fapply(2) / 2.0
        nrep = int(max(5, min(1000, 200.0 / max(est, 1e-3))))
        ms_f = s.bench_fapply(nrep)
        bf = inf["bytes_fapply"]
        gbs = bf / (ms_f / nrep * 1e-3) / 1e9
        fap = {"GBps": gbs, "frac": gbs / peak, "peak": peak, "us_per_apply": 1000.0 * ms_f / nrep,
               "bytes_per_apply": bf, "applies": nrep,
               "note": "q = F p in the persistent kernel (P1 row GEMVs, coarse S_pp^-1 GEMV, column GEMVs, jump; "
                       "4 grid barriers per apply), algorithmic bytes B_F (DESIGN.md §5) / event-timed duration"
                       + ("; working set L2-resident: effective bandwidth" if bf < 60e6 else "")}

    # ---- warm start: same passes, lambda0 = projection on the last 4 solutions ----
    # (an option, not the headline: the paper's PCG starts from lambda0 = 0)
    warm = None
    if world == 1 and not args.no_roofline:
        it_cold = s.history()[0]
        s.set_warm_start(4)
        one_pass()
        ms_w, kw = 0.0, max(1, min(3, args.steps))
        for _ in range(kw):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one_pass()
            e1.record(stream)
            e1.synchronize()
            ms_w += e0.elapsed_time(e1)
        it_w = s.history()[0]
        s.set_warm_start(0)
        warm = {"value": n_t * kw / (ms_w / 1000.0), "unit": "steps/s", "passes": kw,
                "pcg_iters_per_step": float(np.mean(it_w)), "cold_pcg_iters_per_step": float(np.mean(it_cold)),
                "note": "tcg_set_warm_start(4): PCG from the Galerkin projection on the previous 4 solutions "
                        "(DESIGN.md R20), one extra preconditioner apply per step; same timing protocol as value"}

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        tt = []
        h2d = d2h = 0
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            u = make_solver(None)
            u.configure(prob)
            u.setup()
            u.step(n_t)
            a = u.coefficients(1)
            ii = u.info()
            u.close()
            tt.append(time.perf_counter() - t0)
            h2d, d2h = ii["h2d_bytes"], ii["d2h_bytes"]
        e2e_val = (1 if sharded else world) * n_t / float(np.median(tt))
        e2e = {"value": e2e_val, "unit": "steps/s", "h2d_bytes_per_step": h2d / n_t, "d2h_bytes_per_step": d2h / n_t,
               "note": "per pass: create + host arrays + setup (plan, H2D, assembly, factorisation) + n_t steps + "
                       "coefficient readback; wall clock, median of %d" % args.e2e_steps}

    # ---- cpu baseline (oracle, rank 0, N=1 only) ----
    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        t_setup, ts = oracle_sample(prob, 3)
        cpu = {"value": oracle_rate(prob, t_setup, ts), "unit": "steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{prob.name}: oracle setup ({t_setup:.1f} s) + 3 implicit-Euler steps "
                         f"({np.mean(ts):.2f} s each), extrapolated to n_t={n_t}; single thread"}

    if rank == 0:
        iters_per_step = inf["total_iters"] / max(inf["steps_done"], 1)
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": config_desc(prob), "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": (f"patch-sharded over {world} GPUs (x-slabs; NVLink peer memory, one "
                                       "persistent kernel per rank)") if sharded else
                                      ("replicas" if world > 1 else "single GPU"),
                       "patches": prob.n_patches, "m": inf["m"], "n_c": inf["n_c"]},
            "pcg_iters_per_s": value * iters_per_step,
            "pcg_iters_per_step": iters_per_step,
            "setup_ms": inf["ms_assembly"] + inf["ms_factor"] + inf["ms_coarse"],
            "roofline": roof, "fapply": fap, "warm_start": warm, "kernel_shares": shares, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
