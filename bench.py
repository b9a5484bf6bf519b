#!/usr/bin/env python
"""bench.py — implicit-Euler steps/s of the tree-cotree IETI-DP hot path on B200.

One bench "step" = one pass of the whole hot path over one batch of synthetic input
(SURVEY §8(a) rows a2, b1, b2, c1-c3): assembly of W^_s, batched Cholesky + coarse
factorisation (tcg_refactor) and all n_t implicit-Euler steps (tcg_step(n_t)).
Default workload: cfg5 (BASELINE.json configs[4], 2048 patches, n_t = 100), the largest
configuration and the one that fits one GPU (BASELINE.json's metric names no config, so the
rule "largest single-GPU configuration" applies). value = implicit-Euler steps per second of
that whole pass (setup amortised over n_t), timed with CUDA events on the library's stream,
L2 flushed (256 MiB write) between timed steps outside the event pairs, max over ranks.

Extras on the same line (N = 1): `configs` holds cfg1-cfg4 measured the same way (fewer
passes): steps/s, PCG iterations/s, k_steps algorithmic HBM fraction, F-apply GB/s, local
factorisation TFLOP/s against the FP64 (DMMA) peak. `cpu_baseline` is the oracle on all host
cores (direct run for cfg1/cfg2, per-patch-type samples extrapolated for cfg3-cfg5).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl reference]
Under torchrun (N>1) the patches of ONE solve are sharded over the N GPUs (x-slabs; ranks
read interface/coarse/lambda values from peer memory over NVLink inside one persistent
kernel per rank; NCCL only bootstraps), value = n_t * K / max_rank_time, scaling "strong".
TCG_BENCH_REPLICAS=1 runs N independent replicas instead (scaling "weak").
"""
from __future__ import annotations

import argparse
import copy
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
METRIC = "implicit-Euler steps/s (whole pass: assembly + factorisation + n_t steps)"
# FP64 peak of the factorisation kernels (DMMA m8n8k4 == DFMA rate on B200): the builder's
# microbenchmark tools/dmma_peak.cu, profiles/round1_dmma_peak.txt (best of 8 configurations);
# nominal 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s.
FP64_PEAK_TFLOPS = 37.10


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cores():
    return len(os.sched_getaffinity(0))


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
# oracle (CPU) legs: cpu_baseline and --impl reference. The oracle as it stands (same
# arithmetic as Oracle(prob)), its per-patch work on every host core (Oracle(workers=cores)).
# ---------------------------------------------------------------------------------------
def oracle_direct(prob, n_euler, cores):
    """cfg1/cfg2: run the oracle itself: setup once + n_euler implicit-Euler steps.
    Returns (steps/s extrapolated to n_t, description, per-step seconds)."""
    from oracle.ietidp import Oracle
    t0 = time.perf_counter()
    o = Oracle(copy.deepcopy(prob), workers=cores)
    t_setup = time.perf_counter() - t0
    ts = []
    for _ in range(n_euler):
        t1 = time.perf_counter()
        o.step()
        ts.append(time.perf_counter() - t1)
    rate = prob.n_steps / (t_setup + prob.n_steps * float(np.mean(ts)))
    desc = (f"{prob.name}: oracle run directly on {cores} cores: setup {t_setup:.1f} s + {n_euler} implicit-Euler "
            f"steps ({np.mean(ts):.2f} s each), extrapolated to n_t={prob.n_steps}")
    return rate, desc, t_setup / prob.n_steps + float(np.mean(ts))


class OracleModel:
    """cfg3-cfg5: the oracle's whole run does not fit a bounded sample (cfg5: ~2048 x 5 s of
    element-loop assembly, a 36.8k dense coarse Cholesky), so it is timed piecewise on the
    full workload and extrapolated:
      plan      Oracle(prob, assemble=False): topology, tree, partition (timed whole)
      setup     local_operators (assembly + local factorisations) of `cores` sampled patches
                per class (conductor / insulator) run concurrently on `cores` processes ->
                wall per wave x ceil(#class / cores) waves
      coarse    cho_factor of an SPD matrix of size min(n_c, 3000) on `cores` BLAS threads,
                scaled by (n_c / size)^3; cho_solve scaled by (n_c / size)^2
      per step  iters x (F-apply + preconditioner) + rhs/recovery, each from the sampled
                patches' solves run concurrently on `cores` threads (waves as above) plus
                the coarse solves and the full-size B / B^T gathers
    iters = the PCG iterations per step of the GPU run of the same problem (identical to the
    oracle's within +-1, tests/test_gpu_golden.py)."""

    def __init__(self, prob, cores):
        from oracle.ietidp import Oracle
        self.prob = copy.deepcopy(prob)
        self.cores = cores
        t0 = time.perf_counter()
        self.o = Oracle(self.prob, assemble=False)
        self.t_plan = time.perf_counter() - t0
        sig = np.asarray(prob.sigma)
        self.classes = {"conductor": np.nonzero(sig > 0)[0], "insulator": np.nonzero(sig == 0)[0]}
        self._coarse = None

    def _coarse_times(self):
        if self._coarse is None:
            import scipy.linalg as sla
            from threadpoolctl import threadpool_limits
            nc = self.o.part.nc
            n = max(1, min(nc, 3000))
            rng = np.random.default_rng(0)
            A = rng.standard_normal((n, n))
            A = A @ A.T + n * np.eye(n)
            with threadpool_limits(self.cores):
                t0 = time.perf_counter()
                cf = sla.cho_factor(A, lower=True)
                tf = time.perf_counter() - t0
            b = rng.standard_normal(n)
            with threadpool_limits(1):
                t0 = time.perf_counter()
                for _ in range(5):
                    sla.cho_solve(cf, b)
                ts = (time.perf_counter() - t0) / 5
            self._coarse = (tf * (nc / n) ** 3, ts * (nc / n) ** 2)
        return self._coarse

    def sample(self):
        """One bounded sample: the component times (seconds) of the estimate. The first call
        times the per-patch setup of the sampled patches; later calls reuse those patches'
        operators and re-time only the per-step solves (keeps the reference arm's K + W steps
        within minutes)."""
        import multiprocessing as mp
        from concurrent.futures import ThreadPoolExecutor
        from threadpoolctl import threadpool_limits
        from oracle.ietidp import _local_job, _solve
        pr, pt, c = self.prob, self.o.part, self.cores
        t_setup_local, t_F, t_M, t_rhs = 0.0, 0.0, 0.0, 0.0
        if not hasattr(self, "_locs"):
            self._locs, self._t_setup_local = {}, 0.0
        for name, ids in self.classes.items():
            if len(ids) == 0:
                continue
            pick = ids[np.linspace(0, len(ids) - 1, min(c, len(ids))).astype(int)]
            jobs = [(pr, int(s), pt.r_order(s), pt.p_loc[s], len(pt.r_i[s]), self.o.dt, True) for s in pick]
            waves = math.ceil(len(ids) / c)
            with threadpool_limits(1):
                if name not in self._locs:
                    with mp.get_context("fork").Pool(len(jobs)) as pool:
                        t0 = time.perf_counter()
                        self._locs[name] = pool.map(_local_job, jobs)
                        wall = time.perf_counter() - t0
                    self._t_setup_local += wall * waves * len(pick) / len(jobs)
                locs = self._locs[name]

                def solves(loc, reps=3):
                    v = np.ones(loc["Phi"].shape[0])
                    ti = time.perf_counter()
                    for _ in range(reps):
                        _solve(loc["Wrr_cf"], v)
                        loc["Phi"].T @ v
                        loc["Phi"] @ np.ones(loc["Phi"].shape[1])
                    tF = (time.perf_counter() - ti) / reps
                    nb = loc["Wbb"].shape[0]
                    vb = np.ones(nb)
                    ti = time.perf_counter()
                    for _ in range(reps):
                        out = loc["Wbb"] @ vb
                        if loc["Wii_cf"] is not None:
                            out = out - loc["Wbi"] @ _solve(loc["Wii_cf"], loc["Wbi"].T @ vb)
                    tM = (time.perf_counter() - ti) / reps
                    return tF, tM
                reps = 3
                with ThreadPoolExecutor(len(locs)) as ex:
                    t0 = time.perf_counter()
                    res = list(ex.map(lambda lc: solves(lc, reps), locs))
                    wall_all = (time.perf_counter() - t0) / reps  # one round of solves
                tFs = np.array([r[0] for r in res])
                tMs = np.array([r[1] for r in res])
                share = tFs.sum() / max(tFs.sum() + tMs.sum(), 1e-30)
                # wall of one concurrent wave of F solves / of preconditioner solves
                t_F += wall_all * share * waves
                t_M += wall_all * (1 - share) * waves
                t_rhs += 2 * wall_all * share * waves       # x1 = W_rr^-1 f_r and the recovery solve
        tcf, tcs = self._coarse_times()
        lam = np.ones(pt.m)
        t0 = time.perf_counter()
        v = self.o.Bt(lam)
        self.o.Bj(v)
        t_B = time.perf_counter() - t0
        t_F += tcs + t_B
        t_M += t_B
        t_rhs += 2 * tcs + 2 * t_B
        t_setup_local = self._t_setup_local
        return {"t_plan": self.t_plan, "t_setup_local": t_setup_local, "t_coarse_factor": tcf, "t_F": t_F,
                "t_M": t_M, "t_rhs": t_rhs}

    def rate(self, smp, iters_per_step):
        n_t = self.prob.n_steps
        setup = smp["t_plan"] + smp["t_setup_local"] + smp["t_coarse_factor"]
        step = iters_per_step * (smp["t_F"] + smp["t_M"]) + smp["t_rhs"]
        return n_t / (setup + n_t * step), (setup / n_t + step)

    def describe(self, smp, iters_per_step):
        return (f"{self.prob.name}: oracle timed piecewise on {self.cores} cores and extrapolated: plan "
                f"{smp['t_plan']:.1f} s (whole), local setup {smp['t_setup_local']:.1f} s (from {self.cores} "
                f"concurrent patches per class), coarse Cholesky {smp['t_coarse_factor']:.1f} s and solve (scaled from a "
                f"3000^2 sample), per step {iters_per_step:.1f} PCG iterations x (F {smp['t_F']:.2f} s + M^-1 "
                f"{smp['t_M']:.2f} s) + rhs/recovery {smp['t_rhs']:.2f} s")


def cpu_baseline(prob, iters_per_step, cores):
    if prob.name in ("cfg1", "cfg2"):
        rate, desc, _ = oracle_direct(prob, 3, cores)
        return {"value": rate, "unit": "steps/s", "cores": cores, "kind": "oracle", "sample": desc}
    m = OracleModel(prob, cores)
    smp = m.sample()
    rate, _ = m.rate(smp, iters_per_step)
    return {"value": rate, "unit": "steps/s", "cores": cores, "kind": "oracle", "sample": m.describe(smp, iters_per_step),
            "components_s": smp}


def run_reference(args, prob, world, rank):
    if rank != 0:
        return 0
    W, K = args.warmup, args.steps
    cores = host_cores()
    iters = REF_ITERS.get(prob.name, 30.0)
    vals = []
    if prob.name in ("cfg1", "cfg2"):
        from oracle.ietidp import Oracle
        t0 = time.perf_counter()
        o = Oracle(copy.deepcopy(prob), workers=cores)
        t_setup = time.perf_counter() - t0
        ts = []
        for _ in range(W + K):
            t1 = time.perf_counter()
            if o.ell >= prob.n_steps:
                o = Oracle(copy.deepcopy(prob), workers=cores, assemble=True)
            o.step()
            ts.append(time.perf_counter() - t1)
        ts = ts[W:]
        per_step = [t_setup / prob.n_steps + t for t in ts]
        desc = (f"oracle setup once ({t_setup:.1f} s) + {W}+{K} implicit-Euler steps of {prob.name} on {cores} cores; "
                f"each timed step = one Euler step + setup/n_t")
    else:
        m = OracleModel(prob, cores)
        per_step = []
        smp = None
        for i in range(W + K):
            smp = m.sample()
            if i >= W:
                per_step.append(m.rate(smp, iters)[1])
        desc = m.describe(smp, iters) + f"; {W}+{K} samples, each timed step = one sample's estimate"
    ms = 1000.0 * float(np.mean(per_step))
    value = 1000.0 / ms
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": config_desc(prob)},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# PCG iterations per step of each config (GPU == oracle within +-1, tests/test_gpu_golden.py);
# used by the reference arm, which runs without a GPU measurement of its own
REF_ITERS = {"cfg3": 28.0, "cfg4": 33.0, "cfg5": 26.0}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def local_factor_flops(s):
    """Local factorisation + inverse-factor flops (the library's formula, tcg_get_info):
    Cholesky nr^3/3 + p-row TRSM 2 nr^2 np + S^s update 2 nr np^2, then X_rr = L_rr^-1
    (nr^3/3) and X_pr (nr^2 np), per patch, unpadded."""
    import paper_2510_23446_b200 as tcg
    inf = s.info()
    cnt = s.plan_array(tcg.PLAN_PATCH_COUNTS, 3 * inf["n_patches"]).reshape(-1, 3).astype(np.float64)
    nr = cnt[:, 0] + cnt[:, 1]
    npp = cnt[:, 2]
    return float(np.sum(nr ** 3 / 3 + 2 * nr ** 2 * npp + 2 * nr * npp ** 2 + nr ** 3 / 3 + nr ** 2 * npp))


def kstep_roofline(s, one_pass, peak):
    """Algorithmic bytes of one k_steps launch (one launch = n_t steps: per step
    it x (B_F + B_M) + bytes_step_fixed) / its event-timed duration."""
    s.set_profile(7)
    one_pass()
    i2 = s.info()
    s.set_profile(0)
    it, _, _ = s.history()
    bpl = float(sum(k * (i2["bytes_fapply"] + i2["bytes_precond"]) + i2["bytes_step_fixed"] for k in it))
    us = 1000 * i2["prof_ms"] / max(i2["prof_launches"], 1)
    gbs = bpl / (us * 1e-6) / 1e9
    return {"ms_per_pass": i2["prof_ms"], "launches": i2["prof_launches"], "us_per_launch": us,
            "bytes_per_launch": bpl, "achieved": gbs, "frac": gbs / peak}


def fapply_rate(s, peak):
    inf = s.info()
    lam = np.random.default_rng(0).standard_normal(inf["m"])
    s.apply_F(lam)
    est = s.bench_fapply(2) / 2.0
    nrep = int(max(5, min(1000, 200.0 / max(est, 1e-3))))
    ms_f = s.bench_fapply(nrep)
    bf = inf["bytes_fapply"]
    gbs = bf / (ms_f / nrep * 1e-3) / 1e9
    return {"GBps": gbs, "frac": gbs / peak, "peak": peak, "us_per_apply": 1000.0 * ms_f / nrep,
            "bytes_per_apply": bf, "applies": nrep, "l2_resident": bool(bf < 60e6)}


def factor_rate(s, flops_local):
    inf = s.info()
    tf = flops_local / (inf["ms_factor"] * 1e-3) / 1e12
    return {"local_TFLOPs": tf, "frac": tf / FP64_PEAK_TFLOPS, "peak_TFLOPs": FP64_PEAK_TFLOPS,
            "ms_local": inf["ms_factor"], "ms_assembly": inf["ms_assembly"], "ms_coarse": inf["ms_coarse"],
            "local_flops": flops_local, "coarse_flops": inf["flops_factor"] - flops_local,
            "coarse_sparse": bool(inf["coarse_sparse"])}


def measure_extra(tcg, name, stream, flush, peak, passes):
    """cfg1-cfg4 beside the headline: the same pass (refactor + n_t steps), fewer repetitions."""
    import torch
    prob = workloads.get(name)
    s = tcg.Solver(stream=stream.cuda_stream).configure(prob)
    s.setup()
    n_t = prob.n_steps

    def one_pass():
        s.refactor()
        s.step(n_t)

    one_pass()
    tot = 0.0
    for _ in range(passes):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_pass()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    inf = s.info()
    it = s.history()[0]
    value = n_t * passes / (tot / 1000.0)
    out = {"workload": config_desc(prob), "steps_per_s": value, "pcg_iters_per_step": float(np.mean(it)),
           "pcg_iters_per_s": value * float(np.mean(it)), "ms_per_pass": tot / passes, "passes": passes,
           "m": inf["m"], "n_c": inf["n_c"], "k_steps": kstep_roofline(s, one_pass, peak),
           "fapply": fapply_rate(s, peak), "factor": factor_rate(s, local_factor_flops(s))}
    out["k_steps"]["l2_resident"] = out["fapply"]["l2_resident"]
    s.close()
    return out


def measure_nonlinear(tcg, name, stream, flush, passes):
    """the nonlinear workload's pass (refactor + n_t steps, each
    step Newton's method: per iterate re-assembly of the nonlinear patches' tangent matrices,
    their re-factorisation + coarse, one stepper launch), event-timed like the headline."""
    import torch
    prob = workloads.get(name)
    s = tcg.Solver(stream=stream.cuda_stream).configure(prob)
    s.setup()
    n_t = prob.n_steps

    def one_pass():
        s.refactor()
        s.step(n_t)

    one_pass()
    tot = 0.0
    num0 = 0.0
    for _ in range(passes):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_pass()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
        num0 += s.info()["ms_newton_numeric"]
    inf = s.info()
    ni, si, _ = s.newton()
    value = n_t * passes / (tot / 1000.0)
    out = {"workload": config_desc(prob) + f", {int(inf['n_nonlinear'])} nonlinear patches (Brauer {tuple(prob.nl[prob.nl.any(1)][0])}), "
                                           f"source amplitude {prob.source_params[0]}",
           "steps_per_s": value, "newton_iters_per_step": float(np.mean(ni)), "pcg_iters_per_solve": float(np.mean(si)),
           "linear_solves_per_s": value * float(np.mean(ni)), "ms_per_pass": tot / passes, "passes": passes,
           "newton_numeric_share": num0 / tot,
           "note": "per Newton iterate: k_nl_quad + k_nl_assemble + k_nl_g, re-factorisation of the nonlinear patches "
                   "and the coarse problem (newton_numeric_share of the pass), one k_steps launch; host loop per iterate"}
    s.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip cfg1-cfg4 beside the headline config")
    ap.add_argument("--extra-configs", default="cfg1,cfg2,cfg3,cfg4")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--nonlinear", default="nl2", help="nonlinear workload beside the headline (SURVEY f4); '' = none")
    args = ap.parse_args()
    t_start = time.perf_counter()
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
    it_main = s.history()[0]
    peak, peak_kind = peaks()

    # ---- roofline of the dominant kernel (separate instrumented pass) ----
    roof = None
    shares = {}
    if not args.no_roofline:
        ks = kstep_roofline(s, one_pass, peak)
        shares["k_steps"] = {k: ks[k] for k in ("ms_per_pass", "launches", "us_per_launch", "bytes_per_launch")}
        traffic, traffic_src = None, None
        for fn in ("round2_ncu_k_steps.json", "round1_ncu_k_steps.json"):
            try:  # DRAM bytes of this kernel from the committed ncu --set full capture (profiles/)
                with open(os.path.join(ROOT, "profiles", fn)) as f:
                    nc = json.load(f).get(prob.name)
                if nc and nc.get("kernel") == "k_steps":
                    traffic = nc["dram_bytes_read"] + nc["dram_bytes_write"]
                    traffic_src = f"profiles/{fn}"
                    break
            except Exception:
                pass
        roof = {"kernel": "k_steps", "bound": "hbm", "achieved": ks["achieved"], "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": ks["frac"], "traffic": traffic,
                "traffic_over_algorithmic": (traffic / ks["bytes_per_launch"]) if traffic else None,
                "share_of_pass": ks["ms_per_pass"] / (max_ms / args.steps),
                "note": "achieved = algorithmic bytes per launch (one launch = all n_t steps: per step it x (B_F + B_M) "
                        "+ bytes_step_fixed, DESIGN.md §5) / event-timed launch duration (CUDA events on the library "
                        f"stream); traffic = ncu dram__bytes_read+write of one launch ({traffic_src})"}

    # ---- F-apply (BASELINE metric's second half) and factorisation rate ----
    fap = fac = None
    if world == 1 and not args.no_roofline:
        fap = fapply_rate(s, peak)
        fap["note"] = ("q = F p in the persistent kernel (P1 row GEMVs, coarse solve, column GEMVs, jump; "
                       "4 grid barriers per apply), algorithmic bytes B_F (DESIGN.md §5) / event-timed duration")
        fac = factor_rate(s, local_factor_flops(s))
        fac["note"] = ("local batched Cholesky + inverse factors (k_potrf/k_trsm/k_update/k_xinv_row, DMMA): "
                       "unpadded flops / event-timed duration; peak = FP64 DMMA microbenchmark "
                       "(tools/dmma_peak.cu, profiles/round1_dmma_peak.txt)")

    # ---- warm start: same passes, lambda0 = projection on the last 4 solutions ----
    warm = None
    if world == 1 and not args.no_roofline:
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
                "pcg_iters_per_step": float(np.mean(it_w)), "cold_pcg_iters_per_step": float(np.mean(it_main)),
                "note": "tcg_set_warm_start(4): PCG from the Galerkin projection on the previous 4 solutions "
                        "(DESIGN.md R20), one extra preconditioner apply per step; same timing protocol as value"}
    device_gb = s.info()["device_bytes"] / 1e9
    s.close()
    del s

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
                       "coefficient readback (layout 1); wall clock, median of %d" % args.e2e_steps}

    # ---- the other configs (N = 1) ----
    extras = None
    if world == 1 and not args.no_extras:
        extras = {}
        for name in [c for c in args.extra_configs.split(",") if c and c != args.config]:
            extras[name] = measure_extra(tcg, name, stream, flush, peak, passes=3 if name != "cfg4" else 2)

    nonlin = None
    if world == 1 and not args.no_extras and args.nonlinear:
        nonlin = measure_nonlinear(tcg, args.nonlinear, stream, flush, passes=2)

    # ---- cpu baseline (oracle, rank 0, N=1 only) ----
    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        cpu = cpu_baseline(prob, float(np.mean(it_main)), host_cores())

    if rank == 0:
        iters_per_step = float(np.mean(it_main))
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": config_desc(prob), "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": (f"patch-sharded over {world} GPUs (x-slabs; NVLink peer memory, one "
                                       "persistent kernel per rank)") if sharded else
                                      ("replicas" if world > 1 else "single GPU"),
                       "patches": prob.n_patches, "m": inf["m"], "n_c": inf["n_c"],
                       "coarse": "sparse (nested dissection)" if inf["coarse_sparse"] else "dense S_pp^-1",
                       "device_GB": device_gb},
            "pcg_iters_per_s": value * iters_per_step,
            "pcg_iters_per_step": iters_per_step,
            "setup_ms": inf["ms_assembly"] + inf["ms_factor"] + inf["ms_coarse"],
            "roofline": roof, "fapply": fap, "factorisation": fac, "warm_start": warm, "kernel_shares": shares,
            "configs": extras, "nonlinear": nonlin, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "wall_s": time.perf_counter() - t_start,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
