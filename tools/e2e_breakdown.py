"""Wall-clock breakdown of one end-to-end pass through the public API (bench.py's e2e leg):
create, configure (host arrays), setup (plan, H2D, assembly, factorisation), steps, readback."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, workloads, paper_2510_23446_b200 as tcg
for name in sys.argv[1:] or ["cfg2"]:
    prob = workloads.get(name)
    for rep in range(int(os.environ.get("E2E_REPS", "4"))):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        u = tcg.Solver(device=0); t.append(time.perf_counter())
        u.configure(prob); t.append(time.perf_counter())
        u.setup(); torch.cuda.synchronize(); t.append(time.perf_counter())
        u.step(prob.n_steps); t.append(time.perf_counter())
        a = u.coefficients(1); t.append(time.perf_counter())
        inf = u.info(); u.close(); t.append(time.perf_counter())
        d = [1e3 * (b - a) for a, b in zip(t[:-1], t[1:])]
        print(name, rep, "ms: create %.2f configure %.2f setup %.2f (plan %.2f assembly %.2f factor %.2f coarse %.2f) steps %.2f readback %.2f close %.2f total %.2f"
              % (d[0], d[1], d[2], inf["ms_plan"], inf["ms_assembly"], inf["ms_factor"], inf["ms_coarse"], d[3], d[4], d[5], sum(d)))
