import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads, paper_2510_23446_b200 as tcg
import torch
torch.cuda.init()
pr = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
for rep in range(4):
    t = [time.perf_counter()]
    s = tcg.Solver(); t.append(time.perf_counter())
    s.configure(pr); t.append(time.perf_counter())
    s.plan(); t.append(time.perf_counter())
    s.setup(); t.append(time.perf_counter())
    s.step(pr.n_steps); t.append(time.perf_counter())
    a = s.coefficients(1); t.append(time.perf_counter())
    s.close(); t.append(time.perf_counter())
    d = np.diff(t) * 1000
    print("create %.1f configure %.1f plan %.1f setup %.1f step %.1f coef %.1f close %.1f  total %.1f ms" % (*d, sum(d)))
