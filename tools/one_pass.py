"""One setup + one pass (refactor + n steps) of a config: the target of ncu captures.
  python tools/one_pass.py cfg5 [n_steps [rtol]]   (rtol = 1: steps of 0 PCG iterations, the per-step fixed part)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads, paper_2510_23446_b200 as tcg
name = sys.argv[1]
pr = workloads.get(name)
n = int(sys.argv[2]) if len(sys.argv) > 2 else pr.n_steps
s = tcg.Solver().configure(pr)
if len(sys.argv) > 3:
    s.set_solver(rtol=float(sys.argv[3]))
s.setup()
s.step(n)
it = s.history()[0]
print(name, "steps", n, "iters", list(map(int, it))[:8], "ms_steps", s.info()["ms_steps"])
s.close()
