"""Small driver for ncu: setup + a few implicit-Euler steps of one config (no timing)."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
import paper_2510_23446_b200 as tcg
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="cfg2"); ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
pr = workloads.get(a.config)
s = tcg.Solver().configure(pr); s.setup(); s.step(a.steps)
it, fr, h = s.history(); inf = s.info()
print("iters", list(map(int, it)), "launches", inf["kernel_launches"], "ms_factor", inf["ms_factor"], "ms_steps", inf["ms_steps"])
s.close()
