"""Ad-hoc GPU-vs-oracle diagnostics (prints, never asserts)."""
import copy, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from oracle.ietidp import Oracle
import paper_2510_23446_b200 as tcg

def run(pr, steps):
    t0 = time.time()
    s = tcg.Solver().configure(pr)
    try:
        s.setup()
        s.step(steps)
    except tcg.TcgError as e:
        print("GPU error:", e); return None
    a1 = s.coefficients(1); it, fr, h = s.history(); inf = s.info(); s.close()
    return a1, it, inf, time.time() - t0

cases = [(workloads.cfg1(), 3),
         (workloads.custom((1, 1, 1), 2, (2, 2, 2), [5.0], [0.5], n_steps=2, name="single-C"), 2),
         (workloads.custom((2, 1, 1), 2, (2, 2, 2), [1.0, 0.0], [1.0, 1.0], n_steps=2, name="two"), 2),
         (workloads.custom((1, 1, 1), 2, (2, 2, 2), [0.0], [1.0], n_steps=2, name="single-I"), 2)]
for pr, n in cases:
    o = Oracle(copy.deepcopy(pr)); o.run(n)
    r = run(pr, n)
    if r is None: continue
    a1, it, inf, dt = r
    ref = o.coefficients(1)
    print(pr.name, "err", np.linalg.norm(a1 - ref) / max(np.linalg.norm(ref), 1e-300), "gpu it", list(it), "oracle it", o.iters,
          "|a|", np.linalg.norm(a1), "|ref|", np.linalg.norm(ref), "t", round(dt, 2))
    print("   info", {k: inf[k] for k in ("m", "n_c", "nr_min", "nr_max", "nb_max", "np_max", "ms_assembly", "ms_factor", "ms_coarse", "ms_steps")})
