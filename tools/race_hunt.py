"""Race hunt: the exact test flow (oracle, then GPU) for cfg1 then floating-centre, sparse coarse."""
import os, sys, copy
os.environ.setdefault("TCG_COARSE", "sparse")
sys.path.insert(0, os.getcwd())
import numpy as np, workloads, paper_2510_23446_b200 as tcg
from oracle.ietidp import Oracle
fc = workloads.custom((3, 3, 3), 1, (2, 2, 2), [1.0 if s == 13 else 0.0 for s in range(27)], np.linspace(0.5, 1.5, 27),
                      n_steps=3, name="floating-centre")
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    cc = workloads.custom((2, 2, 2), 2, (2, 2, 2), [0, 0, 0, 0, 0, 0, 0, 10.0], [1, 2, 3, 4, 5, 6, 7, 8], n_steps=3,
                          name="corner-conductor")
    for pr in (workloads.cfg1(), cc, fc):
        o = Oracle(copy.deepcopy(pr)); o.run(pr.n_steps)
        s = tcg.Solver().configure(pr); s.setup(); s.step(pr.n_steps)
        a1 = s.coefficients(1); a0 = s.coefficients(0); it, fr, hist = s.history(); inf = s.info(); s.close()
        ref = o.coefficients(1)
        err = float(np.linalg.norm(a1 - ref) / np.linalg.norm(ref))
        print(rep, pr.name, list(map(int, it)), o.iters, f"{err:.2e}", flush=True)
