import copy, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from oracle.ietidp import Oracle
from oracle.monolithic import Monolithic
import paper_2510_23446_b200 as tcg

def gpu(pr, n):
    s = tcg.Solver().configure(pr); s.setup(); s.step(n)
    a0 = s.coefficients(0); a1 = s.coefficients(1); it, fr, h = s.history(); s.close()
    return a0, a1, it

variants = [
  workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast"),
  workloads.custom((2, 2, 1), 3, (2, 2, 2), [1.0, 0, 1.0, 0], [1, 1, 1, 1], n_steps=3, name="p3-plain"),
  workloads.custom((2, 2, 1), 2, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast-p2"),
  workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1, 1, 1, 1], n_steps=3, name="sigma-only"),
  workloads.custom((2, 2, 1), 3, (2, 2, 2), [1, 0, 1, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="nu-only"),
  workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast-rtol12"),
]
variants[-1].rtol = 1e-12
for pr in variants:
    n = pr.n_steps
    o = Oracle(copy.deepcopy(pr)); mono = Monolithic(o)
    for _ in range(n): o.step(); mono.step()
    a0, a1, it = gpu(pr, n)
    ref = o.coefficients(1); mref = mono.coefficients()
    nrm = np.linalg.norm(ref)
    print(pr.name, "gpu-oracle", np.linalg.norm(a1-ref)/nrm, "gpu-mono", np.linalg.norm(a1-mref)/nrm, "oracle-mono", np.linalg.norm(ref-mref)/nrm, list(it), o.iters)
    ref0 = o.coefficients(0); nl = len(ref0)//pr.n_patches
    print("   per patch rel err:", [float("%.2e" % (np.linalg.norm(a0[s*nl:(s+1)*nl]-ref0[s*nl:(s+1)*nl])/max(np.linalg.norm(ref0[s*nl:(s+1)*nl]),1e-300))) for s in range(pr.n_patches)])
