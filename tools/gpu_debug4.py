"""Step-level comparison: GPU rhs-stage X1 vs numpy recomputation from the oracle's W and f."""
import copy, sys, os, ctypes as C
os.environ["TCG_DEBUG_KEEP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.linalg as sla
import workloads
from oracle.ietidp import Oracle
import paper_2510_23446_b200 as tcg
L = tcg.lib()
L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
def dbg(s, what, idx, n):
    out = np.zeros(n); st = L.tcg_debug_array(s.h, what, idx, out.ctypes.data_as(C.POINTER(C.c_double)), n)
    assert st == 0, L.tcg_last_error(s.h); return out
for pr in [workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast"),
           workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, source=2, name="contrast-mms")]:
    o = Oracle(copy.deepcopy(pr))
    s = tcg.Solver().configure(pr); s.setup()
    cnt = s.plan_array(tcg.PLAN_PATCH_COUNTS, 3*pr.n_patches).reshape(-1,3)
    for step in range(3):
        a_prev = [a.copy() for a in o.a]
        o.step(); s.step(1)
        a0 = s.coefficients(0); ref0 = o.coefficients(0); nl = len(ref0)//pr.n_patches
        print(pr.name, "step", step+1, "err", np.linalg.norm(s.coefficients(1)-o.coefficients(1))/np.linalg.norm(o.coefficients(1)),
              "per patch", ["%.1e" % (np.linalg.norm(a0[p*nl:(p+1)*nl]-ref0[p*nl:(p+1)*nl])/np.linalg.norm(ref0[p*nl:(p+1)*nl])) for p in range(pr.n_patches)])
        t = (step+1)*o.dt
        for p in range(pr.n_patches):
            ni, nb, np_ = cnt[p]; Ti=-(-ni//64); Tb=-(-nb//64); Tp=-(-np_//64); T=Ti+Tb+Tp
            aug = dbg(s, 2, p, 64*T).astype(int)
            X1 = dbg(s, 4, p, 64*T)
            f = o.M[p] @ a_prev[p] / o.dt + o.source_factor(p, t) * o.jS[p]
            ridx = np.concatenate([np.arange(ni), 64*Ti + np.arange(nb)]); pidx = 64*(Ti+Tb) + np.arange(np_)
            r = aug[ridx]; pl = aug[pidx]
            W = o.W(p); Lrr = np.linalg.cholesky(W[np.ix_(r, r)])
            z = sla.solve_triangular(Lrr, f[r], lower=True)
            Lpr = sla.solve_triangular(Lrr, W[np.ix_(r, pl)], lower=True).T
            xp = f[pl] - Lpr @ z
            print("    patch", p, "z err", np.linalg.norm(X1[ridx]-z)/np.linalg.norm(z), "xp err", np.linalg.norm(X1[pidx]-xp)/max(np.linalg.norm(xp),1e-300), "|z|", np.linalg.norm(z), "|f|", np.linalg.norm(f))
    s.close()
