"""Assembly-level comparison: GPU assembled W^ (aug order) vs oracle W^."""
import copy, sys, os, ctypes as C
os.environ["TCG_DEBUG_KEEP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
from oracle.ietidp import Oracle
import paper_2510_23446_b200 as tcg

L = tcg.lib()
L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
def dbg(s, what, idx, n):
    out = np.zeros(n); st = L.tcg_debug_array(s.h, what, idx, out.ctypes.data_as(C.POINTER(C.c_double)), n)
    assert st == 0, L.tcg_last_error(s.h); return out
def unpack(tp, T):
    R = 64*T; M = np.zeros((R, R))
    for I in range(T):
        for J in range(I+1):
            M[I*64:(I+1)*64, J*64:(J+1)*64] = tp[(I*(I+1)//2+J)*4096:(I*(I+1)//2+J+1)*4096].reshape(64,64)
    return M
for pr in [workloads.custom((2, 2, 1), 3, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast"),
           workloads.custom((2, 2, 1), 2, (2, 2, 2), [1e6, 0, 1e6, 0], [1e-3, 1, 1, 1e-2], n_steps=3, name="contrast-p2")]:
    o = Oracle(copy.deepcopy(pr))
    s = tcg.Solver().configure(pr); s.setup()
    inf = s.info()
    cnt = s.plan_array(tcg.PLAN_PATCH_COUNTS, 3*pr.n_patches).reshape(-1,3)
    for p in range(pr.n_patches):
        ni, nb, np_ = cnt[p]; T = -(-ni//64) + -(-nb//64) + -(-np_//64)
        aug = dbg(s, 2, p, 64*T).astype(int)
        A = unpack(dbg(s, 0, p, T*(T+1)//2*4096), T)
        W = o.W(p)
        idx = np.nonzero(aug >= 0)[0]
        Ag = np.tril(A[np.ix_(idx, idx)]); Wo = np.tril(W[np.ix_(aug[idx], aug[idx])])
        print(pr.name, "patch", p, "sigma", pr.sigma[p], "max|A-W|/max|W|", np.abs(Ag-Wo).max()/np.abs(Wo).max(),
              "max rel entry err", np.max(np.abs(Ag-Wo)/np.maximum(np.abs(Wo), 1e-300)*(np.abs(Wo)>0)))
    # coarse
    Tc = -(-inf["n_c"]//64)
    Cg = unpack(dbg(s, 3, 0, Tc*(Tc+1)//2*4096), Tc)[:inf["n_c"], :inf["n_c"]]
    Co = o.Spp
    print("coarse: max|C-S|/max|S|", np.abs(np.tril(Cg)-np.tril(Co)).max()/np.abs(Co).max(),
          "cond S", np.linalg.cond(Co))
    rel = np.abs(np.tril(Cg)-np.tril(Co))/np.maximum(np.abs(np.tril(Co)), 1e-300)
    print("  coarse max rel entry", rel[np.tril(Co)!=0].max(), "diag entries range", np.abs(np.diag(Co)).min(), np.abs(np.diag(Co)).max())
    s.close()
