"""Per-block phase work (PCG iteration 2, TCG_PHASE_TIMING) against the block's SM id: is
the systematic per-block imbalance a placement effect (SM / die) or an item-cost effect?"""
import os, sys, ctypes as C
os.environ["TCG_PHASE_TIMING"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np, workloads, paper_2510_23446_b200 as tcg
L = tcg.lib(); L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
NT = 8 * 64 + 16 + 8 * 4096 + 8 * 64
for name in sys.argv[1:]:
    s = tcg.Solver().configure(workloads.get(name)); s.setup(); s.step(1)
    out = np.zeros(NT); L.tcg_debug_array(s.h, 7, 0, out.ctypes.data_as(C.POINTER(C.c_double)), NT)
    t = out[:512].reshape(64, 8)
    w = out[528:528 + 8 * 4096].reshape(4096, 8); nb = int((w[:, 0] > 0).sum()); w = w[:nb]
    sm = w[:, 4].astype(int)
    print(name, "blocks", nb, "distinct SMs", len(set(sm)), "first 12 smids", list(sm[:12]))
    for ph in range(4):
        a = (w[:, ph] - t[2, ph]) / 1e3
        lo = sm < 74
        print(" phase", ph, "median work SM<74 %.2f  SM>=74 %.2f  | slowest 8 blocks:" % (np.median(a[lo]), np.median(a[~lo])),
              [(int(b), int(sm[b]), round(float(a[b]), 1)) for b in np.argsort(-a)[:8]])
    s.close()
