"""Per-level timing of the sparse coarse solves (TCG_PHASE_TIMING=1, block-0 stamps of the
first 8 coarse solves of a launch: R3, PCG iterations, ...)."""
import os, sys, ctypes as C
os.environ["TCG_PHASE_TIMING"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np, workloads, paper_2510_23446_b200 as tcg
L = tcg.lib(); L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
NT = 8 * 64 + 16 + 8 * 4096 + 8 * 64
for name in sys.argv[1:] or ["cfg4"]:
    s = tcg.Solver().configure(workloads.get(name)); s.setup(); s.step(1)
    lv = s.info()["coarse_levels"]
    out = np.zeros(NT); L.tcg_debug_array(s.h, 7, 0, out.ctypes.data_as(C.POINTER(C.c_double)), NT)
    t = out[528 + 8 * 4096:].reshape(8, 64)[:, : 2 * lv + 1]
    d = np.diff(t, axis=1)[2:6] / 1000.0  # solves 2..5 (PCG iterations)
    m = d.mean(axis=0)
    print(name, "levels", lv, "fw per level us:", np.round(m[:lv], 1), "bw per level (top down) us:", np.round(m[lv:], 1), "total", round(float(m.sum()), 1))
    s.close()
