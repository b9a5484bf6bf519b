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
    for ph in range(4):
        a = w[:, ph] - t[2, ph]; b = w[:, 4 + ph] - t[3, ph]
        print(name, "phase", ph, "corr it2/it3 %.3f" % np.corrcoef(a, b)[0, 1], "max-med it2 %.2f it3 %.2f us" % ((a.max()-np.median(a))/1e3, (b.max()-np.median(b))/1e3),
              "top5 blocks it2", list(np.argsort(-a)[:5]), "it3", list(np.argsort(-b)[:5]))
    s.close()
