"""Per-level structure of the sparse coarse tree (needs setup on a GPU)."""
import os, sys, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, workloads, paper_2510_23446_b200 as tcg
L = tcg.lib(); L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
for name in sys.argv[1:] or ["cfg4"]:
    s = tcg.Solver().configure(workloads.get(name)); s.setup(); nn = s.info()["coarse_nodes"]
    out = np.zeros(5 * nn); L.tcg_debug_array(s.h, 9, 0, out.ctypes.data_as(C.POINTER(C.c_double)), 5 * nn)
    t = out.reshape(nn, 5); s.close()
    print(name, "nodes", nn)
    for h in range(int(t[:, 0].max()) + 1):
        m = t[:, 0] == h
        v, b, tv, tb = t[m, 1], t[m, 2], t[m, 3], t[m, 4]
        byt = 8 * (v * (v + 1) / 2 + v * b)
        print(f"  height {h}: nodes {int(m.sum())} fw items {int((tv + tb).sum())} bw items {int(tv.sum())} maxTV {int(tv.max())} maxTB {int(tb.max())} bytes/dir {byt.sum()/1e6:.1f} MB")
