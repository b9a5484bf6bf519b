import os, sys, ctypes as C
os.environ["TCG_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads, paper_2510_23446_b200 as tcg
L = tcg.lib(); L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
for name in sys.argv[1:] or ["cfg2"]:
    pr = workloads.get(name)
    s = tcg.Solver().configure(pr); s.setup(); s.step(2)
    out = np.zeros(528); L.tcg_debug_array(s.h, 7, 0, out.ctypes.data_as(C.POINTER(C.c_double)), 528)
    ss = out[512:522]; sd = np.diff(ss) / 1000.0
    print('  step phases us:', dict(zip(['R1 rhs','R2 fwd','R3 p0','R4 y','R5 z0','PCG loop','E1','E2','E3 bwd'], np.round(sd, 2))))
    it, _, _ = s.history(); n = int(it[-1])
    t = out[:512].reshape(64, 8)[:n, :5]
    d = np.diff(np.concatenate([t, np.roll(t[:, :1], -1, axis=0)], axis=1), axis=1)[:-1] / 1000.0
    names = ["P1 X_bb/PhiT", "PC coarse", "P5 y + pFp", "P7 symv + rz", "tail"]
    print(name, "iters", n, "mean us per phase:", {k: round(float(v), 2) for k, v in zip(names, d.mean(axis=0))}, "total/iter", round(float(d.sum(axis=1).mean()), 2))
    inf = s.info(); print("  steps ms", inf["ms_steps"], "ms/step", inf["ms_steps"] / 2)
    s.close()
