"""Phase timing of the persistent stepper (TCG_PHASE_TIMING=1, %globaltimer stamps).
Per step-0 phase (block 0) and per PCG phase; for PCG iteration 2 also the per-block
work-end stamps: 'work' = last block's work end - phase start, 'bar' = barrier release in
block 0 - last block's work end, 'spread' = last - median work end."""
import os, sys, ctypes as C
os.environ["TCG_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads, paper_2510_23446_b200 as tcg
L = tcg.lib(); L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
NT = 8 * 64 + 16 + 8 * 4096 + 8 * 64
for name in sys.argv[1:] or ["cfg2"]:
    pr = workloads.get(name)
    s = tcg.Solver().configure(pr); s.setup(); s.step(2)
    out = np.zeros(NT)
    assert L.tcg_debug_array(s.h, 7, 0, out.ctypes.data_as(C.POINTER(C.c_double)), NT) == 0, L.tcg_last_error(s.h)
    ss = out[512:522]; sd = np.diff(ss) / 1000.0
    print(name, ' step phases us:', dict(zip(['R1 rhs','R2 fwd','R3 p0','R4 y','R5 z0','PCG loop','E1','E2','E3 bwd'], np.round(sd, 2))))
    it, _, _ = s.history(); n = int(it[-1])
    t = out[:512].reshape(64, 8)[:min(n, 64), :5]
    d = np.diff(np.concatenate([t, np.roll(t[:, :1], -1, axis=0)], axis=1), axis=1)[:-1] / 1000.0
    names = ["P1 X_bb/PhiT", "PC coarse", "P5 y + pFp", "P7 symv + rz", "tail"]
    print("  iters", n, "mean us per phase:", {k: round(float(v), 2) for k, v in zip(names, d.mean(axis=0))},
          "total/iter", round(float(d.sum(axis=1).mean()), 2))
    w = out[528:528 + 8 * 4096].reshape(4096, 8)[:, :4]
    nb = int((w[:, 0] > 0).sum())
    w = w[:nb]
    start = t[2, :4]  # phase starts in block 0 (iteration 2)
    for ph in range(4):
        we = w[:, ph]
        release = t[2, ph + 1]
        print(f"  it2 {names[ph]:14s} work {1e-3*(we.max()-start[ph]):6.2f}  median-block work {1e-3*(np.median(we)-start[ph]):6.2f}"
              f"  min {1e-3*(we.min()-start[ph]):6.2f}  bar {1e-3*(release-we.max()):6.2f} us  (blocks {nb})")
    sub = out[528:528 + 8 * 4096].reshape(4096, 8)[:nb, 4:8]
    has = sub[:, 1] > 0
    if has.any():
        st = start[2]
        q = (sub[has] - st) / 1000.0
        print("  it2 P5 sub-stamps (us from phase start; max / median over item blocks): -, gather+gemv, Y-write, block_sum:",
              np.round(q.max(axis=0), 2), np.round(np.median(q, axis=0), 2), "item blocks", int(has.sum()))
    inf = s.info(); print("  steps ms", inf["ms_steps"], "ms/step", inf["ms_steps"] / 2)
    s.close()
