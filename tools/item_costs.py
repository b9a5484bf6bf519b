"""Measured per-item durations (PCG iteration 2, TCG_PHASE_TIMING) against the dealing's cost
model: per block, model load vs measured load; per item class, ns per modelled tile."""
import os, sys, ctypes as C, json
os.environ["TCG_PHASE_TIMING"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np, workloads, paper_2510_23446_b200 as tcg
L = tcg.lib(); L.tcg_debug_array.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_size_t]
def arr(s, what, idx, n):
    out = np.zeros(n); st = L.tcg_debug_array(s.h, what, idx, out.ctypes.data_as(C.POINTER(C.c_double)), n)
    assert st == 0, L.tcg_last_error(s.h); return out
res = {}
for name in sys.argv[1:]:
    s = tcg.Solver().configure(workloads.get(name)); s.setup(); s.step(1)
    for ph, pname in ((0, "P1"), (2, "P5"), (3, "SY")):
        it = arr(s, 11, ph, 9 * 200000)
        n = int(len(it) // 9)
        rows = it.reshape(-1, 9)
        rows = rows[: np.count_nonzero(rows.any(axis=1)) + 1]
        t = arr(s, 10, ph, 200000)[: len(rows)]
        blk, sidx, I, part, gat, Tb, Tp = (rows[:, k] for k in range(7))
        if ph == 0: model = np.where(I < Tb, I + 1, Tb)
        elif ph == 2: model = np.where(part == 1, Tp, Tb - I)
        else: model = Tb
        model = model + 2
        nbk = int(blk.max()) + 1
        ml = np.bincount(blk.astype(int), model, nbk); tl = np.bincount(blk.astype(int), t, nbk)
        print(f"{name} {pname}: items {len(rows)}, model load max/median {ml.max()/np.median(ml):.3f}, measured load max/median {tl.max()/np.median(tl):.3f}, corr(model,measured) {np.corrcoef(ml, tl)[0,1]:.3f}")
        ns_tile = t / model
        for key, mask in (("gat0", gat == 0), ("gat1", gat == 1), ("gat2", gat == 2), ("part1", part == 1), ("part0", part == 0)):
            if mask.any(): print(f"   {key}: n {int(mask.sum())} ns/model-tile median {np.median(ns_tile[mask]):.0f} p90 {np.percentile(ns_tile[mask], 90):.0f}")
        # fit t = a * model + b * gathers
        X = np.column_stack([model - 2, (gat > 0).astype(float), np.ones(len(t))])
        coef = np.linalg.lstsq(X, t, rcond=None)[0]
        print("   fit ns = %.0f * tiles + %.0f * gathers + %.0f" % tuple(coef))
        slow = np.argsort(-tl)[:4]
        for b in slow:
            m = blk == b
            print(f"   slow block {b}: measured {tl[b]/1e3:.1f} us model {ml[b]}: items", [(int(a), int(c), int(d), int(e), round(float(f)/1e3, 2)) for a, c, d, e, f in zip(sidx[m], I[m], part[m], gat[m], t[m])][:8])
    s.close()
