import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads, paper_2510_23446_b200 as tcg
for name in sys.argv[1:]:
    pr = workloads.get(name); s = tcg.Solver().configure(pr); s.plan()
    inf = s.info(); cnt = s.plan_array(tcg.PLAN_PATCH_COUNTS, 3 * pr.n_patches).reshape(-1, 3)
    ti = -(-cnt[:, 0] // 64); tb = -(-cnt[:, 1] // 64); tp = -(-cnt[:, 2] // 64); T = ti + tb + tp
    ls = ((tb * (tb + 1) // 2 + tp * tb) * 32768).sum(); sbb = ((tb * (tb + 1) // 2) * 32768).sum()
    tc = -(-inf["n_c"] // 64); sinv = tc * tc * 32768; A = ((T * (T + 1) // 2) * 32768).sum()
    nb, npp = cnt[:, 1].astype(float), cnt[:, 2].astype(float)
    print(name, "P", pr.n_patches, "m", inf["m"], "n_c", inf["n_c"], "nb", nb.min(), nb.max(), "np", npp.min(), npp.max(),
          "nr", (cnt[:, 0] + cnt[:, 1]).min(), (cnt[:, 0] + cnt[:, 1]).max())
    print("   LS %.1f MB  Sbb %.1f MB  Sinv %.1f MB  A %.1f MB" % (ls / 1e6, sbb / 1e6, sinv / 1e6, A / 1e6))
    print("   per-iter actual reads: P1 %.1f  P5 %.1f  P7(2x offdiag) %.1f  PC %.1f  = %.1f MB;  algorithmic B_F+B_M %.1f MB" % (
        ls / 1e6, ls / 1e6, (2 * sbb - (tb * 32768).sum()) / 1e6, sinv / 1e6, (2 * ls + 2 * sbb + sinv) / 1e6,
        (inf["bytes_fapply"] + inf["bytes_precond"]) / 1e6))
    s.close()
