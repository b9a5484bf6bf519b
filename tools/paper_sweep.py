"""The paper's Fig. 1 sweep on the GPU: for every
(deg, divs, steps) the two-patch cube with the prescribed solution (TCG_SOURCE_PAPER), PCG
without scaling at tolerance 1e-6; writes the paper's CSV columns
deg,divs,steps,errBa,errEa,iter,pri (iter = mean PCG iterations over the time steps, pri =
primal DOFs) and prints the fitted slopes.
  python tools/paper_sweep.py [out.csv]"""
import csv, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
import paper_2510_23446_b200 as tcg

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/paper_fig1_gpu.csv"
rows = []
t0 = time.time()
for deg in (1, 2, 3):
    for divs in (2, 4, 8, 16):
        for steps in (2, 8, 32, 128, 512, 2048, 8192):
            if deg == 3 and divs == 16 and steps > 2048:
                continue
            pr = workloads.paper(deg, divs, steps)
            s = tcg.Solver().configure(pr)
            s.setup()
            s.step(steps)
            eb, ee = s.errors()
            it = s.history()[0]
            rows.append(dict(deg=deg, divs=divs, steps=steps, errBa=eb, errEa=ee, iter=float(np.mean(it)),
                             pri=s.info()["n_c"]))
            s.close()
            print(rows[-1], f"{time.time() - t0:.0f}s", flush=True)
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
    w.writeheader()
    w.writerows(rows)
# slopes: time (finest space, steps 512 -> 2048), space (most steps, divs 8 -> 16)
for deg in (1, 2, 3):
    r = {(x["divs"], x["steps"]): x for x in rows if x["deg"] == deg}
    st = [(r[(16, a)], r[(16, b)]) for a, b in ((32, 128), (128, 512)) if (16, a) in r and (16, b) in r]
    sp = [(r[(a, 2048)], r[(b, 2048)]) for a, b in ((4, 8), (8, 16)) if (a, 2048) in r and (b, 2048) in r]
    for name, pairs, base in (("time", st, 4.0), ("space", sp, 2.0)):
        for x, y in pairs:
            print(f"deg {deg} {name}: eps_B slope {math.log(x['errBa'] / y['errBa'], base):.2f}, "
                  f"eps_E slope {math.log(x['errEa'] / y['errEa'], base):.2f}")
