"""Setup + n isolated F-applies (k_steps mode 1) of a config: the target of ncu captures.
  python tools/fapply_only.py cfg5 [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads, paper_2510_23446_b200 as tcg
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = tcg.Solver().configure(workloads.get(name))
s.setup()
ms = s.bench_fapply(n)
inf = s.info()
print(name, "fapply n", n, "ms", ms, "bytes_fapply", inf["bytes_fapply"], "bytes_precond", inf["bytes_precond"],
      "bytes_step_fixed", inf["bytes_step_fixed"], "coarse_factor_bytes", inf["coarse_factor_bytes"])
s.close()
