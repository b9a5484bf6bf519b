"""One setup (plan + assembly + factorisation + inverse factors + coarse) of a config; for
ncu launch lists of the setup kernels."""
import os, sys
sys.path.insert(0, os.getcwd())
import workloads, paper_2510_23446_b200 as tcg
for name in sys.argv[1:] or ["cfg3"]:
    s = tcg.Solver().configure(workloads.get(name)); s.setup()
    inf = s.info()
    print(name, "setup ms: assembly %.2f factor %.2f coarse %.2f" % (inf["ms_assembly"], inf["ms_factor"], inf["ms_coarse"]))
    s.close()
