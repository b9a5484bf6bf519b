"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of the tree-cotree IETI-DP
time stepper of Mally, Vazquez, Schoeps, "Tree-Cotree-Based IETI-DP for Eddy
Current Problems in Time-Domain" (arXiv 2510.23446; /root/reference/PAPER.md,
cited as P:Lnnn).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import, call or execute anything in this package. The
product path (paper_2510_23446_b200/) never touches it and shares no code with
it: no kernels, helpers, tables or constants.

FP64 (numpy float64) throughout. Library primitives used as steps: numpy
einsum/matmul, scipy.linalg.cho_factor/cho_solve (LAPACK potrf/potrs),
numpy.polynomial.legendre.leggauss.

Modules
  splines    1D open knot vectors, Cox-de Boor B-splines, Curry-Schoenberg D-splines, Gauss rules
  assembly   element-loop Gauss quadrature of K (curl-curl), M (mass), load j
  topology   glued control grid, global edges, owners, classes, regions
  gauge      ranked-Kruskal spanning tree and e/p/r partition
  ietidp     local operators, coarse problem, F, Dirichlet preconditioner, PCG, implicit Euler step
  monolithic glued conforming direct solve of the same gauged system (pin P11)

Pinning status: every function is pinned by a `-m "not gpu"` test
in tests/test_oracle_*.py against closed forms, library routines, brute force,
paper-derived counts or the monolithic solve. No function is "parity unpinned".
"""
