/*
 * tcg_ietidp.h — C ABI of the B200-native tree-cotree IETI-DP time stepper.
 *
 * Method: Mally, Vazquez, Schoeps, "Tree-Cotree-Based IETI-DP for Eddy Current
 * Problems in Time-Domain", arXiv 2510.23446 (cited P:Lnnn = line of PAPER.md).
 *   PDE            curl(nu curl A) + sigma dA/dt = J, A x n = 0 on dOmega    (eq. formA*)
 *   discretisation spline edge elements (degrees (p-1,p,p) cyclic) per box patch,
 *                  conforming interfaces, Boolean multiplier coupling
 *   time stepping  implicit Euler [W dtB^T; dtB 0][a;m] = [f;0]             (eq. euler)
 *   solver         tree-cotree gauge + IETI-DP (e/p/r splitting, primal coarse
 *                  problem, PCG on the multipliers, Dirichlet preconditioner)
 * Readings of passages the paper leaves open are listed in DESIGN.md §3 (R1..R18).
 *
 * Conventions
 *   patch id      s = ix + Px*(iy + Py*iz)
 *   local DOFs    per patch: component-major (x, y, z); within a component k slowest,
 *                 then j, then i fastest; component c has (n_c - 1) indices along c and
 *                 n_d = elems_d + p along the other directions d.
 *   glued edges   the glued control grid has N_d = P_d (n_d - 1) + 1 vertices per
 *                 direction; edge (c,i,j,k) joins vertex (i,j,k) to its +1 neighbour
 *                 along c; ids are component-major with i fastest (R3).
 *   precision     IEEE FP64 throughout (R14).
 *
 * Ownership: the caller owns every input array (copied during the call) and every
 * output buffer (written during the call; a too-short `len` returns TCG_EINVAL and
 * the required length in tcg_last_error). The library owns all device memory,
 * streams and, for world > 1, its NCCL communicator.
 *
 * State machine: create -> set_* (any order, all required except source/solver)
 *                -> [plan] -> setup -> step* -> get_* -> destroy.
 *   set_* after plan/setup -> TCG_ESTATE.  After TCG_ENOTSPD only get_* / destroy.
 * Errors: every call returns a tcg_status; tcg_last_error(h) holds a message with
 *   the details (ENOTSPD: patch id or "coarse", pivot index, pivot value;
 *   ENOCONV: step, iterations, relative residual).
 * Threading: one handle per host thread; calls on one handle are not thread-safe.
 */
#ifndef TCG_IETIDP_H
#define TCG_IETIDP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tcg_ctx* tcg_handle;

typedef enum {
  TCG_OK = 0,
  TCG_EINVAL = -1,   /* invalid argument (p<1, counts<1, nu<=0, sigma<0, short buffer ...) */
  TCG_ESTATE = -2,   /* call not allowed in the current state                               */
  TCG_ENOTSPD = -3,  /* a Cholesky pivot <= 0 (gauging bug)                    */
  TCG_ENOCONV = -4,  /* PCG hit max_iter                                           */
  TCG_ECUDA = -5,    /* CUDA runtime error, or no usable sm_100 device                      */
  TCG_ENCCL = -6,    /* NCCL error                                                          */
  TCG_ENOMEM = -7    /* device allocation failed                                            */
} tcg_status;

/* source kinds: J = phi_s(t) S(x) */
#define TCG_SOURCE_NONE 0
#define TCG_SOURCE_CURL_PSI 1 /* S = curl(0,0,sin(pi x)sin(pi y)sin(pi z)), phi = sin(2 pi t)  (BASELINE.json configs) */
#define TCG_SOURCE_MMS 2      /* S = (sin pi y sin pi z, sin pi x sin pi z, sin pi x sin pi y),
                                 phi_s = 2 pi^2 nu_s (1-e^-t) + sigma_s e^-t  (manufactured, R16) */
#define TCG_SOURCE_PAPER 3    /* the paper's experiment: A = e^-t (sin x cos y cos z, -2 cos x sin y cos z,
                                 cos x cos y sin z), J = e^-t (3 nu_s - sigma_s) S; inhomogeneous Dirichlet data
                                 a_D(t) = e^-t (Pi_h S)_D and A(0) = Pi_h S by the commuting spline projection
                                 (R21); requires elements + p <= 72 per patch and direction */

/* preconditioner scaling (P:L170 uses none; BASELINE.json north_star says "scaled") */
#define TCG_SCALING_NONE 0
#define TCG_SCALING_RHO 1     /* rho_s = diagonal of W^_s at the interface DOF (R5) */

/* plan arrays for tcg_get_plan (host-side tree-cotree results, integer) */
#define TCG_PLAN_EDGE_CLASS 0  /* per glued edge: 0 D, 1 WB, 2 F, 3 I                          */
#define TCG_PLAN_EDGE_REGION 1 /* per glued edge: bit0 = has a conductor owner, bit1 = has an insulator owner */
#define TCG_PLAN_TREE 2        /* per glued edge: 1 if in the spanning tree                     */
#define TCG_PLAN_PART 3        /* per glued edge: 0 GAUGE(e), 1 primal, 2 remaining, 3 Dirichlet(e) */
#define TCG_PLAN_PATCH_COUNTS 4 /* per patch: n_i, n_b, n_p (3 values each)                     */
#define TCG_PLAN_LAMBDA 5      /* per multiplier k: glued edge id, patch(+1), patch(-1)          */
#define TCG_PLAN_PRIMAL 6      /* per primal group: glued edge id                               */
#define TCG_PLAN_RANK_OF_PATCH 7 /* per patch: owning rank (x-slab sharding)                     */

typedef struct tcg_info {
  int64_t n_patches, n_local, n_edges, n_verts;
  int64_t m;            /* number of multipliers (lambda)                                */
  int64_t n_c;          /* number of primal groups (coarse size)                         */
  int64_t n_gauge, n_dirichlet, n_primal_local_total;
  int64_t nr_min, nr_max, nb_min, nb_max, np_min, np_max;
  int64_t steps_done, total_iters;
  int64_t device_bytes; /* bytes of device memory held by the handle                      */
  int64_t kernel_launches; /* kernels launched by this handle so far (cumulative)         */
  double bytes_fapply;  /* algorithmic HBM bytes of one F-apply (all patches + coarse)    */
  double bytes_precond; /* algorithmic HBM bytes of one preconditioner apply             */
  double bytes_step_fixed; /* algorithmic HBM bytes of one step outside the PCG iterations
                              (conductor forward/backward solves, p0 / dual rhs / recovery, z0) */
  double flops_factor;  /* local + coarse factorisation and inverse-factor flops (unpadded) */
  double ms_plan, ms_assembly, ms_factor, ms_coarse, ms_steps; /* device-event timings     */
  double ms_pcg_last_step;
  double prof_ms;       /* summed device time of the profiled kernel's working launches (tcg_set_profile) */
  int64_t prof_launches; /* number of those launches                                      */
  double prof_bytes_per_launch; /* algorithmic HBM bytes of one launch of the profiled kernel */
  int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by this handle (cumulative)  */
  int32_t rank, world;
  int32_t pad_;
  int32_t coarse_sparse;  /* 1: nested-dissection multifrontal coarse, 0: dense S_pp^-1 */
  int64_t coarse_nodes;   /* separator-tree nodes of the sparse coarse (0 if dense)          */
  int64_t coarse_levels;  /* tree height + 1: forward + backward phases per coarse solve     */
  double coarse_factor_bytes; /* bytes of the coarse inverse factors read per coarse solve   */
  int64_t n_nonlinear;    /* patches with a nonlinear reluctivity (tcg_set_nonlinear)          */
  int64_t newton_iters;   /* Newton iterations over all steps done (= linear solves)           */
  int64_t linear_solves;  /* IETI-DP linear solves done (one per step without nonlinear patches) */
  int64_t hist_len;       /* entries of the concatenated relres history (tcg_get_history)      */
  double ms_newton_numeric; /* device time of the Newton re-assemblies and factorisations      */
} tcg_info;

/* Create a handle (the solver object of BASELINE.json north_star "build patches, materials
 * and source; setup and factorise; step(n); read coefficients A and residual history";
 * SURVEY §8(b)). device: CUDA ordinal used by setup; rank/world: this process's place
 * in the job (world=1 for one GPU, world <= 8); nccl_id: 128-byte ncclUniqueId when world > 1
 * (NULL iff world == 1), used only to bootstrap (CUDA IPC handles of every rank's buffers are
 * all-gathered; the solve itself reads/writes peer memory over NVLink inside one persistent
 * kernel per tcg_step); cuda_stream: cudaStream_t to use, or NULL for an owned stream.
 * No CUDA call is made before tcg_setup. setup/refactor/step/get_coefficients are collective. */
tcg_status tcg_create(tcg_handle* out, int device, int rank, int world,
                      const unsigned char* nccl_id, void* cuda_stream);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 of a multi-GPU job calls this and
 * broadcasts the bytes to the other ranks, e.g. through torch.distributed). */
tcg_status tcg_nccl_unique_id(unsigned char* out);

/* Testing/emulation: shard the solve over `vranks` virtual ranks that all live on this
 * process's GPU (separate allocations, one cooperative grid, the same peer-table dataflow and
 * two-level barrier as a multi-GPU job). Requires world == 1; call before tcg_plan. */
tcg_status tcg_set_virtual_ranks(tcg_handle h, int vranks);

/* Multipatch domain (P:L56-60 Omega = union of patches Omega^(i), each the image of the unit
 * cube; P:L74-77 spline edge spaces of degrees (p-1,p,p) cyclic on each patch): a uniform box
 * grid of npatch[0] x npatch[1] x npatch[2] axis-aligned patches on [lo,hi] (identity
 * geometry maps), spline degree p >= 1, elems[d] >= 1 elements per patch per direction
 * (S:L124-152). Errors: TCG_EINVAL (null, p < 1, counts < 1, lo >= hi), TCG_ESTATE (after
 * plan/setup). Arrays are read during the call only. */
tcg_status tcg_set_patches(tcg_handle h, const int npatch[3], const double lo[3], const double hi[3],
                           int degree_p, const int elems[3]);

/* Materials (Omega = Omega_C u Omega_I with sigma > 0 in the conductor and sigma = 0
 * in the insulator; nu > 0 bounded, piecewise constant; here constant per patch):
 * sigma[n] >= 0, nu[n] > 0, finite, n = #patches in patch-id order (copied during the call).
 * Errors: TCG_EINVAL (length, range), TCG_ESTATE (before set_patches, after plan/setup). */
tcg_status tcg_set_materials(tcg_handle h, const double* sigma, const double* nu, size_t n);

/* Source current density J of the eddy-current problem (P:L42 right-hand side of eq.
 * formA*; its Galerkin load j_i = <J_i, w_j>): J(x,t) = amp * phi_s(t) * S(x) with
 * kind (TCG_SOURCE_*) and params[nparams] (NULL/0 = defaults, copied during the call):
 *   TCG_SOURCE_CURL_PSI  params {amp = 1, freq = 1}: phi = sin(2 pi freq t)
 *   TCG_SOURCE_MMS       params {amp = 1}
 *   TCG_SOURCE_PAPER     params {amp = 1}: A = amp e^-t S (boundary data and A(0) scale with amp)
 *   TCG_SOURCE_NONE      no params (J = 0)
 * Default: TCG_SOURCE_CURL_PSI with amp = freq = 1 (the BASELINE.json configs).
 * Errors: TCG_EINVAL (unknown kind, too many params, non-finite), TCG_ESTATE (after setup). */
tcg_status tcg_set_source(tcg_handle h, int kind, const double* params, size_t nparams);

/* Time grid of the implicit Euler method (eq. euler: W a^(l+1) = f^(l+1) with
 * W = M + dt K, f^(l+1) = M a^(l) + dt j^(l+1)): interval (0,T], n_steps uniform steps,
 * dt = T/n_steps, A(0) = 0. Errors: TCG_EINVAL (T <= 0, n_steps < 1), TCG_ESTATE (after setup). */
tcg_status tcg_set_time(tcg_handle h, double T, int n_steps);

/* Solver parameters: PCG on the multipliers with the Dirichlet preconditioner (P:L170,
 * "PCG tolerance" P:L544); stopping rule sqrt(r^T z) <= rtol sqrt(r0^T z0) (R6),
 * max_iter (a step that reaches it fails the call with TCG_ENOCONV); scaling TCG_SCALING_*
 * (P:L170 none, R5 rho); tree_order of the tree-cotree gauge (0: ascending
 * edge ids within a Kruskal rank, 1: descending, the gauge-invariance test; R2).
 * Defaults 1e-10, 5000, RHO, 0. Errors: TCG_EINVAL (rtol <= 0, max_iter < 1, unknown
 * scaling/order), TCG_ESTATE (after plan/setup). */
tcg_status tcg_set_solver(tcg_handle h, double rtol, int max_iter, int scaling, int tree_order);

/* Collective on world > 1 handles: every rank must make the same calls at the same step (each
 * tcg_step checks the agreement over NCCL and fails with TCG_EINVAL otherwise).
 * Warm start (the paper's outlook P:L550 on cheaper PCG; R20).
 * k = 0 (default): the paper's lambda0 = 0. k in 1..4: from step 1 on the PCG starts from the
 * Galerkin projection of the step's solution on the span of the previous k solutions W_j:
 * lambda0 = sum_j c_j W_j, G c = W^T d, G_ij = (W_i^T FW_j + W_j^T FW_i)/2 with FW_j = d_j - r_j
 * (each step's right-hand side minus its final PCG residual, i.e. F W_j to the tolerance: no
 * extra F-apply), solved by Cholesky in step order skipping columns with pivot <= 1e-12
 * max G_ii; r0 = d - sum_j c_j FW_j, then one preconditioner apply (not counted as an
 * iteration). The stopping reference stays sqrt(d^T M^-1 d) (the cold r0^T z0), so warm and
 * cold runs stop at one absolute residual; a step whose start already meets it takes 0
 * iterations; d = 0 gives lambda = 0. tcg_refactor restarts the history (step 0 is cold).
 * Takes effect from the next tcg_step; changing k restarts the history (the next step is
 * cold), as does tcg_refactor. Device memory (2*4+1 = 9 lambda-length vectors per rank,
 * sized for the largest k) is allocated at the first warm step. EINVAL unless 0 <= k <= 4. */
tcg_status tcg_set_warm_start(tcg_handle h, int k);

/* Nonlinear reluctivity (the paper: "nonlinear behavior can be modeled as a
 * simple extension"; law and linearisation are DESIGN.md R25). k[3n] holds per patch the
 * Brauer parameters (k1, k2, k3) of nu(|B|) = k1 exp(k2 |B|^2) + k3 (k1, k2 >= 0, k3 > 0; an all-zero
 * triple keeps the linear patch and its nu_s; n = 0 / k = NULL: no nonlinear patch). Every
 * tcg_step then runs Newton's method per implicit-Euler step from a_0 = a^(l): iterate k
 * re-assembles the nonlinear patches' tangent matrices J = Kt(a_k) + sigma/dt M,
 * Kt_jk = <(nu I + 2 dnu/d|B|^2 B B^T) curl w_k, curl w_j> by (p+1)-point Gauss quadrature,
 * re-factorises (local Cholesky, inverse factors, coarse problem) and solves
 * J a_{k+1} = (Kt - K)(a_k) a_k + sigma/dt M a^(l) + j^(l+1) with the IETI-DP PCG; it stops when
 * ||a_{k+1} - a_k||_2 <= newton_tol ||a_{k+1}||_2 over all patches' local vectors, and fails the
 * call with TCG_ENOCONV after newton_max iterations. Defaults: no nonlinear patch, 1e-8, 20.
 * tcg_get_history then reports per step the PCG iterations summed over its Newton solves, the
 * last solve's final relres, and every solve's relres history (tcg_info.hist_len entries).
 * Requires p <= 7, a source of kind 0-2, no warm start and no error tracking.
 * Errors: TCG_EINVAL (length, parameter range), TCG_ESTATE (before set_patches, after plan/setup). */
tcg_status tcg_set_nonlinear(tcg_handle h, const double* k, size_t n, double newton_tol, int newton_max);

/* Newton statistics after the steps done: newton_iters[nsteps] (Newton iterations per step) and,
 * per linear solve in order, solve_iters[nsolves] (PCG iterations) and increments[nsolves]
 * (||a_{k+1} - a_k|| / ||a_{k+1}||); any pointer may be NULL. Without nonlinear patches nothing is
 * recorded. Errors: TCG_EINVAL (more steps / solves than recorded). */
tcg_status tcg_get_newton(tcg_handle h, int* newton_iters, size_t nsteps, int* solve_iters, double* increments,
                          size_t nsolves);

/* Error norms of the paper's experiment: with on = 1 (source TCG_SOURCE_PAPER,
 * single-process handle, before the first step) every tcg_step runs one step per launch and
 * accumulates on the device, by (p+1)-point Gauss quadrature per element,
 *   e_B(t_l) = ||B(t_l) - curl A_h(t_l)||^2_{L2(Omega)},
 *   e_E(t_l) = ||E_C(t_l) + (A_h(t_l) - A_h(t_{l-1}))/dt||^2_{L2(Omega_C)},
 *   eps_B = sqrt(max_l e_B + dt sum_l e_B),  eps_E = sqrt(dt sum_l e_E)   (reset by tcg_refactor).
 * Errors: TCG_EINVAL (other source, world > 1), TCG_ESTATE (steps already done). */
tcg_status tcg_set_error_tracking(tcg_handle h, int on);

/* eps_B, eps_E after the steps done so far (either pointer may be NULL) and, if per_step !=
 * NULL, the per-step (e_B, e_E) pairs of the first nsteps steps (2*nsteps doubles, caller-owned).
 * Errors: TCG_ESTATE (tracking off), TCG_EINVAL (nsteps > steps done). */
tcg_status tcg_get_errors(tcg_handle h, double* eps_B, double* eps_E, double* per_step, size_t nsteps);

/* Host-only planning (no CUDA): topology, ranked-Kruskal tree, e/p/r partition,
 * multiplier and primal numbering, patch->rank sharding. Idempotent. */
tcg_status tcg_plan(tcg_handle h);

/* Copy a plan array (TCG_PLAN_*) into out[len] (int64). Requires tcg_plan. */
tcg_status tcg_get_plan(tcg_handle h, int what, int64_t* out, size_t len);

/* Collective: plan (if needed), device assembly of W^_s = nu_s K_s + sigma_s/dt M_s
 * (P:L83-87 K_i, M_C, j_i; P:L133 W), batched FP64 Cholesky of the gauged local matrices
 * ("two sequential Schur complements"; the gauge makes them SPD), coarse problem
 * S_pp = sum_s N_s^T S^s N_s (P:L138 N) assembly and factorisation.
 * Errors: TCG_ENOTSPD (a pivot <= 0: patch id or "coarse", pivot index and value in
 * tcg_last_error; a gauging bug; the handle then accepts only get_* / destroy),
 * TCG_ENOMEM, TCG_ECUDA (no sm_100 device, launch failure), TCG_ENCCL, TCG_ESTATE. */
tcg_status tcg_setup(tcg_handle h);

/* Re-run the numeric setup of tcg_setup on the existing
 * allocations and reset the time stepping to t = 0, A = 0 (one "pass over one batch of input"
 * for benchmarking; the plan and device memory are reused). Collective. Errors as tcg_setup. */
tcg_status tcg_refactor(tcg_handle h);

/* Collective: n implicit-Euler steps (P:L133 eq. euler; each step: right-hand side
 * f = M a^(l)/dt + j^(l+1), the 3x3 block system of P:L139-153 reduced to F lam = d and solved by
 * PCG from lam0 = 0, recovery of a = (a_e = 0, a_p = N p, a_r)). One persistent
 * kernel launch per call. Errors: TCG_EINVAL (n < 0, more steps than set_time allows),
 * TCG_ENOCONV (PCG reached max_iter: step, iterations and relres in tcg_last_error; the
 * handle then accepts only get_* / destroy), TCG_ESTATE (before setup / failed handle). */
tcg_status tcg_step(tcg_handle h, int n);

/* Coefficients of A (the spline coefficient vector a of P:L88-121 / P:L133) after the last
 * step, written to the caller's out[len] (len too short: TCG_EINVAL with the needed length).
 * layout 0: per-patch local vectors concatenated
 * (n_patches * n_local; eliminated DOFs 0); layout 1: one value per glued edge taken
 * from the lowest-id owning patch (n_edges). */
tcg_status tcg_get_coefficients(tcg_handle h, int layout, double* out, size_t len);

/* Residual history of the PCG of P:L170 (iteration counts are the paper's scalability
 * indicator): per-step PCG iteration counts iters[nsteps] and final relative residuals
 * final_relres[nsteps] (either may be NULL); if relres_hist != NULL, the concatenated
 * per-step histories sqrt(r_k^T z_k / r_0^T z_0), k = 0..iters (sum(iters+1) values; with
 * nonlinear patches every Newton solve's history, tcg_info.hist_len values in all). */
tcg_status tcg_get_history(tcg_handle h, int* iters, double* final_relres, size_t nsteps,
                           double* relres_hist, size_t hist_len);

/* Counts of the plan (#multipliers m, #primal groups n_c, gauge and Dirichlet
 * DOFs), algorithmic byte and flop counts, timings and profiling results.
 * Valid in any state (zeros before tcg_plan). */
tcg_status tcg_get_info(tcg_handle h, tcg_info* out);

/* The dual operator of the IETI-DP system ("two sequential Schur complements";
 * SURVEY §8(a) c2):  q = F lam = B W~^-1 B^T lam
 *   = B_r W_rr^-1 B_r^T lam + B_r Phi N S_pp^-1 N^T Phi^T B_r^T lam,
 * computed exactly as one PCG iteration computes it (X_bb / Phi_b^T row GEMVs, coarse
 * S_pp^-1 GEMV, X_bb^T / Phi_b column GEMVs, jump) inside the persistent stepper kernel.
 * lam, q: host arrays of m = tcg_info.m doubles in multiplier order (caller-owned; lam is
 * copied in, q written). The lambda operand stays resident for tcg_bench_fapply.
 * Errors: TCG_EINVAL (m mismatch, NULL, multi-process handle), TCG_ESTATE (no setup). */
tcg_status tcg_fapply(tcg_handle h, const double* lam, double* q, size_t m);

/* Benchmark hook: `n` applications of the dual operator F (the exact per-iteration
 * sequence: P1 row GEMVs -> coarse -> column GEMVs -> jump, 4 grid barriers each) in one
 * launch of the persistent kernel, on the operand of the last tcg_fapply (zeros before);
 * returns the device time in *ms. Requires setup; single-process handles. */
tcg_status tcg_bench_fapply(tcg_handle h, int n, double* ms);

/* Time every launch of the persistent stepper kernel (kernel_id 7; 0 = off) with CUDA events
 * on the library stream during subsequent tcg_step calls. Results in tcg_info.prof_*.
 * Resets the accumulators. */
tcg_status tcg_set_profile(tcg_handle h, int kernel_id);

/* Message of the last failed call on h (owned by the handle, valid until the next call). */
const char* tcg_last_error(tcg_handle h);
/* Release every device allocation, stream and communicator of h (NULL is a no-op). */
void tcg_destroy(tcg_handle h);

#ifdef __cplusplus
}
#endif
#endif /* TCG_IETIDP_H */
