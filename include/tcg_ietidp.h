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
} tcg_info;

/* Create a handle. device: CUDA ordinal used by setup; rank/world: this process's place
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

/* Uniform box grid of npatch[0] x npatch[1] x npatch[2] patches on [lo,hi], spline degree
 * p >= 1 and elems[d] >= 1 elements per patch per direction. */
tcg_status tcg_set_patches(tcg_handle h, const int npatch[3], const double lo[3], const double hi[3],
                           int degree_p, const int elems[3]);

/* Per-patch conductivity sigma >= 0 (0 = insulator) and reluctivity nu > 0, n = #patches
 * (sigma = 0 in Omega_I, nu bounded away from 0). */
tcg_status tcg_set_materials(tcg_handle h, const double* sigma, const double* nu, size_t n);

/* Source kind (TCG_SOURCE_*). Default TCG_SOURCE_CURL_PSI. */
tcg_status tcg_set_source(tcg_handle h, int kind);

/* Time interval (0,T], n_steps implicit-Euler steps, dt = T/n_steps, A(0) = 0. */
tcg_status tcg_set_time(tcg_handle h, double T, int n_steps);

/* PCG stopping rule sqrt(r^T z) <= rtol sqrt(r0^T z0), max_iter (ENOCONV beyond);
 * scaling TCG_SCALING_*; tree_order 0: ascending edge ids within a Kruskal rank,
 * 1: descending (gauge-invariance test). Defaults 1e-10, 5000, RHO, 0. */
tcg_status tcg_set_solver(tcg_handle h, double rtol, int max_iter, int scaling, int tree_order);

/* Warm start (the paper's outlook P:L550 on cheaper PCG; R20).
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
 * cold), as does tcg_refactor. Device memory (2k+1 lambda-length vectors per rank) is
 * allocated at the first warm step. EINVAL unless 0 <= k <= 4. */
tcg_status tcg_set_warm_start(tcg_handle h, int k);

/* Host-only planning (no CUDA): topology, ranked-Kruskal tree, e/p/r partition,
 * multiplier and primal numbering, patch->rank sharding. Idempotent. */
tcg_status tcg_plan(tcg_handle h);

/* Copy a plan array (TCG_PLAN_*) into out[len] (int64). Requires tcg_plan. */
tcg_status tcg_get_plan(tcg_handle h, int what, int64_t* out, size_t len);

/* Collective: plan (if needed), device assembly of W^_s = nu_s K_s + sigma_s/dt M_s,
 * batched FP64 Cholesky, coarse problem assembly and factorisation. */
tcg_status tcg_setup(tcg_handle h);

/* Re-run the numeric setup (assembly, batched Cholesky, coarse factorisation) on the
 * existing allocations and reset the time stepping to t = 0, A = 0 (one "pass over one
 * batch of input" for benchmarking; the plan and device memory are reused). */
tcg_status tcg_refactor(tcg_handle h);

/* Collective: n implicit-Euler steps (each: rhs, PCG on lambda, recovery). */
tcg_status tcg_step(tcg_handle h, int n);

/* Coefficients of A after the last step. layout 0: per-patch local vectors concatenated
 * (n_patches * n_local; eliminated DOFs 0); layout 1: one value per glued edge taken
 * from the lowest-id owning patch (n_edges). */
tcg_status tcg_get_coefficients(tcg_handle h, int layout, double* out, size_t len);

/* Per-step PCG iteration counts iters[nsteps] and final relative residuals
 * final_relres[nsteps] (either may be NULL); if relres_hist != NULL, the concatenated
 * per-step histories sqrt(r_k^T z_k / r_0^T z_0), k = 0..iters (sum(iters+1) values). */
tcg_status tcg_get_history(tcg_handle h, int* iters, double* final_relres, size_t nsteps,
                           double* relres_hist, size_t hist_len);

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

const char* tcg_last_error(tcg_handle h);
void tcg_destroy(tcg_handle h);

#ifdef __cplusplus
}
#endif
#endif /* TCG_IETIDP_H */
