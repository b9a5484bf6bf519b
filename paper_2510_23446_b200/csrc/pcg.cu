// pcg.cu — step c of the hot path: implicit-Euler time stepping (rhs, PCG on lambda,
// recovery) as chain-free GEMV work items inside ONE persistent cooperative kernel that
// runs n time steps (k_steps). No host round trip between steps or PCG iterations.
//
// Paper: implicit Euler (eq. euler), the 3x3 block system after the e/p/r split
// (P:L139-153), "two sequential Schur complements", PCG with the Dirichlet
// preconditioner; recurrences DESIGN.md R6.
// Setup (chol.cu) overwrites each patch's augmented Cholesky factor with its inverse
//   Xaug = [X_rr = L_rr^-1 ; Phi^T = W_pr W_rr^-1]      (trailing b block of X_rr = L_bb^-1)
// and builds S_pp^-1 = X_c^T X_c (full symmetric). Per step (phases separated by grid barriers):
//   R1  f = (sigma/dt) M a + phi(t) j_S  (conductors);  insulators: Z = phi(t) XJ
//   R2  Z_r = X_rr f_r,  Z_p = f_p - Phi^T f_r         (= L^-1 f, f_p - W_pr W_rr^-1 f_r)
//   R3  Pc = S_pp^-1 sum_s N_s^T Z_p                     (p0)
//   R4  y = X_bb^T Z_b - Phi_b N Pc ; d = B y            (dual rhs)
//   R5  u = B_D^T d, S_bb u, rho0 = sum u.S u ; r = d, lambda = 0
//   PCG iterations (4 barriers each):
//   P1  p = z + beta p_prev (z gathered from the last S_bb apply); v = B^T p;
//       w = X_bb v, (-g) = -Phi_b^T v
//   PC  Pc = S_pp^-1 sum N^T (-g)
//   P5  y = X_bb^T w - Phi_b N Pc ; p^T F p = sum_s v_s . y_s
//   P7  alpha; lambda += alpha p; r -= alpha B y; u = B_D^T r, S_bb u; r^T z = sum u.S u
//   E1  v = B^T lambda ; w, -Phi^T v                      (recovery)
//   E2  Pc = S_pp^-1 sum N^T (Z_p + Phi^T v)              (= p)
//   E3  a_r = X_rr^T (Z_r - [0; w_b]) - Phi N Pc ; a_p = N Pc ; a_e = 0
// Partials are summed in one fixed order by every block: deterministic, identical scalars.
//
// Latency design (the small configs are L2-resident and bound by dependent-load chains):
// each block's items are fixed for the whole launch (host LPT dealing, ItemDesc carries the
// patch scalars) and the per-iteration item lists and the block's lambda-chunk index data are
// copied to shared memory once per launch; every GEMV issues its first tile's loads before
// the gather of its input vector, so the two latencies overlap.
#include "common.cuh"
#include "device.h"

namespace tcg {

// Barrier / reduction memory of one rank (in that rank's device memory).
struct BarMem {
  unsigned int local_count;   // arrivals of this rank's blocks (monotone)
  unsigned int local_gen;     // release generation for this rank's blocks
  unsigned int global_count;  // (rank 0 only) arrivals of rank leaders (monotone)
  unsigned int pad;
  double rank_part[2];        // this rank's partial of the current reduction (by round parity)
  double pad2[6];
};

// lambda-chunk index data of one multiplier (shared-memory cache of the block's chunk)
struct LamC {
  int64_t ip, im;  // aug-vector indices of the + and - side
  double wp, wm;   // B_D weights of the two sides
  int pp, pm;      // patches of the two sides
};

// Arguments of the persistent stepper. Every per-rank buffer is a table indexed by rank:
// writes go to the launching block's own rank, reads of values owned elsewhere (interface
// partners, lambda chunks, coarse rows) go to the owner's buffer (peer memory over NVLink on
// a multi-GPU job; another allocation of the same device for virtual ranks).
constexpr int KW = 4;                         // largest warm-start subspace
constexpr int KW_NV = KW + KW * (KW + 1) / 2;  // W_j.d and the upper triangle of G
__host__ __device__ constexpr int kw_idx(int i, int j) { return KW + i * KW - i * (i - 1) / 2 + (j - i); }  // i <= j
struct StepArgs {
  // lambda-space vectors (m, valid on the owner of each chunk)
  double* lam[MAXR];
  double* r[2][MAXR];
  double* pk[2][MAXR];
  // per-patch aug-ordered vectors (global layout, valid on the patch owner)
  double* F[MAXR];     // R1 output (conductor rhs f)
  double* Z[MAXR];     // R2 output (Z_r = L^-1 f_r, Z_p = f_p - h)
  double* XJ[MAXR];    // setup: forward of j_S (insulator rhs template)
  double* JS[MAXR];
  double* XW[MAXR];    // P1/E1 output: b part w, p part -g
  double* Y[MAXR];     // P5/R4 output: b part y, X_bb^T part (y = Y + Y2)
  double* Y2[MAXR];    // P5/R4 output: b part y, -Phi_b N Pc part
  double* PW[MAXR];    // S_bb apply output: b part
  double* a_loc[MAXR]; // local coefficient vectors (npatch x nloc)
  // Newton iterate of a nonlinear step (nonlinear.cu; null otherwise): R1's mass term reads
  // a^l from a_old instead of a_loc, and the right-hand side gains gnl (aug order)
  double* a_old[MAXR];
  double* gnl[MAXR];
  // coarse
  const double* Sinv[MAXR];  // full symmetric S_pp^-1 (replicated), Tc x Tc row-major tiles
  double* Ppart[MAXR];       // Tc x maxch x 64 chunk partials of Pc (rows of the owning rank)
  double* Pc[MAXR];          // materialised coarse solution (standalone kernels)
  const int* crow_owner;     // coarse row block -> rank
  int ch, maxch;
  double* partials[MAXR];    // per block partial sums (own rank)
  BarMem* bar[MAXR];
  // per-step outputs (written by each rank's block 0 into its own buffers)
  double* hist[MAXR];
  int* iters[MAXR];
  PcgState* st[MAXR];
  // work items per phase: block gb = rank * nbr + bl owns items[ph][boff[ph][gb] .. boff[ph][gb+1])
  const ItemDesc* items[NPH];
  const int* boff[NPH];
  const int64_t* pcprog;  // PC gather programs: per item offs[nE+1], then (owner << 56 | aug index)
  int cache_pcprog;  // 1: the block's PC programs are copied to shared memory
  const int* bpl;     // per block: (patch, cache offset) pairs of the patches whose b records it caches
  const int* bploff;  // block gb owns pairs bploff[gb] .. bploff[gb+1]
  int cache_bpos;     // 1: b-position records cached (ItemDesc::bc valid)
  int cache_items;  // 1: the block's per-iteration item lists are copied to shared memory
  int cache_lam;    // 1: the block's lambda-chunk index data are copied to shared memory
  int scratch;      // doubles of item scratch (after the prefetch tiles) in dynamic shared memory (even)
  int npf;          // tiles of the next phase's first item bulk-copied to shared memory during a barrier
  int mode;         // 0: nsteps implicit-Euler steps; 1: nsteps applications q = F p (p = pk[0], q -> r[1])
  int dbg_stop;     // debug: 1 = return after the first step's R3 coarse solve
  int warm;         // k > 0: PCG starts from the Galerkin projection on the previous k solutions (f2)
  int warm_base;        // warm start: history starts at this step (set when k changes; refactor: 0)
  double* Wr[MAXR];     // warm start: ring of the previous k solutions (slot = global step % k), own rank
  double* FWr[MAXR];    // and of d_j - r_j (= F W_j up to the tolerance)
  double* dsave[MAXR];  // this step's d (lambda level)
  double* wpart[MAXR];  // per-block partial dot products (2 x nbr x KW_NV), one rank
  // sparse coarse: per level forward rows / backward columns of the node factors
  int sparse;
  int cf_levels;                 // tree height + 1
  const ItemDesc* cf_fw;         // block gb, level lv: items [cf_fw_off[lv * nbr + gb], .. + 1)
  const int* cf_fw_off;
  const ItemDesc* cf_bw;
  const int* cf_bw_off;
  const double* FR;              // node inverse factors [L_VV^-1 ; L_BV L_VV^-1] (tile-packed)
  const int64_t* cf_prog;        // forward gather sources: cf_kw tagged slots per frontal position
  int cf_kw;
  const int* cf_vl;              // node V groups
  const int* cf_bl;              // node B groups
  // per rank: every rank runs the whole (replicated) coarse solve on its own blocks
  double* CW[MAXR];              // node forward vectors (y_V ; f_B - L_BV y_V)
  double* Pcs[MAXR];             // coarse solution by primal group
  double* cf_pb[MAXR];           // backward chunk partial sums (64 per chunk)
  unsigned int* cf_cnt[MAXR];    // backward chunk arrival counters (monotone)
  const int4* cf_node;           // per node: parent, #fw items, #bw items, #children's fw items
  const int2* cf_bwdep;          // per node: nearest ancestor with bw items and their count, or (-1, #own fw items)
  unsigned int* cf_dflow[MAXR];  // [0, nn): children's fw items done; [nn, 2nn): own fw; [2nn, 3nn): own bw
  int cf_nn;
  int cf_sync;                   // 1: level-synchronous (grid barrier per level) instead of dataflow
  unsigned long long* tstamp;  // optional phase timestamps (rank 0 block 0)
  double* itime;               // optional per-item durations (ns), [phase * itime_stride + item]
  int itime_stride;
  double rtol;
  int max_iter;
  // ranks
  int nranks;     // ranks of the job (real GPUs or virtual ranks)
  int nbr;        // persistent blocks per rank
  int rank_base;  // rank of block 0 of this launch (real multi-GPU: this process's rank)
  int sys_scope;  // 1 when ranks are different GPUs (system-scope fences/atomics)
  int64_t lam_chunk;  // lambda entries per (rank, block): owner of k = (k / lam_chunk) / nbr
  // time stepping
  int source;
  double src_amp, src_freq;  // J = src_amp * phi(t; src_freq) * S(x) (tcg_set_source params)
  // the paper's experiment (source 3, mms.cu): Dirichlet DOFs (s * nloc + a) and their
  // template values; a_D(t) = src_amp e^-t aD0 is written into a_loc after every step
  const int64_t* dlist;
  const double* aD0;
  int64_t nd;
  double dt;
  int step0;    // steps done before this launch
  int nsteps;   // steps to run
  int64_t hist_off;  // offset of this launch's history in hist
  unsigned int round0;  // barrier rounds completed before this launch (counters are monotone)
  Tables1D tb;
  Geom G;
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- bulk async copies (TMA engine, cp.async.bulk) into shared memory, mbarrier-tracked ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(mb)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double2 lds2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

// fixed-order block reduction of one value per thread: xor-butterfly warp sums (lane 0's
// value), then the 8 warp sums in warp order. Every thread returns the same value.
__device__ __forceinline__ double block_sum(double local, double* red) {
  const double w = warp_sum(local);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int i = 0; i < NTHR / 32; ++i) r += red[i];
  __syncthreads();
  return r;
}

// Coarse solution entry g from the PC chunk partials (fixed chunk order), read on the rank
// that owns coarse row block g/64. Loads are issued 4 at a time, summed in chunk order.
template <bool MULTI>
__device__ __forceinline__ double pc_get(const StepArgs& A, int64_t g) {
  const int I = (int)(g >> 6);
  const double* p = A.Ppart[MULTI ? A.crow_owner[I] : 0] + ((int64_t)I * A.maxch) * TS + (g & 63);
  double v = 0.0;
  int c = 0;
  for (; c + 4 <= A.maxch; c += 4) {
    const double a0 = ldcg(p + (int64_t)c * TS), a1 = ldcg(p + (int64_t)(c + 1) * TS),
                 a2 = ldcg(p + (int64_t)(c + 2) * TS), a3 = ldcg(p + (int64_t)(c + 3) * TS);
    v += a0;
    v += a1;
    v += a2;
    v += a3;
  }
  for (; c < A.maxch; ++c) v += ldcg(p + (int64_t)c * TS);
  return v;
}

// ---- tile GEMVs with the input gather overlapped ------------------------------------------
// Warp w owns rows 8w..8w+7 of every 64x64 tile, lane l columns 2l, 2l+1. The first two
// tiles are prefetched into L1 (non-binding, no registers held), then gather() fills the
// input vector in shared memory, then the tiles are streamed (2 tiles of loads in flight).
// experiment switches (TCG_STEP_FLAGS): bit 0 = no L1 prefetch of the first tiles; bits 4+ph =
// no bulk-copy prefetch for phase ph
__constant__ int c_step_flags;
__device__ __forceinline__ void prefetch_l1(const double* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
template <class TileF>
__device__ __forceinline__ void prefetch_tiles(TileF tile, int J0, int J1) {
  const int off = (threadIdx.x >> 5) * 8 * TS + 2 * (threadIdx.x & 31);
  for (int J = J0; J < min(J1, J0 + 2); ++J) {
    const double* t = tile(J) + off;
#pragma unroll
    for (int r = 0; r < 8; ++r) prefetch_l1(t + r * TS);
  }
}
// row:  part[r] += sum_{J=J0}^{J1-1} tile(J)[row0+r][:] . x[(J-J0)*64 : ]
// The first npf tiles were copied to shared memory (pft) by a bulk copy issued during the
// preceding grid barrier; the rest stream from global memory.
template <class TileF, class Gather>
__device__ __forceinline__ void gemv_row_g(TileF tile, int J0, int J1, const double* x, Gather gather,
                                           double (&part)[8], const double* pft = nullptr, int npf = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const int off = row0 * TS + 2 * lane;
  if (!(c_step_flags & 1)) prefetch_tiles(tile, J0 + npf, J1);
  gather();
  __syncthreads();
  for (int J = J0; J < min(J1, J0 + npf); ++J) {
    const double* t = pft + (J - J0) * TSZ + off;
    const double2 xv = *reinterpret_cast<const double2*>(x + (J - J0) * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = lds2(t + r * TS);

#pragma unroll
    for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
  }
#pragma unroll 2
  for (int J = J0 + npf; J < J1; ++J) {
    const double* t = tile(J) + off;
    const double2 xv = *reinterpret_cast<const double2*>(x + (J - J0) * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
  }
}
// col:  c[0..1] += sum_{I=I0}^{I1-1} tile(I)[row0+r][2*lane..] * x[(I-I0)*64 + row0 + r]
template <class TileF, class Gather>
__device__ __forceinline__ void gemv_col_g(TileF tile, int I0, int I1, const double* x, Gather gather, double& c0,
                                           double& c1, const double* pft = nullptr, int npf = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const int off = row0 * TS + 2 * lane;
  if (!(c_step_flags & 1)) prefetch_tiles(tile, I0 + npf, I1);
  gather();
  __syncthreads();
  for (int I = I0; I < min(I1, I0 + npf); ++I) {
    const double* t = pft + (I - I0) * TSZ + off;
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = lds2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double xr = x[(I - I0) * TS + row0 + r];
      c0 += a[r].x * xr;
      c1 += a[r].y * xr;
    }
  }
#pragma unroll 2
  for (int I = I0 + npf; I < I1; ++I) {
    const double* t = tile(I) + off;
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double xr = x[(I - I0) * TS + row0 + r];
      c0 += a[r].x * xr;
      c1 += a[r].y * xr;
    }
  }
}
// finish a column GEMV: cross-warp sum into out64[0..63] (threads < 64 hold valid results)
__device__ __forceinline__ double col_finish(double c0, double c1, double* cr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  cr[warp * TS + 2 * lane] = c0;
  cr[warp * TS + 2 * lane + 1] = c1;
  __syncthreads();
  double acc = 0.0;
  if (threadIdx.x < TS) {
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) acc += cr[w * TS + threadIdx.x];
  }
  return acc;
}

// ---- P1 / E1: [X_bb; Phi_b^T] v, v = B_s^T p gathered per b position ---------------------
// vsrc(it, b, pos) returns (B_s^T p)_pos, b = b_off + pos. Output XW: +w (b rows), -g (p rows).
// Xr = the rank's inverse-factor store.
// gat = false: sv still holds this patch's v from the previous item of the same patch
template <class Src>
__device__ __forceinline__ void p1_item(const ItemDesc& it, const double* Xr, Src vsrc, double* XW, double* sv,
                                        const double* pft = nullptr, int npf = 0, int gat = 1) {
  const int I = it.I, Ti = it.Ti, Tb = it.Tb, nb = it.nb;
  const int Jn = (I < Tb) ? I + 1 : Tb;
  const double* X = Xr + it.a_off;
  double part[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) part[r] = 0.0;
  gemv_row_g([&](int J) { return X + tri_off(Ti + I, J); }, Ti, Ti + Jn, sv,
             [&] {
               if (gat) {
                 const int ne = (gat == 2) ? Tb * TS : Jn * TS;  // the full vector only if reused
                 for (int e = threadIdx.x; e < ne; e += blockDim.x) sv[e] = (e < nb) ? vsrc(it, it.b_off + e, e) : 0.0;
               }
             },
             part, pft, npf);
  const double sum = warp_reduce8(part);
  const int lane = threadIdx.x & 31, row0 = (threadIdx.x >> 5) * 8;
  if ((lane & 3) == 0) XW[it.vec_off + (int64_t)(Ti + I) * TS + row0 + warp_reduce8_row()] = (I < Tb) ? sum : -sum;
  __syncthreads();
}

// ---- PC: Ppart[I][c] = sum_{J in chunk c} Sinv_IJ G_J,  G_g = sum_{csr e of g} gsrc(e) -----------
// prog: this item's gather program: offs[0..nE] (relative to the entry list), then one
// entry (owner rank << 56 | aug-vector index) per csr element of the chunk's groups.
constexpr int64_t kIdxMask = (1ll << 56) - 1;
template <class GS>
__device__ __forceinline__ void pc_item(const DevPlan& D, const StepArgs& A, const double* Sinv, int I, int c,
                                        const int64_t* prog, GS gsrc, double* Ppart, double* sm,
                                        const double* pft = nullptr, int npf = 0) {
  const int Tc = D.Tc;
  const int J0 = c * A.ch, J1 = min(Tc, J0 + A.ch);
  const int nE = (J1 - J0) * TS;
  const int64_t* ent = prog + nE + 1;
  const int lane = threadIdx.x & 31, row0 = (threadIdx.x >> 5) * 8;
  const double* rowp = Sinv + ((int64_t)I * Tc) * TSZ;
  double part[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) part[r] = 0.0;
  gemv_row_g([&](int J) { return rowp + (int64_t)J * TSZ; }, J0, J1, sm,
             [&] {
               for (int e = threadIdx.x; e < nE; e += blockDim.x) {
                 const int q0 = (int)prog[e], q1 = (int)prog[e + 1];
                 double val = 0.0;
                 for (int q = q0; q < q1; ++q) {
                   const int64_t v = ent[q];
                   val += gsrc(v & kIdxMask, (int)(v >> 56));
                 }
                 sm[e] = val;
               }
             },
             part, pft, npf);
  const double sum = warp_reduce8(part);
  if ((lane & 3) == 0) Ppart[((int64_t)I * A.maxch + c) * TS + row0 + warp_reduce8_row()] = sum;
  __syncthreads();
}

#define SUBSTAMP(k) \
  if (sub) { __syncthreads(); if (threadIdx.x == 0) sub[k] = gtimer(); }
// ---- P5 / R4: y_J = sum_{I>=J} X_bb,IJ^T w_I - sum_{p rows} PhiT_IJ^T (N Pc)_I -------------
// Split in two items so no single item streams more than max(Tb, Tp) tiles: part 0 the X_bb^T
// tiles (-> Y), part 1 the Phi_b tiles (-> Y2); consumers read y = Y + Y2. Returns this item's
// share of v_J . y_J (vsrc gives (B_s^T p)_pos; pass zero for R4).
template <class PcF, class Src>
__device__ __forceinline__ double p5_item(const ItemDesc& it, const double* Xr, const double* W, const int* p_grp,
                                          PcF pc, Src vsrc, double* Y, double* Y2, double* sm, double* red,
                                          unsigned long long* sub = nullptr, const double* pft = nullptr,
                                          int npf = 0, int gat = 1) {
  const int J = it.I, Ti = it.Ti, Tb = it.Tb, np = it.np, nb = it.nb;
  const bool ppart = (it.part & 1) != 0;
  const bool merged = (it.part & 2) != 0;  // whole column J: X_bb^T tiles then Phi_b tiles (-> Y)
  const int I0 = ppart ? Tb : J, I1 = (ppart || merged) ? Tb + it.Tp : Tb;
  // the whole b (part 0) or p (part 1) input of the patch, reused by the next item of the
  // same patch and part (gat = false)
  const int G0 = ppart ? Tb : 0;
  double* sfull = sm;                   // (I1 - G0) * 64
  double* sw = sm + (I0 - G0) * TS;     // rows I0.. of the input
  double* cr = sm + (I1 - G0) * TS;     // 8 * 64
  const int* grp = p_grp + it.p_off;
  const int64_t vo = it.vec_off + (int64_t)Ti * TS;
  const double* X = Xr + it.a_off;
  // v_J entry of this thread (threads < 64), fetched early so its latency overlaps the gather
  double vj = 0.0;
  if (threadIdx.x < TS && J * TS + (int)threadIdx.x < nb)
    vj = vsrc(it, it.b_off + J * TS + threadIdx.x, J * TS + threadIdx.x);
  double c0 = 0.0, c1 = 0.0;
  gemv_col_g([&](int I) { return X + tri_off(Ti + I, Ti + J); }, I0, I1, sw,
             [&] {
               if (gat)
                 for (int e = (gat == 2 ? 0 : (I0 - G0) * TS) + threadIdx.x; e < (I1 - G0) * TS; e += blockDim.x) {
                   double val;
                   if (merged) val = (e < Tb * TS) ? ldcg(W + vo + e) : ((e - Tb * TS < np) ? -pc(grp[e - Tb * TS]) : 0.0);
                   else if (!ppart) val = ldcg(W + vo + e);
                   else val = (e < np) ? -pc(grp[e]) : 0.0;
                   sfull[e] = val;
                 }
             },
             c0, c1, pft, npf);
  SUBSTAMP(1);
  const double acc = col_finish(c0, c1, cr);
  double contrib = 0.0;
  if (threadIdx.x < TS) {
    (ppart ? Y2 : Y)[vo + (int64_t)J * TS + threadIdx.x] = acc;
    contrib = vj * acc;
  }
  SUBSTAMP(2);
  return contrib;  // this thread's share of v_J . y_J; the caller block-sums once per phase
}

// ---- P7 / R5, whole-patch dealing (ItemDesc part 2): the S_bb apply of one patch with every
// stored tile read once. Tile (I,J), I > J, gives its row contribution S_IJ u_J to y_I and its
// column contribution S_IJ^T u_I to y_J from the same registers; column blocks J run outer and
// row blocks I >= J inner, so y_J is complete when column block J ends (its row contributions
// come from tiles (J, J' <= J)). Warp w owns rows 8w..8w+7 of each tile (row sums by
// warp_reduce8 into y, exclusive per warp), lane l columns 2l, 2l+1 (column sums in registers
// over the column block, then over the 8 warps in warp order): deterministic. One
// __syncthreads per column block (double-buffered warp partials).
template <class Src>
__device__ __forceinline__ double symv_patch(const ItemDesc& it, const double* Sr, double* PW, Src usrc, double* sm,
                             const double* pft, int npf, const double* Xr = nullptr, double* XW = nullptr) {
  const int Ti = it.Ti, Tb = it.Tb, nb = it.nb;
  double* u = sm;             // Tb*64 input
  double* y = u + Tb * TS;    // Tb*64 row contributions
  double* cw = y + Tb * TS;   // 2 x 8 warps x 64 column partials
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const int off = row0 * TS + 2 * lane;
  const double* S = Sr + it.sbb_off;
  if (!(c_step_flags & 1)) prefetch_tiles([&](int I) { return S + tri_off(I, 0); }, npf > 0 ? 1 : 0, Tb);
  for (int i = threadIdx.x; i < Tb * TS; i += blockDim.x) {
    u[i] = (i < nb) ? usrc(it, it.b_off + i, i) : 0.0;
    y[i] = 0.0;
  }
  __syncthreads();
  double contrib = 0.0;
  for (int J = 0; J < Tb; ++J) {
    const double2 uJ = *reinterpret_cast<const double2*>(u + J * TS + 2 * lane);
    double c0 = 0.0, c1 = 0.0;
#pragma unroll 2
    for (int I = J; I < Tb; ++I) {
      double2 a[8];
      // diagonal tiles: only the lower triangle is used (row part c <= r, column part c < r);
      // rows / columns at or beyond nb (padding) are not loaded: the product is the same and
      // the DRAM sectors of the skipped entries are never fetched
      const bool edge = (I == J) || ((I == Tb - 1) && (nb & (TS - 1)));
      if (I == 0 && npf > 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = lds2(pft + off + r * TS);
      } else if (!edge) {
        const double* t = S + tri_off(I, J) + off;
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
      } else {
        const double* t = S + tri_off(I, J) + off;
        const int rlim = nb - I * TS - row0, cl = 2 * lane;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const bool ok = r < rlim && J * TS + cl < nb && (I != J || cl <= row0 + r);
          a[r] = ok ? ldg2(t + r * TS) : make_double2(0.0, 0.0);
        }
      }
      if (I == J) {  // mask the strict upper triangle (the .y of a pair straddling the diagonal)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (2 * lane > row0 + r) a[r].x = 0.0;
          if (2 * lane + 1 > row0 + r) a[r].y = 0.0;
        }
      }
      double part[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) part[r] = a[r].x * uJ.x + a[r].y * uJ.y;
      {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const double xr = u[I * TS + row0 + r];
          // column part of the strict lower triangle: diagonal entries only in the row part
          const double ax = (I == J && 2 * lane == row0 + r) ? 0.0 : a[r].x;
          const double ay = (I == J && 2 * lane + 1 == row0 + r) ? 0.0 : a[r].y;
          c0 += ax * xr;
          c1 += ay * xr;
        }
      }
      const double rs = warp_reduce8(part);
      if ((lane & 3) == 0) y[I * TS + row0 + warp_reduce8_row()] += rs;
    }
    double* cb = cw + (J & 1) * 8 * TS;
    cb[warp * TS + 2 * lane] = c0;
    cb[warp * TS + 2 * lane + 1] = c1;
    __syncthreads();
    if (threadIdx.x < TS) {
      double v = y[J * TS + threadIdx.x];
#pragma unroll
      for (int w = 0; w < NTHR / 32; ++w) v += cb[w * TS + threadIdx.x];
      PW[it.vec_off + (int64_t)(Ti + J) * TS + threadIdx.x] = v;
      contrib += u[J * TS + threadIdx.x] * v;
    }
  }
  if (it.part & 4) {
    // the F-apply's Phi_b^T rows on the same input (P1 with sbbinv): -g_I = -sum_J PhiT_IJ v_J,
    // rows Tb..Tb+Tp-1 of the inverse-factor store, into XW (as p1_item's p rows)
    const double* X = Xr + it.a_off;
    for (int I = Tb; I < Tb + it.Tp; ++I) {
      double part[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) part[r] = 0.0;
      const int rlim = it.np - (I - Tb) * TS - row0;  // primal rows of this block (padding skipped)
#pragma unroll 2
      for (int J = 0; J < Tb; ++J) {
        const double* t = X + tri_off(Ti + I, Ti + J) + off;
        const double2 xv = *reinterpret_cast<const double2*>(u + J * TS + 2 * lane);
        const bool cok = J * TS + 2 * lane < nb;
        double2 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = (r < rlim && cok) ? ldg2(t + r * TS) : make_double2(0.0, 0.0);
#pragma unroll
        for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
      }
      const double sum = warp_reduce8(part);
      if ((lane & 3) == 0) XW[it.vec_off + (int64_t)(Ti + I) * TS + row0 + warp_reduce8_row()] = -sum;
    }
  }
  __syncthreads();  // the next item overwrites u / y
  return contrib;
}

// ---- P5 with sbbinv, whole-patch dealing (ItemDesc part 3): y2_J = -sum_I PhiT_IJ^T (N Pc)_I
// for every column block J of the patch, N Pc gathered once. Warp w owns column blocks
// J = w, w + 8, ...; lane l columns 2l, 2l+1 of them, streaming the Tp tiles of the column
// row by row (coalesced 512-byte rows) with the sums in registers: no cross-warp reduction and
// no block barrier per column (fixed row order: deterministic). Returns this thread's share of
// v . y2 (vsrc gives v = (B_s^T p)_pos).
template <class PcF, class Src>
__device__ __forceinline__ double p5_phi_patch(const ItemDesc& it, const double* Xr, const int* p_grp, PcF pc, Src vsrc, double* Y2,
                               double* sm) {
  const int Ti = it.Ti, Tb = it.Tb, Tp = it.Tp, np = it.np, nb = it.nb;
  double* g = sm;  // Tp*64: -(N Pc) on the patch's primal rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* grp = p_grp + it.p_off;
  const double* X = Xr + it.a_off;
  const int64_t vo = it.vec_off + (int64_t)Ti * TS;
  for (int e = threadIdx.x; e < Tp * TS; e += blockDim.x) g[e] = (e < np) ? -pc(grp[e]) : 0.0;
  __syncthreads();
  double contrib = 0.0;
  // column blocks J and J + 8 of a warp are streamed together (twice the loads in flight; with
  // Tb <= 16 every warp has at most these two)
  for (int J0 = warp; J0 < Tb; J0 += 2 * (NTHR / 32)) {
    const int J1 = J0 + NTHR / 32;
    const bool two = J1 < Tb;
    const int ca = J0 * TS + 2 * lane, cb = J1 * TS + 2 * lane;
    const bool oka = ca < nb, okb = two && cb < nb;  // padded columns and rows are not loaded
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int I = 0; I < Tp; ++I) {
      const double* ta = X + tri_off(Ti + Tb + I, Ti + J0) + 2 * lane;
      const double* tb = two ? X + tri_off(Ti + Tb + I, Ti + J1) + 2 * lane : ta;
      const double* gi = g + I * TS;
      const int rn = min(TS, np - I * TS);
#pragma unroll 8
      for (int r = 0; r < rn; ++r) {
        const double2 x = oka ? ldg2(ta + r * TS) : make_double2(0.0, 0.0);
        const double2 z = okb ? ldg2(tb + r * TS) : make_double2(0.0, 0.0);
        const double gr = gi[r];
        a0 += x.x * gr;
        a1 += x.y * gr;
        b0 += z.x * gr;
        b1 += z.y * gr;
      }
    }
    *reinterpret_cast<double2*>(Y2 + vo + ca) = make_double2(a0, a1);
    double va0 = 0.0, va1 = 0.0;
    if (ca < nb) va0 = vsrc(it, it.b_off + ca, ca);
    if (ca + 1 < nb) va1 = vsrc(it, it.b_off + ca + 1, ca + 1);
    contrib += va0 * a0 + va1 * a1;
    if (two) {
      *reinterpret_cast<double2*>(Y2 + vo + cb) = make_double2(b0, b1);
      double vb0 = 0.0, vb1 = 0.0;
      if (cb < nb) vb0 = vsrc(it, it.b_off + cb, cb);
      if (cb + 1 < nb) vb1 = vsrc(it, it.b_off + cb + 1, cb + 1);
      contrib += vb0 * b0 + vb1 * b1;
    }
  }
  __syncthreads();  // the next item overwrites g
  return contrib;
}

// ---- P7 / R5: symmetric S_bb apply, one row block I of one patch --------------------------
// usrc(it, b, pos) returns (B_D^(s)T r)_pos. Returns this item's share of u^T S_bb u.
template <class Src>
__device__ __forceinline__ double symv_item(const ItemDesc& it, const double* Sr, double* PW, Src usrc, double* sm,
                                            double* red, const double* pft = nullptr, int npf = 0, bool gat = true) {
  if (it.part & 2) return symv_patch(it, Sr, PW, usrc, sm, pft, npf);
  const int I = it.I, Ti = it.Ti, Tb = it.Tb, nb = it.nb;
  double* u = sm;            // Tb*64
  double* cr = u + Tb * TS;  // 9 * 64
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const double* S = Sr + it.sbb_off;
  double part[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) part[q] = 0.0;
  // row part: S_IJ u_J (J <= I), the u gather overlapped with the first tile's loads
  gemv_row_g([&](int J) { return S + tri_off(I, J); }, 0, I + 1, u,
             [&] {
               if (gat)
                 for (int i = threadIdx.x; i < Tb * TS; i += blockDim.x) u[i] = (i < nb) ? usrc(it, it.b_off + i, i) : 0.0;
             },
             part, pft, npf);
  double c0 = 0.0, c1 = 0.0;
#pragma unroll 2
  for (int J = I + 1; J < Tb; ++J) {  // column part: S_JI^T u_J
    const double* t = S + tri_off(J, I) + row0 * TS + 2 * lane;
    double2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = ldg2(t + q * TS);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double xr = u[J * TS + row0 + q];
      c0 += a[q].x * xr;
      c1 += a[q].y * xr;
    }
  }
  cr[warp * TS + 2 * lane] = c0;
  cr[warp * TS + 2 * lane + 1] = c1;
  const double rs = warp_reduce8(part);
  __syncthreads();
  if ((lane & 3) == 0) {
    const int row = row0 + warp_reduce8_row();
    double acc = rs;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) acc += cr[w * TS + row];
    cr[8 * TS + row] = acc;
  }
  __syncthreads();
  double contrib = 0.0;
  if (threadIdx.x < TS) {
    const double v = cr[8 * TS + threadIdx.x];
    PW[it.vec_off + (int64_t)(Ti + I) * TS + threadIdx.x] = v;
    contrib = u[I * TS + threadIdx.x] * v;
  }
  return contrib;  // this thread's share of u^T S_bb u; the caller block-sums once per phase
}

// ---- R2: forward item (conductor patch s, aug row block I): Z_I = X_IJ f_J / f_p - Phi^T f_r --
__device__ __forceinline__ void fw_item(const ItemDesc& it, const double* Xr, const double* Fv, double* Zv, double* sm) {
  const int I = it.I, Tr = it.Ti + it.Tb;
  const int Jn = (I < Tr) ? I + 1 : Tr;
  const int64_t vo = it.vec_off;
  const double* X = Xr + it.a_off;
  double part[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) part[r] = 0.0;
  gemv_row_g([&](int J) { return X + tri_off(I, J); }, 0, Jn, sm,
             [&] {
               for (int e = threadIdx.x; e < Jn * TS; e += blockDim.x) sm[e] = ldcg(Fv + vo + e);
             },
             part);
  const double sum = warp_reduce8(part);
  const int lane = threadIdx.x & 31, row0 = (threadIdx.x >> 5) * 8;
  if ((lane & 3) == 0) {
    const int64_t idx = vo + (int64_t)I * TS + row0 + warp_reduce8_row();
    Zv[idx] = (I < Tr) ? sum : ldcg(Fv + idx) - sum;
  }
  __syncthreads();
}

// ---- E3: backward item (patch s, r column block J): a_J = X_rr^T u - Phi N Pc, scattered ----
template <class PcF>
__device__ __forceinline__ void bw_item(const DevPlan& D, const ItemDesc& it, const double* Xr, const double* Zv, const double* XWv,
                        PcF pc, double* a_loc, int nloc, double* sm) {
  const int s = it.s, J = it.I, Ti = it.Ti, Tr = Ti + it.Tb, T = it.T, np = it.np;
  const int64_t vo = it.vec_off;
  const int* grp = D.p_grp + it.p_off;
  const int* aug = D.aug + D.aug_off[s];
  const double* X = Xr + it.a_off;
  double* sx = sm;                 // (T - J) * 64
  double* cr = sm + (T - J) * TS;  // 8 * 64
  double c0 = 0.0, c1 = 0.0;
  gemv_col_g([&](int I) { return X + tri_off(I, J); }, J, T, sx,
             [&] {
               for (int e = threadIdx.x; e < (T - J) * TS; e += blockDim.x) {
                 const int i = J * TS + e;
                 double val;
                 if (i < Ti * TS) val = ldcg(Zv + vo + i);
                 else if (i < Tr * TS) val = ldcg(Zv + vo + i) - ldcg(XWv + vo + i);
                 else {
                   const int t = i - Tr * TS;
                   val = (t < np) ? -pc(grp[t]) : 0.0;
                 }
                 sx[e] = val;
               }
             },
             c0, c1);
  const double acc = col_finish(c0, c1, cr);
  double* as = a_loc + (int64_t)s * nloc;
  if (threadIdx.x < TS) {
    const int a = aug[J * TS + threadIdx.x];
    if (a >= 0) as[a] = acc;
  }
  // primal values a_p = N Pc (written by the items of column block 0)
  if (J == 0)
    for (int t = threadIdx.x; t < np; t += blockDim.x) as[aug[Tr * TS + t]] = pc(grp[t]);
  __syncthreads();
}

// ---- sparse coarse forward row I of node x: y_V = L_VV^-1 f_V (rows < TV) or the update
// f_B - L_BV L_VV^-1 f_V (rows >= TV), f gathered by the node's program: tag bit 55 set = the
// child's forward vector (CW), else gsrc(aug index, owner rank) of a patch's primal row.
// Rows are split into column chunks of Tp tiles (ItemDesc: part = chunk, bc = chunks,
// sbb_off = first partial slot, Ti = counter): each chunk writes its partial row (chunk 0 also
// the row's own f for B rows), the last arriving chunk adds them in chunk order.
constexpr int64_t kTag = 1ll << 55, kIdx55 = kTag - 1;
constexpr int kKwMax = 8;  // sources per frontal position (host checks)
template <class GS>
__device__ __forceinline__ void fwc_item(const ItemDesc& it, const double* FR, const int64_t* prog, int kw, GS gsrc,
                                         double* CW, double* PB, unsigned int* cnt, double* sm) {
  const int I = it.I, TV = it.Tb, T = it.T;
  const int Jn = (I < TV) ? I + 1 : TV;
  const int nch = it.bc, c = it.part;
  const int cw = it.Tp;  // chunk width (tiles), chosen per level by the host
  const int J0 = (nch > 1) ? c * cw : 0, J1 = (nch > 1) ? min(Jn, J0 + cw) : Jn;
  const double* X = FR + it.a_off;
  __shared__ int s_lastf;
  // fixed-width sources: kw slots per frontal position (-1 = none), all issued at once
  auto fval = [&](int e) {
    const int64_t* sp = prog + it.p_off + (int64_t)e * kw;
    int64_t en[kKwMax];
#pragma unroll
    for (int q = 0; q < kKwMax; ++q) en[q] = (q < kw) ? sp[q] : -1;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kKwMax; ++q)
      if (en[q] >= 0) v += (en[q] & kTag) ? ldcg(CW + (en[q] & kIdx55)) : gsrc(en[q] & kIdx55, (int)(en[q] >> 56));
    return v;
  };
  const int lane = threadIdx.x & 31, row0 = (threadIdx.x >> 5) * 8;
  const int row = I * TS + row0 + warp_reduce8_row();
  // the row's own f (B rows, chunk 0): loads issued before the GEMV
  double frow = 0.0;
  if (I >= TV && c == 0 && (lane & 3) == 0) frow = fval(row);
  double part[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) part[r] = 0.0;
  gemv_row_g([&](int J) { return X + tri_off(I, J); }, J0, J1, sm,
             [&] {
               for (int e = threadIdx.x; e < (J1 - J0) * TS; e += blockDim.x) sm[e] = fval(J0 * TS + e);
             },
             part);
  const double sum = warp_reduce8(part);
  const double mine = (I < TV) ? sum : frow - sum;  // this chunk's share of the output
  if (nch == 1) {
    if ((lane & 3) == 0) CW[it.vec_off + row] = mine;
    __syncthreads();
    return;
  }
  if ((lane & 3) == 0) PB[(it.sbb_off + c) * TS + row0 + warp_reduce8_row()] = mine;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_lastf = ((atomicAdd(cnt + it.Ti, 1u) + 1) % (unsigned)nch) == 0;
  __syncthreads();
  if (s_lastf) {
    __threadfence();
    if (threadIdx.x < TS) {
      double v = 0.0;
      for (int q = 0; q < nch; ++q) v += ldcg(PB + (it.sbb_off + q) * TS + threadIdx.x);
      CW[it.vec_off + I * TS + threadIdx.x] = v;
    }
  }
  __syncthreads();
}
// ---- sparse coarse backward column block J of node x: x_V = L_VV^-T y_V - (L_BV L_VV^-1)^T x_B
// Long columns (B can hold thousands of groups) are split into row chunks (ItemDesc: part =
// chunk, bc = chunks, p_off = first partial slot, Ti = counter): each chunk writes its partial
// column sum, the last arriving chunk (monotone counter) adds the partials in chunk order.
// Rows are streamed through the shared scratch `ch` tiles at a time.
template <class Dummy = int>
__device__ __forceinline__ void bwc_item(const ItemDesc& it, const double* FR, const double* CW, const int* vl,
                                         const int* bl, double* Pcs, double* PB, unsigned int* cnt, double* sm,
                                         int ch) {
  const int J = it.I, TV = it.Tb, T = it.T, nV = it.np, nB = it.nb;
  const int nch = it.bc, c = it.part;
  const int cw = it.Tp;  // chunk height (tiles), chosen per level by the host
  const int Ib = J + c * cw, Ie = (nch > 1) ? min(T, Ib + cw) : T;
  const double* X = FR + it.a_off;
  double* sx = sm;
  double* cr = sm + (int64_t)ch * TS;
  __shared__ int s_last;
  double c0 = 0.0, c1 = 0.0;
  for (int I0 = Ib; I0 < Ie; I0 += ch) {
    const int I1 = min(Ie, I0 + ch);
    gemv_col_g([&](int I) { return X + tri_off(I, J); }, I0, I1, sx,
               [&] {
                 for (int e = threadIdx.x; e < (I1 - I0) * TS; e += blockDim.x) {
                   const int i = I0 * TS + e;
                   double val;
                   if (i < TV * TS) val = ldcg(CW + it.vec_off + i);
                   else {
                     const int t = i - TV * TS;
                     val = (t < nB) ? -ldcg(Pcs + bl[it.b_off + t]) : 0.0;
                   }
                   sx[e] = val;
                 }
               },
               c0, c1);
    __syncthreads();  // sx reused by the next chunk
  }
  const double acc = col_finish(c0, c1, cr);
  if (nch == 1) {
    if (threadIdx.x < TS) {
      const int j = J * TS + threadIdx.x;
      if (j < nV) Pcs[vl[it.sbb_off + j]] = acc;
    }
    __syncthreads();
    return;
  }
  if (threadIdx.x < TS) PB[(it.p_off + c) * TS + threadIdx.x] = acc;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = ((atomicAdd(cnt + it.Ti, 1u) + 1) % (unsigned)nch) == 0;
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x < TS) {
      double v = 0.0;
      for (int q = 0; q < nch; ++q) v += ldcg(PB + (it.p_off + q) * TS + threadIdx.x);
      const int j = J * TS + threadIdx.x;
      if (j < nV) Pcs[vl[it.sbb_off + j]] = v;
    }
  }
  __syncthreads();
}

constexpr unsigned long long kBarrierTimeoutNs = 30ull * 1000000000ull;  // 30 s watchdog

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p, int sys) {
  unsigned int v;
  if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_scope(int sys) {
  if (sys) __threadfence_system();
  else __threadfence();
}

// The per-block partials are double-buffered by round parity: a fast block may already write
// the partial of the next reducing barrier while a slow one still sums the previous round's
// (P5 and P7 reduce back to back; blocks without items run ahead).
// Barrier over every block of every rank, with an optional fused fixed-order sum of one
// value per block. `round` counts barriers (the same sequence in every block of every rank;
// the counters are monotone across launches).
//  * one rank: every block arrives on the rank counter and polls it; the sum is formed by
//    every block from the per-block partials in block order (lane-strided + xor butterfly).
//  * several ranks: two levels. The last arriving block of a rank (its leader) sums the
//    rank's partials in block order, publishes the rank partial, arrives on rank 0's global
//    counter (system scope for real GPUs), waits for all rank leaders and releases its rank;
//    every block then sums the rank partials in rank order. Identical totals everywhere.
struct NoHook {
  __device__ void operator()() const {}
};
// hook(): run by thread 0 right after this block's arrival, before it waits (used to issue the
// bulk copies of the next phase's first tiles so they stream in during the wait)
template <class Hook = NoHook>
__device__ __forceinline__ double grid_barrier(const StepArgs& A, int me, int bl, unsigned int& round, bool reduce, double value,
                               double* bcast, Hook hook = Hook()) {
  __shared__ int s_leader;
  __syncthreads();
  ++round;
  const int sys = A.sys_scope;
  BarMem* mine = A.bar[me];
  if (A.nranks == 1) {
    // arrival = release-add on the rank counter (orders this block's writes, made visible
    // to thread 0 by the __syncthreads above); departure = acquire poll
    if (threadIdx.x == 0) {
      if (reduce) A.partials[me][(round & 1) * A.nbr + bl] = value;
      red_release_gpu(&mine->local_count, 1u);
      hook();
      const unsigned long long t0 = gtimer();
      while ((int)(ld_acquire_u32(&mine->local_count, 0) - round * (unsigned int)A.nbr) < 0) {
        if (gtimer() - t0 > kBarrierTimeoutNs) __trap();  // a missing block: fail, never hang
      }
    }
    __syncthreads();
    if (!reduce) return 0.0;
    // fixed-order sum of the block partials, loaded by all threads in one round trip
    double t = 0.0;
    for (int j = threadIdx.x; j < A.nbr; j += NTHR) t += __ldcg(A.partials[me] + (round & 1) * A.nbr + j);
    return block_sum(t, bcast);
  }
  if (threadIdx.x == 0) {
    if (reduce) A.partials[me][(round & 1) * A.nbr + bl] = value;
    fence_scope(sys);
    const unsigned int old = atomicAdd(&mine->local_count, 1u);
    s_leader = (old + 1 == round * (unsigned int)A.nbr);
    hook();
  }
  __syncthreads();
  if (s_leader) {
    if (reduce) {
      double t = 0.0;
      for (int j = threadIdx.x; j < A.nbr; j += NTHR) t += __ldcg(A.partials[me] + (round & 1) * A.nbr + j);
      t = block_sum(t, bcast);
      if (threadIdx.x == 0) mine->rank_part[round & 1] = t;
    }
    if (threadIdx.x == 0) {
      fence_scope(sys);
      unsigned int* gc = &A.bar[0]->global_count;
      if (sys) atomicAdd_system(gc, 1u);
      else atomicAdd(gc, 1u);
      const unsigned long long t0 = gtimer();
      while ((int)(ld_acquire_u32(gc, sys) - round * (unsigned int)A.nranks) < 0) {
        if (gtimer() - t0 > kBarrierTimeoutNs) __trap();  // a missing rank: fail, never hang
      }
      fence_scope(sys);
      atomicExch(&mine->local_gen, round);
    }
  } else if (threadIdx.x == 0) {
    const unsigned long long t0 = gtimer();
    while ((int)(ld_acquire_u32(&mine->local_gen, 0) - round) < 0) {
      if (gtimer() - t0 > kBarrierTimeoutNs) __trap();
    }
  }
  if (threadIdx.x == 0) {
    fence_scope(sys);
    if (reduce) {
      double t = 0.0;
      for (int r = 0; r < A.nranks; ++r) t += *(volatile double*)&A.bar[r]->rank_part[round & 1];
      *bcast = t;
    }
  }
  __syncthreads();
  double total = 0.0;
  if (reduce) total = *bcast;
  __syncthreads();
  return total;
}

// rhs item (R1). c in {0,1,2}: component c of conductor patch s, F = (sigma/dt) M a + phi j_S
// with the mass apply sum-factorised (M_c = F_z (x) F_y (x) F_x, F_d = Md along d == c, Mb else;
// banded |i-i'| <= p) through shared memory; c = -1: insulator patch s, Z = phi(t) XJ.
__device__ __forceinline__ void rhs_item(const DevPlan& D, const StepArgs& A, int me, const ItemDesc& it, double t, double* sm) {
  const int s = it.s, c = it.I;
  const double sig = D.sigma[s], nu = D.nu[s];
  double phi = 0.0;
  if (A.source == 1) phi = A.src_amp * sinpi(2.0 * A.src_freq * t);
  else if (A.source == 2) phi = A.src_amp * (2.0 * M_PI * M_PI * nu * (1.0 - exp(-t)) + sig * exp(-t));
  else if (A.source == 3) phi = A.src_amp * exp(-t);  // template (3 nu - sigma) j_S - W^_(r,p)D (Pi_h S)_D (mms.cu)
  const int64_t vo = it.vec_off;
  if (c < 0) {
    const int R = it.T * TS;
    for (int pos = threadIdx.x; pos < R; pos += blockDim.x) A.Z[me][vo + pos] = phi * ldcg(A.XJ[me] + vo + pos);
    return;
  }
  const Geom& G = A.G;
  const Tables1D& tb = A.tb;
  const int p = G.p;
  const int nx = G.cdim[c][0], ny = G.cdim[c][1], nz = G.cdim[c][2];
  const int nn = nx * ny * nz;
  int off = 0;
  for (int cc = 0; cc < c; ++cc) off += G.cdim[cc][0] * G.cdim[cc][1] * G.cdim[cc][2];
  const double* as = (A.a_old[me] ? A.a_old[me] : A.a_loc[me]) + (int64_t)s * G.nloc + off;
  const double* gn = A.gnl[me];
  double* u0 = sm;
  double* u1 = sm + nn;
  const int n0 = tb.el[0] + p, n1 = tb.el[1] + p, n2 = tb.el[2] + p;
  const double* Fx = (c == 0) ? tb.base + tb.off_Md[0] : tb.base + tb.off_Mb[0];
  const double* Fy = (c == 1) ? tb.base + tb.off_Md[1] : tb.base + tb.off_Mb[1];
  const double* Fz = (c == 2) ? tb.base + tb.off_Md[2] : tb.base + tb.off_Mb[2];
  const int ldx = (c == 0) ? n0 - 1 : n0, ldy = (c == 1) ? n1 - 1 : n1, ldz = (c == 2) ? n2 - 1 : n2;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {  // x pass
    const int i = e % nx, jk = e / nx;
    double v = 0.0;
    for (int q = max(0, i - p); q <= min(nx - 1, i + p); ++q) v += Fx[i * ldx + q] * ldcg(as + jk * nx + q);
    u0[e] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {  // y pass
    const int i = e % nx, j = (e / nx) % ny, k = e / (nx * ny);
    double v = 0.0;
    for (int q = max(0, j - p); q <= min(ny - 1, j + p); ++q) v += Fy[j * ldy + q] * u0[i + nx * (q + ny * k)];
    u1[e] = v;
  }
  __syncthreads();
  const int* l2a = D.loc2aug + (int64_t)s * G.nloc + off;
  const double scale = sig / A.dt;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {  // z pass + scatter into aug order
    const int pos = l2a[e];
    if (pos < 0) continue;
    const int ij = e % (nx * ny), k = e / (nx * ny);
    double v = 0.0;
    for (int q = max(0, k - p); q <= min(nz - 1, k + p); ++q) v += Fz[k * ldz + q] * u1[ij + nx * ny * q];
    A.F[me][vo + pos] = scale * v + phi * A.JS[me][vo + pos] + (gn ? gn[vo + pos] : 0.0);
  }
  __syncthreads();
}


#define TSTAMP(slot) \
  if (A.tstamp && me == 0 && bl == 0 && threadIdx.x == 0 && it < 64 && step == 0) A.tstamp[it * 8 + (slot)] = gtimer()
// step-level stamps of step 0 (slots 512..527): R1..R5 ends, loop end, E1..E3 ends
#define SSTAMP(slot) \
  if (A.tstamp && me == 0 && bl == 0 && threadIdx.x == 0 && step == 0) A.tstamp[512 + (slot)] = gtimer()
// per-item durations of PCG iteration 2 of step 0 (phase-timing builds): itime[ph][global item]
#define ITIME_BEGIN unsigned long long it_t0 = 0; if (A.itime && step == 0 && it == 2 && threadIdx.x == 0) it_t0 = gtimer();
#define ITIME_END(ph, j)                                                                                   \
  if (A.itime && step == 0 && it == 2 && threadIdx.x == 0)                                                \
    A.itime[(ph) * A.itime_stride + A.boff[ph][gb] + (j)] = (double)(gtimer() - it_t0);
// per-block work-end stamps of PCG iteration 2 of step 0 (slots 528 + 8*block + phase)
#define WSTAMP(slot)                                                                   \
  if (A.tstamp && step == 0 && it == 2) {                                              \
    __syncthreads();                                                                   \
    if (threadIdx.x == 0 && gb < 4096) A.tstamp[528 + gb * 8 + (slot)] = gtimer();     \
  }

// the coarse phase: this block's PC items with their gather programs (shared or global)
#define PC_PHASE(GS)                                                                      \
  {                                                                                       \
    int64_t po = 0;                                                                       \
    FOR_ITEMS(PH_PC, w) {                                                                 \
      const int64_t* prog = s_pcbase ? s_pcbase + po : A.pcprog + w.vec_off;              \
      po += w.b_off;                                                                      \
      pc_item(D, A, A.Sinv[me], w.s, w.I, prog, GS, A.Ppart[me], smw, PF0(j_w));          \
    }                                                                                     \
  }
// first item of a run of items of the same patch (and P5 part) in this block's list: only it
// gathers the patch's input vector, the following items reuse it from shared memory
// gather code of an item, set by the host in bits 4-5 of ItemDesc::part: 0 = reuse the
// previous item's gather, 1 = gather this item's rows, 2 = gather the whole patch vector (the
// next item of this block is of the same patch and part)
#define GAT(ph, var) (((var).part >> 4) & 3)
// loop over this block's items of phase ph (shared-memory copy or global list)
#define FOR_ITEMS(ph, var)                                  \
  for (int j_##var = 0; j_##var < s_icnt[ph]; ++j_##var)    \
    if (const ItemDesc& var = s_ip[ph][j_##var]; true)

// Side work of the F-apply's sparse coarse solve (TCG_OVERLAP): this block's PH_P1B items
// (y1 = S_bb^-1 v into Y, src = P1's input v) run while the block waits for a coarse dependency;
// *sum collects this thread's share of v . y1 in list order. An item that reuses the patch vector
// gathered by the previous one (GAT 0) gathers again when a coarse item ran in between (the
// scratch is shared).
struct NoSide {
  __device__ __forceinline__ bool left() const { return false; }
  __device__ __forceinline__ void run() {}
  __device__ __forceinline__ void clobber() {}
};
template <class Src>
struct SideWork {
  Src src;
  double* sum;
  int j, n;
  bool clob;
  const ItemDesc* items;
  const double* SI;
  double* Y;
  double* smw;
  double* red;
  // (force-inlined with symv_patch: an out-of-line call would take the address of the kernel's
  // parameter block through src's captures and cost a 3.6 KB local copy per thread)
  __device__ __forceinline__ bool left() const { return j < n; }
  __device__ __forceinline__ void clobber() { clob = true; }
  __device__ __forceinline__ void run() {
    const ItemDesc& w = items[j++];
    if ((w.part & 10) == 10) *sum += symv_patch(w, SI, Y, src, smw, nullptr, 0);
    else *sum += symv_item(w, SI, Y, src, smw, red, nullptr, 0, clob || GAT(PH_P1B, w));
    clob = false;
  }
};

// =======================================================================================
// Persistent cooperative time stepper: A.nsteps implicit-Euler steps in one launch, over
// all ranks of the job. Control flow depends only on values every block of every rank
// computes identically, so all blocks run the same sequence of barriers.
// =======================================================================================
template <bool MULTI, bool BC>
__global__ void __launch_bounds__(NTHR, 2) k_steps(DevPlan D, StepArgs A) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[NTHR];
  __shared__ double bcast[NTHR / 32];
  __shared__ const ItemDesc* s_ip[NPH];
  __shared__ int s_icnt[NPH];
  __shared__ const LamC* s_lc;
  __shared__ const int64_t* s_pcbase;
  __shared__ const BPos* s_bp;
  __shared__ __align__(8) unsigned long long s_mb;  // mbarrier of the tile prefetch
  __shared__ int s_pfn;                            // tiles prefetched for the coming phase
  double* const tbuf = sm;                         // A.npf prefetched tiles
  double* const smw = sm + (size_t)A.npf * TSZ;    // item scratch
  // MULTI = false: one rank, every owner lookup folds to rank 0 at compile time
  const int me = MULTI ? A.rank_base + (int)blockIdx.x / A.nbr : 0;  // this block's rank
  const int bl = MULTI ? (int)blockIdx.x % A.nbr : (int)blockIdx.x;   // block index within the rank
  const int64_t m = D.m;
  const int64_t gb = (int64_t)me * A.nbr + bl;
  const int64_t k0 = min(m, gb * A.lam_chunk), k1 = min(m, k0 + A.lam_chunk);
  const int nk = (int)(k1 - k0);
  unsigned int round = A.round0;
  if (A.tstamp && threadIdx.x == 0 && gb < 4096) {  // phase-timing builds: the block's SM (slot 4)
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    A.tstamp[528 + gb * 8 + 4] = smid;
  }
  const double* Xr = D.Ar[me];
  const double* Sr = D.Sbbr[me];
  const double* SIr = D.SIr[me];
  // ---- per-launch setup: item lists (and lambda-chunk index data) into shared memory ----
  {
    ItemDesc* ic = reinterpret_cast<ItemDesc*>(smw + A.scratch);
    int pos = 0;
    if (threadIdx.x == 0) {
      mbar_init(&s_mb);
      s_pfn = 0;
    }
#pragma unroll
    for (int ph = 0; ph < NPH; ++ph)  // constant indices: no local copy of the parameter block
      if (threadIdx.x == ph) {
        const int b = A.boff[ph][gb], e = A.boff[ph][gb + 1];
        s_icnt[ph] = e - b;
        s_ip[ph] = A.items[ph] + b;
      }
    __syncthreads();
    if (A.cache_items) {
      for (int ph = 0; ph < NCACHE; ++ph) {
        const int n = s_icnt[ph];
        const int4* src = reinterpret_cast<const int4*>(s_ip[ph]);
        int4* dst = reinterpret_cast<int4*>(ic + pos);
        for (int q = threadIdx.x; q < n * (int)(sizeof(ItemDesc) / 16); q += blockDim.x) dst[q] = src[q];
        __syncthreads();
        if (threadIdx.x == 0) s_ip[ph] = ic + pos;
        pos += n;
      }
    }
    int64_t* pcp = reinterpret_cast<int64_t*>(ic + pos);
    int64_t plen = 0;
    if (A.cache_pcprog) {
      const ItemDesc* pit = s_ip[PH_PC];
      for (int j = 0; j < s_icnt[PH_PC]; ++j) {
        const int64_t o = pit[j].vec_off, n = pit[j].b_off;
        for (int64_t q = threadIdx.x; q < n; q += blockDim.x) pcp[plen + q] = A.pcprog[o + q];
        plen += n;
      }
      plen = (plen + 1) & ~(int64_t)1;  // keep 16-byte alignment
    }
    if (threadIdx.x == 0) s_pcbase = A.cache_pcprog ? pcp : nullptr;
    LamC* lc = reinterpret_cast<LamC*>(pcp + plen);
    if (A.cache_lam) {
      for (int q = threadIdx.x; q < nk; q += blockDim.x) {
        const int64_t k = k0 + q;
        lc[q] = LamC{D.lam_idx_p[k], D.lam_idx_m[k], D.wplus[k], D.wminus[k], D.lam_patch_p[k], D.lam_patch_m[k]};
      }
    }
    if (threadIdx.x == 0) s_lc = A.cache_lam ? lc : nullptr;
    BPos* bc = reinterpret_cast<BPos*>(lc + (A.cache_lam ? nk : 0));
    if (BC) {
      for (int q = A.bploff[gb]; q < A.bploff[gb + 1]; ++q) {
        const int s = A.bpl[2 * q], off = A.bpl[2 * q + 1];
        int nbs = 0;
        int64_t bo = 0;
        nbs = D.nb[s];
        bo = D.b_off[s];
        for (int e = threadIdx.x; e < nbs; e += blockDim.x) {
          const int64_t bb = bo + e;
          bc[off + e] = BPos{D.b_part[bb], D.b_lam[bb], 0, D.b_aown[bb], D.b_apart[bb], D.b_sign[bb]};
        }
      }
    }
    if (threadIdx.x == 0) s_bp = bc;
    __syncthreads();
  }
  const LamC* lc = s_lc;
  const BPos* bpc = s_bp;
  // b-position record of (item, bb = b_off + pos): shared cache or the global tables
  auto bget = [&](const ItemDesc& iw, int64_t bb, int pos) -> BPos {
    if (BC && iw.bc >= 0) return bpc[iw.bc + pos];
    return BPos{D.b_part[bb], D.b_lam[bb], 0, D.b_aown[bb], D.b_apart[bb], D.b_sign[bb]};
  };
  auto lidx_p = [&](int64_t k) { return lc ? lc[k - k0].ip : D.lam_idx_p[k]; };
  auto lidx_m = [&](int64_t k) { return lc ? lc[k - k0].im : D.lam_idx_m[k]; };
  auto lw_p = [&](int64_t k) { return lc ? lc[k - k0].wp : D.wplus[k]; };
  auto lw_m = [&](int64_t k) { return lc ? lc[k - k0].wm : D.wminus[k]; };
  auto lpat_p = [&](int64_t k) { return MULTI ? (lc ? lc[k - k0].pp : D.lam_patch_p[k]) : 0; };
  auto lpat_m = [&](int64_t k) { return MULTI ? (lc ? lc[k - k0].pm : D.lam_patch_m[k]) : 0; };
  auto lown = [&](int64_t k) { return MULTI ? ((int)k / (int)A.lam_chunk) / A.nbr : 0; };
  auto pown = [&](int s) { return MULTI ? D.owner[s] : 0; };
  auto own_idx = [&](const ItemDesc& it, int pos) { return it.vec_off + (int64_t)it.Ti * TS + pos; };
  auto pcf = [&](int64_t g) { return A.sparse ? ldcg(A.Pcs[me] + g) : pc_get<MULTI>(A, g); };
  auto yv = [&](int o, int64_t i) { return ldcg(A.Y[o] + i) + ldcg(A.Y2[o] + i); };  // y = Y + Y2
  // partner patch of b position bb (other endpoint of its multiplier)
  auto ppatch = [&](int64_t bb) {
    if (!MULTI) return 0;
    const int k = D.b_lam[bb];
    return D.b_sign[bb] > 0 ? D.lam_patch_m[k] : D.lam_patch_p[k];
  };
  // ---- tile prefetch: the first item of phase ph, up to A.npf tiles (thread 0, in a barrier) ----
  unsigned int pf_par = 0;
  auto pf_issue = [&](int ph) {
    int n = 0;
    const double* src[2] = {nullptr, nullptr};
    if (A.npf > 0 && ph >= 0 && ph < NCACHE && !((c_step_flags >> (4 + ph)) & 1) && s_icnt[ph] > 0) {
      const ItemDesc& w = s_ip[ph][0];
      if (ph == PH_P1 && (w.part & 8)) {  // explicit S_bb^-1 apply (row block I, or patch from I = 0)
        n = min(w.I + 1, A.npf);
        for (int q = 0; q < n; ++q) src[q] = SIr + w.sbb_off + tri_off(w.I, q);
      } else if (ph == PH_P1) {
        const int Jn = (w.I < w.Tb) ? w.I + 1 : w.Tb;
        n = min(Jn, A.npf);
        for (int q = 0; q < n; ++q) src[q] = Xr + w.a_off + tri_off(w.Ti + w.I, w.Ti + q);
      } else if (ph == PH_PC) {
        const int J0 = w.I * A.ch, J1 = min(D.Tc, J0 + A.ch);
        n = min(J1 - J0, A.npf);
        for (int q = 0; q < n; ++q) src[q] = A.Sinv[me] + ((int64_t)w.s * D.Tc + J0 + q) * TSZ;
      } else if (ph == PH_P5) {
        const int I0 = (w.part & 1) ? w.Tb : w.I, I1 = (w.part & 3) ? w.Tb + w.Tp : w.Tb;
        n = min(I1 - I0, A.npf);
        for (int q = 0; q < n; ++q) src[q] = Xr + w.a_off + tri_off(w.Ti + I0 + q, w.Ti + w.I);
      } else if (ph == PH_SY) {
        n = min(w.I + 1, A.npf);
        for (int q = 0; q < n; ++q) src[q] = Sr + w.sbb_off + tri_off(w.I, q);
      }
    }
    if (n > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&s_mb, (uint32_t)(n * TSZ * sizeof(double)));
      for (int q = 0; q < n; ++q) bulk_g2s(tbuf + q * TSZ, src[q], TSZ * sizeof(double), &s_mb);
    }
    s_pfn = n;
  };
  // phase start: wait for the prefetched tiles (all threads); returns their count
  auto pf_wait = [&]() -> int {
    const int n = s_pfn;
    if (n > 0) {
      mbar_wait(&s_mb, pf_par);
      pf_par ^= 1u;
    }
    return n;
  };
  auto hook = [&](int ph) { return [&, ph]() { pf_issue(ph); }; };
  int64_t hoff = A.hist_off;
  int total_status = 0;

  // grid barrier that issues the next phase's tile prefetch during the wait and, after it,
  // waits for the tiles (npf_cur = tiles of that phase's first item now in tbuf)
  int npf_cur = 0;
  auto bar = [&](int ph_next, bool reduce, double v) -> double {
    // every thread orders its generic-proxy reads of tbuf before the async-proxy (bulk copy)
    // overwrite that thread 0 issues after the barrier's __syncthreads (WAR across proxies)
    if (A.npf > 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const double r = grid_barrier(A, me, bl, round, reduce, v, bcast, [&]() { pf_issue(ph_next); });
    npf_cur = pf_wait();
    return r;
  };
#define PF0(j) ((j) == 0 ? tbuf : nullptr), ((j) == 0 ? npf_cur : 0)
  // sparse coarse solve S_pp x = sum_s N_s^T (src): forward levels bottom-up, backward levels
  // top-down, a grid barrier between levels (the caller's barrier follows the last one)
  // (phase-timing builds: block 0 stamps every level of the coarse solves of step 0 into
  // tstamp[528 + 8 * 4096 + ...], slot = call * 64 + level phase)
  int cstamp_call = 0;
  auto cstamp = [&](int k) {
    if (A.tstamp && me == 0 && bl == 0 && threadIdx.x == 0 && cstamp_call < 8 && k < 64)
      A.tstamp[528 + 8 * 4096 + cstamp_call * 64 + k] = gtimer();
  };
  // Dataflow (default): no grid barrier between levels. A forward item of node x waits until
  // all forward items of x's children are done (their B rows are x's input); a backward item
  // waits for the parent's backward items (x_B lives in ancestors, all solved before the
  // parent's) or, at the root, for the root's own forward items. Every block runs its items
  // level by level, dependencies point to earlier levels, and all blocks are co-resident, so
  // the waits always end. Counters are monotone within a launch (zeroed before it): target =
  // solves so far x item count.
  unsigned int cuse = 0;  // coarse solves in this launch (uniform)
  // (side: work of this block that does not depend on the coarse solve, the S_bb^-1 items of
  // PH_P1B. While the awaited counter is short of its target the block runs one side item and
  // polls again; with none left it spins as before. Item order within the side list is fixed, so
  // the sums they return do not depend on the interleaving.)
  auto cwait = [&](const unsigned int* c, unsigned int target, auto& side) {
    while (side.left()) {
      if (__syncthreads_or(threadIdx.x == 0 && (int)(ld_acquire_u32(c, 0) - target) >= 0)) return;
      side.run();
    }
    if (threadIdx.x == 0) {
      const unsigned long long t0 = gtimer();
      while ((int)(ld_acquire_u32(c, 0) - target) < 0)
        if (gtimer() - t0 > kBarrierTimeoutNs) __trap();
    }
    __syncthreads();
  };
  auto coarse_sparse = [&](auto gsrc, auto& side) {
    cstamp(0);
    ++cuse;
    const int nn = A.cf_nn;
    unsigned int* kd = A.cf_dflow[me];
    unsigned int* fd = kd + nn;
    unsigned int* bd = kd + 2 * nn;
    for (int lv = 0; lv < A.cf_levels; ++lv) {
      const int b = A.cf_fw_off[lv * A.nbr + bl], e = A.cf_fw_off[lv * A.nbr + bl + 1];
      for (int j = b; j < e; ++j) {
        const ItemDesc& it = A.cf_fw[j];
        const int4 nd = A.cf_node[it.s];
        if (!A.cf_sync && nd.w > 0) cwait(kd + it.s, cuse * (unsigned int)nd.w, side);
        side.clobber();
        fwc_item(it, A.FR, A.cf_prog, A.cf_kw, gsrc, A.CW[me], A.cf_pb[me], A.cf_cnt[me], smw);
        if (!A.cf_sync && threadIdx.x == 0) {  // fwc_item ended with __syncthreads
          __threadfence();
          if (nd.x >= 0) atomicAdd(kd + nd.x, 1u);
          atomicAdd(fd + it.s, 1u);
        }
      }
      if (A.cf_sync) bar(-1, false, 0.0);
      cstamp(1 + lv);
    }
    for (int lv = A.cf_levels - 1; lv >= 0; --lv) {
      const int b = A.cf_bw_off[lv * A.nbr + bl], e = A.cf_bw_off[lv * A.nbr + bl + 1];
      for (int j = b; j < e; ++j) {
        const ItemDesc& it = A.cf_bw[j];
        if (!A.cf_sync) {  // x_B from the ancestors, y_V from x's own forward rows
          const int2 dp = A.cf_bwdep[it.s];
          if (dp.x >= 0) cwait(bd + dp.x, cuse * (unsigned int)dp.y, side);
          cwait(fd + it.s, cuse * (unsigned int)A.cf_node[it.s].y, side);
        }
        side.clobber();
        bwc_item(it, A.FR, A.CW[me], A.cf_vl, A.cf_bl, A.Pcs[me], A.cf_pb[me], A.cf_cnt[me], smw, A.scratch / TS - 9);
        if (!A.cf_sync && threadIdx.x == 0) {
          __threadfence();
          atomicAdd(bd + it.s, 1u);
        }
      }
      if (A.cf_sync && lv > 0) bar(-1, false, 0.0);
      cstamp(2 * A.cf_levels - lv);
    }
    ++cstamp_call;
    if (side.left()) {  // the rest of the side items (the last coarse item may still read smw)
      __syncthreads();
      while (side.left()) side.run();
    }
  };
  NoSide no_side;
  auto make_side = [&](auto vsrc, double* sum) {
    return SideWork<decltype(vsrc)>{vsrc, sum, 0, s_icnt[PH_P1B], true, s_ip[PH_P1B], SIr, A.Y[me], smw, red};
  };
#define COARSE2(GS, SIDE)         \
  if (A.sparse) {                 \
    coarse_sparse(GS, SIDE);      \
  } else {                        \
    PC_PHASE(GS);                 \
  }
#define COARSE(GS) COARSE2(GS, no_side)
  // ---- mode 1: the dual operator alone, q = F p, A.nsteps times (F-apply benchmark / test) ----
  for (int rep = 0; A.mode == 1 && rep < A.nsteps; ++rep) {
    const int step = -1, it = -1;  // no stamps
    (void)step;
    (void)it;
    {
      auto vsrc = [&](const ItemDesc& iw, int64_t bb, int pos) {
        const BPos q = bget(iw, bb, pos);
        return q.sign * ldcg(A.pk[0][lown(q.k)] + q.k);
      };
      FOR_ITEMS(PH_P1, w) {
        if ((w.part & 10) == 10) symv_patch(w, SIr, A.Y[me], vsrc, smw, PF0(j_w), Xr, A.XW[me]);
        else if (w.part & 8) symv_item(w, SIr, A.Y[me], vsrc, smw, red, PF0(j_w), GAT(PH_P1, w));
        else p1_item(w, Xr, vsrc, A.XW[me], smw, PF0(j_w), GAT(PH_P1, w));
      }
      bar(PH_PC, false, 0.0);
      double unused = 0.0;
      auto side = make_side(vsrc, &unused);
      COARSE2(([&](int64_t i, int o) { return ldcg(A.XW[MULTI ? o : 0] + i); }), side);
    }
    bar(PH_P5, false, 0.0);
    FOR_ITEMS(PH_P5, w) {
      auto zero = [&](const ItemDesc&, int64_t, int) { return 0.0; };
      if ((w.part & 3) == 3) p5_phi_patch(w, Xr, D.p_grp, pcf, zero, A.Y2[me], smw);
      else p5_item(w, Xr, A.XW[me], D.p_grp, pcf, zero, A.Y[me], A.Y2[me], smw, red, nullptr, PF0(j_w), GAT(PH_P5, w));
    }
    bar(-1, false, 0.0);
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x)
      A.r[1][me][k] = yv(pown(lpat_p(k)), lidx_p(k)) - yv(pown(lpat_m(k)), lidx_m(k));
    bar(PH_P1, false, 0.0);
  }
  for (int step = 0; A.mode == 0 && step < A.nsteps; ++step) {
    const double t = (A.step0 + step + 1) * A.dt;
    int it = 0;
    SSTAMP(0);
    // ---- R1 rhs ----
    FOR_ITEMS(PH_RHS, w) rhs_item(D, A, me, w, t, smw);
    bar(-1, false, 0.0);
    SSTAMP(1);
    // ---- R2 forward (conductors) ----
    FOR_ITEMS(PH_FW, w) fw_item(w, Xr, A.F[me], A.Z[me], smw);
    bar(PH_PC, false, 0.0);
    SSTAMP(2);
    // ---- R3 p0 = S_pp^-1 sum N^T Z_p ----
    COARSE(([&](int64_t i, int o) { return ldcg(A.Z[MULTI ? o : 0] + i); }));
    bar(PH_P5, false, 0.0);
    if (A.dbg_stop == 1) break;
    SSTAMP(3);
    // ---- R4 y = X_bb^T Z_b - Phi_b N p0 (the X_bb form of the F-apply's second half) ----
    FOR_ITEMS(PH_E5, w)
      p5_item(w, Xr, A.Z[me], D.p_grp, pcf, [&](const ItemDesc&, int64_t, int) { return 0.0; }, A.Y[me], A.Y2[me], smw,
              red, nullptr, nullptr, 0, GAT(PH_E5, w));
    bar(PH_SY, false, 0.0);
    SSTAMP(4);
    // ---- R5 d = B y; r0 = d, lambda = 0; z0 = M^-1 d, rho0 ----
    // (warm start: rho0 = d^T M^-1 d stays the reference of the stopping rule, so warm and
    // cold runs share one absolute target)
    const int nW = A.warm ? max(0, min(A.step0 + step - A.warm_base, A.warm)) : 0;
    double rho0;
    {
      double loc = 0.0;
      FOR_ITEMS(PH_SY, w)
        loc += symv_item(w, Sr, A.PW[me],
                         [&](const ItemDesc& iw, int64_t bb, int pos) {
                           const BPos q = bget(iw, bb, pos);
                           return q.aown * (yv(me, own_idx(iw, pos)) - yv(pown(ppatch(bb)), q.part));
                         },
                         smw, red, PF0(j_w), GAT(PH_SY, w));
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const double dk = yv(pown(lpat_p(k)), lidx_p(k)) - yv(pown(lpat_m(k)), lidx_m(k));
        A.r[0][me][k] = dk;
        A.pk[0][me][k] = 0.0;
        A.lam[me][k] = 0.0;
        if (A.warm) A.dsave[me][k] = dk;
      }
      loc = block_sum(loc, red);
      rho0 = bar(PH_P1, true, loc);
    }
    SSTAMP(5);
    int status = 0;  // 0 running, 1 converged, 2 failed
    double rz = rho0;
    if (!(rho0 >= 0.0)) status = 2;
    else if (!(rho0 > 0.0) || m == 0) status = 1;  // d = 0: lambda = 0 after 0 iterations
    double rho = rho0, beta = 0.0;
    int rp = 0, pp = 0;
    double rel0 = 1.0;
    if (nW > 0 && status == 0) {
      // ---- W1: Galerkin start on span{W_j} (oracle Oracle.pcg, R20): dot products
      // b_j = W_j.d, G_ij = (W_i.FW_j + W_j.FW_i)/2 over the block's lambda chunk ----
      __shared__ double s_g[KW_NV], s_c[KW];
      const int64_t gs = A.step0 + step;
      double acc[KW_NV];
#pragma unroll
      for (int v = 0; v < KW_NV; ++v) acc[v] = 0.0;
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const double dk = ldcg(A.dsave[me] + k);
        double wv[KW], fv[KW];
#pragma unroll
        for (int j = 0; j < KW; ++j) {
          wv[j] = fv[j] = 0.0;
          if (j < nW) {
            const int64_t so = ((gs - nW + j) % A.warm) * m + k;
            wv[j] = ldcg(A.Wr[me] + so);
            fv[j] = ldcg(A.FWr[me] + so);
          }
        }
#pragma unroll
        for (int j = 0; j < KW; ++j) acc[j] += wv[j] * dk;
#pragma unroll
        for (int i = 0; i < KW; ++i)
#pragma unroll
          for (int j = i; j < KW; ++j) acc[kw_idx(i, j)] += 0.5 * (wv[i] * fv[j] + wv[j] * fv[i]);
      }
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
      for (int v = 0; v < KW_NV; ++v) {
        const double t = warp_sum(acc[v]);
        if (lane == 0) red[warp * KW_NV + v] = t;
      }
      __syncthreads();
      if (threadIdx.x < KW_NV) {
        double t = 0.0;
        for (int w2 = 0; w2 < NTHR / 32; ++w2) t += red[w2 * KW_NV + threadIdx.x];
        if (!MULTI) A.wpart[me][((gs & 1) * A.nbr + bl) * KW_NV + threadIdx.x] = t;
        else s_g[threadIdx.x] = t;
      }
      if (!MULTI) {
        bar(-1, false, 0.0);
        // fixed-order sums over the blocks (warp v % 8 sums value v), identical in every block
        for (int v = warp; v < KW_NV; v += NTHR / 32) {
          double t = 0.0;
          for (int b2 = lane; b2 < A.nbr; b2 += 32) t += ldcg(A.wpart[me] + ((gs & 1) * A.nbr + b2) * KW_NV + v);
          t = warp_sum(t);
          if (lane == 0) s_g[v] = t;
        }
        __syncthreads();
      } else {
        __syncthreads();
        for (int v = 0; v < KW_NV; ++v) {
          const double pv = s_g[v];
          const double t = bar(-1, true, pv);
          __syncthreads();
          if (threadIdx.x == 0) s_g[v] = t;
          __syncthreads();
        }
      }
      // G c = b by Cholesky in index order, skipping columns whose pivot <= 1e-12 max G_ii
      // (the oracle's chol_skip_solve); one thread, broadcast through shared memory
      if (threadIdx.x == 0) {
        double L[KW][KW], y[KW], c[KW];
        bool act[KW];
        double gmax = 0.0;
        for (int i = 0; i < nW; ++i) gmax = fmax(gmax, s_g[kw_idx(i, i)]);
        for (int j = 0; j < KW; ++j) {
          act[j] = false;
          y[j] = c[j] = 0.0;
          for (int i = 0; i < KW; ++i) L[i][j] = 0.0;
        }
        for (int j = 0; j < nW; ++j) {
          double sj = s_g[kw_idx(j, j)];
          for (int q = 0; q < j; ++q)
            if (act[q]) sj -= L[j][q] * L[j][q];
          if (!(sj > 1e-12 * gmax)) continue;
          act[j] = true;
          L[j][j] = sqrt(sj);
          for (int i = j + 1; i < nW; ++i) {
            double t = s_g[kw_idx(j, i)];
            for (int q = 0; q < j; ++q)
              if (act[q]) t -= L[i][q] * L[j][q];
            L[i][j] = t / L[j][j];
          }
        }
        for (int j = 0; j < nW; ++j)
          if (act[j]) {
            double t = s_g[j];
            for (int q = 0; q < j; ++q)
              if (act[q]) t -= L[j][q] * y[q];
            y[j] = t / L[j][j];
          }
        for (int j = nW - 1; j >= 0; --j)
          if (act[j]) {
            double t = y[j];
            for (int q = j + 1; q < nW; ++q)
              if (act[q]) t -= L[q][j] * c[q];
            c[j] = t / L[j][j];
          }
        for (int j = 0; j < KW; ++j) s_c[j] = c[j];
      }
      __syncthreads();
      // lambda0 = sum c_j W_j, r0 = d - sum c_j FW_j (own chunk)
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        double l0 = 0.0, rr = ldcg(A.dsave[me] + k);
        for (int j = 0; j < nW; ++j) {
          const int64_t so = ((gs - nW + j) % A.warm) * m + k;
          l0 += s_c[j] * ldcg(A.Wr[me] + so);
          rr -= s_c[j] * ldcg(A.FWr[me] + so);
        }
        A.lam[me][k] = l0;
        A.r[1][me][k] = rr;
      }
      bar(PH_SY, false, 0.0);
      // ---- W2: z0 = M^-1 r0, rho = r0^T z0 ----
      double loc = 0.0;
      FOR_ITEMS(PH_SY, w)
        loc += symv_item(w, Sr, A.PW[me],
                         [&](const ItemDesc& iw, int64_t bb, int pos) {
                           const BPos q = bget(iw, bb, pos);
                           return q.aown * q.sign * ldcg(A.r[1][lown(q.k)] + q.k);
                         },
                         smw, red, PF0(j_w), GAT(PH_SY, w));
      loc = block_sum(loc, red);
      rz = bar(PH_P1, true, loc);
      rho = rz;
      rp = 1;
      rel0 = sqrt(fmax(rz, 0.0) / rho0);
      if (!(rz == rz)) status = 2;
      else if (rel0 <= A.rtol) status = 1;
    }
    if (me == 0 && bl == 0 && threadIdx.x == 0) A.hist[0][hoff] = rel0;
    while (status == 0) {
      TSTAMP(0);
      double* const* pprev = A.pk[pp];
      double* pcur = A.pk[pp ^ 1][me];
      // P1: p = z + beta p_prev on the fly; v = B^T p; w = X_bb v, -g = -Phi^T v; owners store p
      // (sbbinv: y1 = S_bb^-1 v -> Y instead of w, and its share v . y1 of p^T F p -> loc1)
      double loc1 = 0.0;
      auto vnew = [&](const ItemDesc& iw, int64_t bb, int pos) {
        const BPos q = bget(iw, bb, pos);
        return q.aown * ldcg(A.PW[me] + own_idx(iw, pos)) + q.apart * ldcg(A.PW[pown(ppatch(bb))] + q.part) +
               q.sign * beta * ldcg(pprev[lown(q.k)] + q.k);
      };
      {
        // the block's own lambda chunk first (independent loads in flight before the items)
        double pv = 0.0;
        const int64_t kq = k0 + threadIdx.x;
        if (kq < k1)
          pv = lw_p(kq) * ldcg(A.PW[pown(lpat_p(kq))] + lidx_p(kq)) -
               lw_m(kq) * ldcg(A.PW[pown(lpat_m(kq))] + lidx_m(kq)) + beta * ldcg(pprev[me] + kq);
        FOR_ITEMS(PH_P1, w) {
          ITIME_BEGIN
          if ((w.part & 10) == 10) loc1 += symv_patch(w, SIr, A.Y[me], vnew, smw, PF0(j_w), Xr, A.XW[me]);
          else if (w.part & 8) loc1 += symv_item(w, SIr, A.Y[me], vnew, smw, red, PF0(j_w), GAT(PH_P1, w));
          else p1_item(w, Xr, vnew, A.XW[me], smw, PF0(j_w), GAT(PH_P1, w));
          ITIME_END(PH_P1, j_w)
        }
        if (kq < k1) pcur[kq] = pv;
        for (int64_t k = kq + blockDim.x; k < k1; k += blockDim.x)
          pcur[k] = lw_p(k) * ldcg(A.PW[pown(lpat_p(k))] + lidx_p(k)) -
                    lw_m(k) * ldcg(A.PW[pown(lpat_m(k))] + lidx_m(k)) + beta * ldcg(pprev[me] + k);
      }
      WSTAMP(0);
      bar(PH_PC, false, 0.0);
      TSTAMP(1);
      // PC (the PH_P1B items, if any, run under its dependency waits)
      {
        auto side = make_side(vnew, &loc1);
        COARSE2(([&](int64_t i, int o) { return ldcg(A.XW[MULTI ? o : 0] + i); }), side);
      }
      WSTAMP(1);
      bar(PH_P5, false, 0.0);
      TSTAMP(2);
      // P5 (+ partial p^T F p)
      double* const* pcurt = A.pk[pp ^ 1];
      double pq;
      {
        double loc = loc1;
        auto vcur = [&](const ItemDesc& iw, int64_t bb, int pos) {
          const BPos q = bget(iw, bb, pos);
          return q.sign * ldcg(pcurt[lown(q.k)] + q.k);
        };
        FOR_ITEMS(PH_P5, w) {
          ITIME_BEGIN
          if ((w.part & 3) == 3) loc += p5_phi_patch(w, Xr, D.p_grp, pcf, vcur, A.Y2[me], smw);
          else
          loc += p5_item(w, Xr, A.XW[me], D.p_grp, pcf, vcur,
                         A.Y[me], A.Y2[me], smw, red,
                         (A.tstamp && step == 0 && it == 2 && gb < 4096) ? A.tstamp + 528 + gb * 8 + 4 : nullptr,
                         PF0(j_w), GAT(PH_P5, w));
          ITIME_END(PH_P5, j_w)
        }
        WSTAMP(2);
        loc = block_sum(loc, red);
        pq = bar(PH_SY, true, loc);
      }
      TSTAMP(3);
      if (!(pq > 0.0)) { status = 2; break; }  // lost positive curvature (uniform)
      const double alpha = rho / pq;
      double* const* rc = A.r[rp];
      double* rn = A.r[rp ^ 1][me];
      auto unew = [&](const ItemDesc& iw, int64_t bb, int pos) {
        const BPos q = bget(iw, bb, pos);
        return q.aown * (q.sign * ldcg(rc[lown(q.k)] + q.k) - alpha * (yv(me, own_idx(iw, pos)) - yv(pown(ppatch(bb)), q.part)));
      };
      // P7 (+ partial r^T z)
      {
        // the block's lambda chunk: loads issued before the items, stores after them
        const int64_t kq = k0 + threadIdx.x;
        double lv = 0.0, pv = 0.0, rv = 0.0, yd = 0.0;
        if (kq < k1) {
          lv = A.lam[me][kq];
          pv = ldcg(pcur + kq);
          rv = ldcg(rc[me] + kq);
          yd = yv(pown(lpat_p(kq)), lidx_p(kq)) - yv(pown(lpat_m(kq)), lidx_m(kq));
        }
        double loc = 0.0;
        FOR_ITEMS(PH_SY, w) {
          ITIME_BEGIN
          loc += symv_item(w, Sr, A.PW[me], unew, smw, red, PF0(j_w), GAT(PH_SY, w));
          ITIME_END(PH_SY, j_w)
        }
        if (kq < k1) {
          A.lam[me][kq] = lv + alpha * pv;
          rn[kq] = rv - alpha * yd;
        }
        for (int64_t k = kq + blockDim.x; k < k1; k += blockDim.x) {
          A.lam[me][k] += alpha * ldcg(pcur + k);
          rn[k] = ldcg(rc[me] + k) - alpha * (yv(pown(lpat_p(k)), lidx_p(k)) - yv(pown(lpat_m(k)), lidx_m(k)));
        }
        WSTAMP(3);
        loc = block_sum(loc, red);
        rz = bar(PH_P1, true, loc);
      }
      TSTAMP(4);
      ++it;
      const double rel = sqrt(fmax(rz, 0.0) / rho0);
      if (me == 0 && bl == 0 && threadIdx.x == 0) A.hist[0][hoff + it] = rel;
      rp ^= 1;
      pp ^= 1;
      if (rel <= A.rtol) status = 1;
      else if (it >= A.max_iter || !(rz == rz)) status = 2;
      beta = rz / rho;
      rho = rz;
    }
    if (bl == 0 && threadIdx.x == 0) {
      A.iters[me][A.step0 + step] = it;
      A.st[me]->iter = it;
      A.st[me]->rho0 = rho0;
      A.st[me]->rz = rz;
    }
    if (status == 2) {  // uniform: report and stop the remaining steps
      if (bl == 0 && threadIdx.x == 0) {
        A.st[me]->failed = 1;
        A.st[me]->nan = !(rz == rz);
        A.st[me]->rp = A.step0 + step;  // failing step index
      }
      total_status = 2;
      break;
    }
    hoff += it + 1;
    if (A.warm) {  // this step's solution and d - r (= F lambda) into the ring (own chunk)
      const int64_t so = ((int64_t)(A.step0 + step) % A.warm) * m;
      const double* rf = A.r[rp][me];
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        A.Wr[me][so + k] = A.lam[me][k];
        A.FWr[me][so + k] = ldcg(A.dsave[me] + k) - ldcg(rf + k);
      }
    }
    SSTAMP(6);
    // ---- E1 v = B^T lambda ; w, -Phi^T v (the X_bb form of the F-apply's first half) ----
    FOR_ITEMS(PH_E1, w)
      p1_item(w, Xr,
              [&](const ItemDesc& iw, int64_t bb, int pos) {
                const BPos q = bget(iw, bb, pos);
                return q.sign * ldcg(A.lam[lown(q.k)] + q.k);
              },
              A.XW[me], smw, nullptr, 0, GAT(PH_E1, w));
    bar(PH_PC, false, 0.0);
    SSTAMP(7);
    // ---- E2 p = S_pp^-1 sum N^T (Z_p - XW_p) ----
    COARSE(([&](int64_t i, int o) {
      const int r = MULTI ? o : 0;
      return ldcg(A.Z[r] + i) - ldcg(A.XW[r] + i);
    }));
    bar(-1, false, 0.0);
    SSTAMP(8);
    // ---- E3 a_r = X_rr^T (Z_r - [0; w_b]) - Phi N p, a_p = N p ----
    // insulator coefficients feed no later step (no mass term): recover them only at the last step
    if (step == A.nsteps - 1) {
      FOR_ITEMS(PH_BW, w) bw_item(D, w, Xr, A.Z[me], A.XW[me], pcf, A.a_loc[me], A.G.nloc, smw);
    } else {
      FOR_ITEMS(PH_BWC, w) bw_item(D, w, Xr, A.Z[me], A.XW[me], pcf, A.a_loc[me], A.G.nloc, smw);
    }
    if (A.nd > 0) {  // Dirichlet DOFs of the paper's experiment: a_D(t) = amp e^-t (Pi_h S)_D (mms.cu)
      const double et = A.src_amp * exp(-t);
      for (int64_t q = (int64_t)bl * blockDim.x + threadIdx.x; q < A.nd; q += (int64_t)A.nbr * blockDim.x) {
        const int64_t v = A.dlist[q];
        if (pown((int)(v / A.G.nloc)) == me) A.a_loc[me][v] = et * A.aD0[q];
      }
    }
    bar(-1, false, 0.0);
    SSTAMP(9);
  }
  if (bl == 0 && threadIdx.x == 0) {
    A.st[me]->done = 1;
    if (total_status != 2) A.st[me]->failed = 0;
    A.st[me]->counter[2] = (unsigned int)(hoff - A.hist_off);  // history length written
    A.st[me]->counter[3] = round;                               // barrier rounds after this launch
  }
}

// ---- standalone item kernel (setup precompute of the insulator rhs template), one item
// per block over the given item range.
__global__ void __launch_bounds__(NTHR) k_fw(DevPlan D, const ItemDesc* items, int n, const double* Fv, double* Zv) {
  extern __shared__ __align__(16) double sm[];
  if (blockIdx.x >= n) return;
  fw_item(items[blockIdx.x], D.A, Fv, Zv, sm);
}
}  // namespace tcg
