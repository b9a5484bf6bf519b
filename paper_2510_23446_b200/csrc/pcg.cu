// pcg.cu — step c (the PCG on lambda) as chain-free GEMV work items and one persistent
// cooperative kernel per implicit-Euler step.
//
// Paper: PCG on the interface problem with the Dirichlet preconditioner, the dual
// operator of the two sequential Schur complements; recurrences DESIGN.md R6.
// With the inverse factors built at setup (chol.cu: X_bb = L_bb^-1, Phi^T = L_pb X_bb,
// X_c = L_c^-1) one F-apply is four GEMV phases and a jump:
//   P1  w_s = X_bb v_s,  (-g_s) = -Phi^T v_s          v_s = B_s^T p   (items: patch row blocks)
//   P3  Yc = X_c G,  G = sum_s N_s^T (-g_s)                           (items: coarse row block x column chunk)
//   P4  Pc = X_c^T Yc  (= -S_pp^-1 g)                                 (items: coarse column block x row chunk)
//   P5  y_s = X_bb^T w_s - Phi_b N_s Pc                               (items: patch column blocks)
//   P6  q = B y, p.q                                                  (items: lambda chunks)
// then  P7  S_bb (B_D^T r_new) (packed-lower SYMV, items: patch row blocks; the transposed
//           contributions go to per-tile partials), lambda/r updates
//       P8  z = B_D (S_bb ...), r.z, convergence, beta.
// Every phase is a grid-wide set of items separated by cooperative grid barriers; partial
// results are combined in a fixed order and the PCG scalars are reduced identically by
// every block, so the run is deterministic.
#include <cooperative_groups.h>

#include "common.cuh"
#include "device.h"

namespace cg = cooperative_groups;

namespace tcg {

struct PcgArgs {
  // lambda-space vectors (m)
  double* lam;
  double* r[2];
  double* pk[2];
  double* z;
  double* q;
  // per-patch aug-ordered vectors
  double* XW;    // P1 output: b part w, p part -g
  double* Y;     // P5 output: b part y
  double* PW;    // SYMV row output: b part
  double* PWc;   // SYMV transposed partials: per patch Tb x Tb x 64
  const int64_t* pwc_off;
  // coarse (chunked partials)
  double* Ypart;  // Tc x maxch x 64
  double* Ppart;  // Tc x maxch x 64
  double* Pc;     // materialised coarse solution (standalone kernels)
  int ch;         // tiles per coarse chunk
  int maxch;
  double* partA;
  double* partB;
  double* hist;
  PcgState* st;
  // item lists (sorted by decreasing cost)
  const int2* it_p1;  // (patch, row block)
  const int2* it_p5;  // (patch, column block)
  const int2* it_sy;  // (patch, row block)
  const int2* it_p3;  // (coarse row block, column chunk)
  const int2* it_p4;  // (coarse column block, row chunk)
  int n_p1, n_p5, n_sy, n_p3, n_p4;
  unsigned long long* tstamp;  // optional phase timestamps (block 0), 8 per iteration
  double rtol;
  int max_iter;
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ const double* ls_tile(const DevPlan& D, int s, int Tb, int I, int J) {
  const double* L = D.LS + D.ls_off[s];
  return I < Tb ? L + tri_off(I, J) : L + (tri_tiles(Tb) + (int64_t)(I - Tb) * Tb + J) * TSZ;
}

// Coarse solution entry g from the P4 chunk partials (fixed order).
__device__ __forceinline__ double pc_get(const DevPlan& D, const PcgArgs& A, int64_t g) {
  const int J = (int)(g >> 6);
  const int nch = (D.Tc - J + A.ch - 1) / A.ch;
  const double* p = A.Ppart + ((int64_t)J * A.maxch) * TS + (g & 63);
  double v = 0.0;
  for (int c = 0; c < nch; ++c) v += ldcg(p + (int64_t)c * TS);
  return v;
}

// ---- P1: row GEMV of [X_bb; Phi^T] with v gathered through the signed b-map ---------------
template <class Src>
__device__ void p1_item(const DevPlan& D, int s, int I, Src src, double* XW, double* sv) {
  const int Ti = D.Ti[s], Tb = D.Tb[s], nb = D.nb[s];
  const int Jn = (I < Tb) ? I + 1 : Tb;
  const int* bl = D.b_lam + D.b_off[s];
  const double* bs = D.b_sign + D.b_off[s];
  for (int e = threadIdx.x; e < Jn * TS; e += blockDim.x) sv[e] = (e < nb) ? bs[e] * src(bl[e]) : 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  double part[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) part[r] = 0.0;
#pragma unroll 2
  for (int J = 0; J < Jn; ++J) {
    const double* t = ls_tile(D, s, Tb, I, J) + row0 * TS + 2 * lane;
    const double2 xv = *reinterpret_cast<const double2*>(sv + J * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
  }
  const double sum = warp_reduce8(part);
  if ((lane & 3) == 0) XW[D.vec_off[s] + (int64_t)(Ti + I) * TS + row0 + warp_reduce8_row()] = (I < Tb) ? sum : -sum;
  __syncthreads();
}

// ---- P5: column GEMV  y_J = sum_{I>=J} X_IJ^T w_I - sum_{p rows} PhiT_IJ^T (N Pc)_I -----------
template <class PcF>
__device__ void p5_item(const DevPlan& D, int s, int J, const double* W, PcF pc, double* Y, double* sm) {
  const int Ti = D.Ti[s], Tb = D.Tb[s], Tp = D.Tp[s], np = D.np[s];
  const int Tr = Tb + (np > 0 ? Tp : 0);
  double* sw = sm;                   // (Tr - J) * 64
  double* red = sm + (Tr - J) * TS;  // 8 * 64
  const int* grp = D.p_grp + D.p_off[s];
  const int64_t vo = D.vec_off[s] + (int64_t)Ti * TS;
  for (int e = threadIdx.x; e < (Tr - J) * TS; e += blockDim.x) {
    const int i = J * TS + e;  // row index in [b; p] numbering
    double val;
    if (i < Tb * TS) val = ldcg(W + vo + i);
    else {
      const int t = i - Tb * TS;
      val = (t < np) ? -pc(grp[t]) : 0.0;
    }
    sw[e] = val;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  double c0 = 0.0, c1 = 0.0;
#pragma unroll 2
  for (int I = J; I < Tr; ++I) {
    const double* t = ls_tile(D, s, Tb, I, J) + row0 * TS + 2 * lane;
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double xr = sw[(I - J) * TS + row0 + r];
      c0 += a[r].x * xr;
      c1 += a[r].y * xr;
    }
  }
  red[warp * TS + 2 * lane] = c0;
  red[warp * TS + 2 * lane + 1] = c1;
  __syncthreads();
  if (threadIdx.x < TS) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) acc += red[w * TS + threadIdx.x];
    Y[vo + (int64_t)J * TS + threadIdx.x] = acc;
  }
  __syncthreads();
}

// ---- P3: Ypart[I][c] = sum_{J in chunk c, J<=I} Xc_IJ G_J,  G = sum_csr (src1 - src2) --------
__device__ void p3_item(const DevPlan& D, const PcgArgs& A, const double* CX, int I, int c, const double* src1,
                        const double* src2, double* sm) {
  const int J0 = c * A.ch, J1 = min(I + 1, J0 + A.ch);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  for (int e = threadIdx.x; e < (J1 - J0) * TS; e += blockDim.x) {
    const int64_t g = (int64_t)J0 * TS + e;
    double val = 0.0;
    if (g < D.nc) {
      for (int k = D.coarse_ptr[g]; k < D.coarse_ptr[g + 1]; ++k) {
        const int64_t idx = D.coarse_idx[k];
        val += src2 ? (ldcg(src1 + idx) - ldcg(src2 + idx)) : ldcg(src1 + idx);
      }
    }
    sm[e] = val;
  }
  __syncthreads();
  double part[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) part[r] = 0.0;
#pragma unroll 2
  for (int J = J0; J < J1; ++J) {
    const double* t = CX + tri_off(I, J) + row0 * TS + 2 * lane;
    const double2 xv = *reinterpret_cast<const double2*>(sm + (J - J0) * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
  }
  const double sum = warp_reduce8(part);
  if ((lane & 3) == 0) A.Ypart[((int64_t)I * A.maxch + c) * TS + row0 + warp_reduce8_row()] = sum;
  __syncthreads();
}

// ---- P4: Ppart[J][c] = sum_{I in chunk c, I>=J} Xc_IJ^T Yc_I,  Yc_I = sum_c' Ypart[I][c'] -----
__device__ void p4_item(const DevPlan& D, const PcgArgs& A, const double* CX, int J, int c, double* sm) {
  const int Tc = D.Tc;
  const int I0 = J + c * A.ch, I1 = min(Tc, I0 + A.ch);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  double* red = sm + A.ch * TS;
  for (int e = threadIdx.x; e < (I1 - I0) * TS; e += blockDim.x) {
    const int I = I0 + e / TS;
    const int nch = (I + 1 + A.ch - 1) / A.ch;
    const double* p = A.Ypart + ((int64_t)I * A.maxch) * TS + (e & 63);
    double v = 0.0;
    for (int cc = 0; cc < nch; ++cc) v += ldcg(p + (int64_t)cc * TS);
    sm[e] = v;
  }
  __syncthreads();
  double c0 = 0.0, c1 = 0.0;
#pragma unroll 2
  for (int I = I0; I < I1; ++I) {
    const double* t = CX + tri_off(I, J) + row0 * TS + 2 * lane;
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double xr = sm[(I - I0) * TS + row0 + r];
      c0 += a[r].x * xr;
      c1 += a[r].y * xr;
    }
  }
  red[warp * TS + 2 * lane] = c0;
  red[warp * TS + 2 * lane + 1] = c1;
  __syncthreads();
  if (threadIdx.x < TS) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) acc += red[w * TS + threadIdx.x];
    A.Ppart[((int64_t)J * A.maxch + c) * TS + threadIdx.x] = acc;
  }
  __syncthreads();
}

// ---- P7: packed-lower S_bb SYMV, one row block I of one patch ------------------------------
// row part  PW_I = sum_{J<=I} S_IJ v_J ;  transposed part PWc[I][J] = S_IJ^T v_I (J < I)
template <class Src>
__device__ void symv_item(const DevPlan& D, const PcgArgs& A, int s, int I, Src src, double* sm) {
  const int Ti = D.Ti[s], Tb = D.Tb[s], nb = D.nb[s];
  double* v = sm;                   // (I+1)*64
  double* colp = v + (I + 1) * TS;  // 8 warps x I x 64
  const int* bl = D.b_lam + D.b_off[s];
  const double* bs = D.b_sign + D.b_off[s];
  for (int i = threadIdx.x; i < (I + 1) * TS; i += blockDim.x) {
    double val = 0.0;
    if (i < nb) {
      const int k = bl[i];
      const double sg = bs[i];
      val = sg * (sg > 0 ? D.wplus[k] : D.wminus[k]) * src(k);
    }
    v[i] = val;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const double* S = D.Sbb + D.sbb_off[s];
  double part[8], xr[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    part[q] = 0.0;
    xr[q] = v[I * TS + row0 + q];
  }
#pragma unroll 2
  for (int J = 0; J <= I; ++J) {
    const double* t = S + tri_off(I, J) + row0 * TS + 2 * lane;
    const double2 xv = *reinterpret_cast<const double2*>(v + J * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = ldg2(t + q * TS);
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      part[q] += a[q].x * xv.x + a[q].y * xv.y;
      c0 += a[q].x * xr[q];
      c1 += a[q].y * xr[q];
    }
    if (J < I) {
      colp[(warp * I + J) * TS + 2 * lane] = c0;
      colp[(warp * I + J) * TS + 2 * lane + 1] = c1;
    }
  }
  const double sum = warp_reduce8(part);
  if ((lane & 3) == 0) A.PW[D.vec_off[s] + (int64_t)(Ti + I) * TS + row0 + warp_reduce8_row()] = sum;
  __syncthreads();
  double* pc = A.PWc + A.pwc_off[s] + (int64_t)I * Tb * TS;
  for (int e = threadIdx.x; e < I * TS; e += blockDim.x) {
    const int J = e / TS, cc = e % TS;
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) acc += colp[(w * I + J) * TS + cc];
    pc[e] = acc;
  }
  __syncthreads();
}

// value of (S_bb v) at b position pos of patch s: row part + transposed partials of rows below
__device__ __forceinline__ double symv_value(const DevPlan& D, const PcgArgs& A, int s, int pos, int64_t idx) {
  const int Tb = D.Tb[s];
  const int J = pos >> 6, c = pos & 63;
  double v = ldcg(A.PW + idx);
  const double* p = A.PWc + A.pwc_off[s] + (int64_t)J * TS + c;
  for (int I = J + 1; I < Tb; ++I) v += ldcg(p + (int64_t)I * Tb * TS);
  return v;
}

// ---- jumps with a fused fixed-order block reduction ------------------------------------------
__device__ __forceinline__ double block_sum(double local, double* red) {
  red[threadIdx.x] = local;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// q_k = Y[+] - Y[-]; returns the block's partial of sum_k dotv(k) q_k
template <class Dot>
__device__ double jump_q(const DevPlan& D, const double* Y, double* out, int64_t k0, int64_t k1, Dot dotv, double* red) {
  double local = 0.0;
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    const double val = ldcg(Y + D.lam_idx_p[k]) - ldcg(Y + D.lam_idx_m[k]);
    out[k] = val;
    local += val * dotv(k);
  }
  return block_sum(local, red);
}

// z_k = w+ (S v)[+] - w- (S v)[-]; returns the block's partial of sum_k dotv(k) z_k
template <class Dot>
__device__ double jump_z(const DevPlan& D, const PcgArgs& A, int64_t k0, int64_t k1, Dot dotv, double* red) {
  double local = 0.0;
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    const double yp = symv_value(D, A, D.lam_patch_p[k], D.lam_pos_p[k], D.lam_idx_p[k]);
    const double ym = symv_value(D, A, D.lam_patch_m[k], D.lam_pos_m[k], D.lam_idx_m[k]);
    const double val = D.wplus[k] * yp - D.wminus[k] * ym;
    A.z[k] = val;
    local += val * dotv(k);
  }
  return block_sum(local, red);
}

// Sum of the per-block partials in one fixed order (lane-strided + xor butterfly in warp 0),
// broadcast through shared memory: bit-identical in every block.
__device__ __forceinline__ double sum_partials(const double* part, int n, double* bcast) {
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int b = threadIdx.x; b < n; b += 32) t += ldcg(part + b);
    t = warp_sum(t);
    if (threadIdx.x == 0) *bcast = t;
  }
  __syncthreads();
  const double r = *bcast;
  __syncthreads();
  return r;
}

#define TSTAMP(slot) \
  if (A.tstamp && b == 0 && threadIdx.x == 0 && it < 64) A.tstamp[it * 8 + (slot)] = gtimer()

// =======================================================================================
// Persistent cooperative PCG (one launch per implicit-Euler step). Input: r[0] = d,
// lam = 0. Output: lam, history, state. All blocks run the same number of grid barriers.
// =======================================================================================
__global__ void __launch_bounds__(NTHR) k_pcg(DevPlan D, PcgArgs A, const double* __restrict__ CX) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ double red[NTHR];
  const int NB = gridDim.x, b = blockIdx.x;
  const int64_t m = D.m;
  const int64_t chunk = (m + NB - 1) / NB;
  const int64_t k0 = min(m, (int64_t)b * chunk), k1 = min(m, k0 + chunk);
  double* r0 = A.r[0];
  int it = 0;

  // ---- prologue: z = M^-1 r0, rho0 = r0.z ----
  for (int i = b; i < A.n_sy; i += NB)
    symv_item(D, A, A.it_sy[i].x, A.it_sy[i].y, [&](int k) { return ldcg(r0 + k); }, sm);
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    A.pk[0][k] = 0.0;
    A.pk[1][k] = 0.0;
  }
  __threadfence();
  grid.sync();
  {
    const double loc = jump_z(D, A, k0, k1, [&](int64_t k) { return ldcg(r0 + k); }, red);
    if (threadIdx.x == 0) A.partB[b] = loc;
  }
  __threadfence();
  grid.sync();
  const double rho0 = sum_partials(A.partB, NB, red);
  if (b == 0 && threadIdx.x == 0) {
    A.hist[0] = 1.0;
    A.st->rho0 = rho0;
    A.st->rho = rho0;
    A.st->iter = 0;
  }
  if (!(rho0 > 0.0) || m == 0) {
    if (b == 0 && threadIdx.x == 0) {
      A.st->done = 1;
      if (!(rho0 >= 0.0)) { A.st->failed = 1; A.st->nan = 1; }
    }
    return;  // uniform across blocks
  }
  double rho = rho0, beta = 0.0;
  int rp = 0, pp = 0;
  int status = 0;  // 0 running, 1 converged, 2 failed
  double rel = 1.0, rz = rho0;
  for (;;) {
    TSTAMP(0);
    const double* z = A.z;
    const double* pprev = A.pk[pp];
    double* pcur = A.pk[pp ^ 1];
    // P1: v = B^T pcur, pcur = z + beta pprev (on the fly); owners materialise pcur
    for (int i = b; i < A.n_p1; i += NB)
      p1_item(D, A.it_p1[i].x, A.it_p1[i].y, [&](int k) { return ldcg(z + k) + beta * ldcg(pprev + k); }, A.XW, sm);
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) pcur[k] = ldcg(z + k) + beta * ldcg(pprev + k);
    __threadfence();
    grid.sync();
    TSTAMP(1);
    // P3 coarse lower (chunk partials)
    for (int i = b; i < A.n_p3; i += NB) p3_item(D, A, CX, A.it_p3[i].x, A.it_p3[i].y, A.XW, nullptr, sm);
    __threadfence();
    grid.sync();
    TSTAMP(2);
    // P4 coarse upper (chunk partials)
    for (int i = b; i < A.n_p4; i += NB) p4_item(D, A, CX, A.it_p4[i].x, A.it_p4[i].y, sm);
    __threadfence();
    grid.sync();
    TSTAMP(3);
    // P5 y
    for (int i = b; i < A.n_p5; i += NB)
      p5_item(D, A.it_p5[i].x, A.it_p5[i].y, A.XW, [&](int64_t g) { return pc_get(D, A, g); }, A.Y, sm);
    __threadfence();
    grid.sync();
    TSTAMP(4);
    // P6 q = B y, pcur.q
    {
      const double loc = jump_q(D, A.Y, A.q, k0, k1, [&](int64_t k) { return ldcg(pcur + k); }, red);
      if (threadIdx.x == 0) A.partA[b] = loc;
    }
    __threadfence();
    grid.sync();
    TSTAMP(5);
    const double pq = sum_partials(A.partA, NB, red);
    if (!(pq > 0.0)) { status = 2; break; }  // lost positive curvature (uniform)
    const double alpha = rho / pq;
    const double* rc = A.r[rp];
    double* rn = A.r[rp ^ 1];
    // P7: updates + SYMV with r_new on the fly
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      A.lam[k] += alpha * ldcg(pcur + k);
      rn[k] = ldcg(rc + k) - alpha * ldcg(A.q + k);
    }
    for (int i = b; i < A.n_sy; i += NB)
      symv_item(D, A, A.it_sy[i].x, A.it_sy[i].y, [&](int k) { return ldcg(rc + k) - alpha * ldcg(A.q + k); }, sm);
    __threadfence();
    grid.sync();
    TSTAMP(6);
    // P8 z = B_D (S_bb ...), r_new.z
    {
      const double loc = jump_z(D, A, k0, k1, [&](int64_t k) { return ldcg(rn + k); }, red);
      if (threadIdx.x == 0) A.partB[b] = loc;
    }
    __threadfence();
    grid.sync();
    TSTAMP(7);
    rz = sum_partials(A.partB, NB, red);
    ++it;
    rel = sqrt(fmax(rz, 0.0) / rho0);
    if (b == 0 && threadIdx.x == 0) A.hist[it] = rel;
    rp ^= 1;
    pp ^= 1;
    if (rel <= A.rtol) { status = 1; break; }
    if (it >= A.max_iter || !(rz == rz)) { status = 2; break; }
    beta = rz / rho;
    rho = rz;
  }
  if (b == 0 && threadIdx.x == 0) {
    A.st->iter = it;
    A.st->rz = rz;
    A.st->done = 1;
    A.st->failed = (status == 2);
    A.st->nan = (status == 2 && !(rz == rz));
    A.st->rp = rp;
  }
}

// ---- standalone item kernels (rhs stage, recovery, F-apply benchmark): one item per block ----
__global__ void __launch_bounds__(NTHR) k_p1_lam(DevPlan D, const int2* items, int n, const double* __restrict__ lam,
                                                 double* XW) {
  extern __shared__ double sm[];
  if (blockIdx.x >= n) return;
  p1_item(D, items[blockIdx.x].x, items[blockIdx.x].y, [&](int k) { return lam[k]; }, XW, sm);
}
__global__ void __launch_bounds__(NTHR) k_p3(DevPlan D, PcgArgs A, const double* __restrict__ CX, const double* src1,
                                             const double* src2) {
  extern __shared__ double sm[];
  if (blockIdx.x >= A.n_p3) return;
  p3_item(D, A, CX, A.it_p3[blockIdx.x].x, A.it_p3[blockIdx.x].y, src1, src2, sm);
}
__global__ void __launch_bounds__(NTHR) k_p4(DevPlan D, PcgArgs A, const double* __restrict__ CX) {
  extern __shared__ double sm[];
  if (blockIdx.x >= A.n_p4) return;
  p4_item(D, A, CX, A.it_p4[blockIdx.x].x, A.it_p4[blockIdx.x].y, sm);
}
// materialise Pc from the P4 partials
__global__ void k_pc_sum(DevPlan D, PcgArgs A) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < D.nc; g += (int64_t)gridDim.x * blockDim.x)
    A.Pc[g] = pc_get(D, A, g);
}
__global__ void __launch_bounds__(NTHR) k_p5(DevPlan D, PcgArgs A, const double* W) {
  extern __shared__ double sm[];
  if (blockIdx.x >= A.n_p5) return;
  p5_item(D, A.it_p5[blockIdx.x].x, A.it_p5[blockIdx.x].y, W, [&](int64_t g) { return ldcg(A.Pc + g); }, A.Y, sm);
}
// d = B y -> r[0], lam = 0
__global__ void k_dual_rhs(DevPlan D, const double* Y, double* r0, double* lam) {
  __shared__ double red[256];
  const int64_t m = D.m;
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = min(m, (int64_t)blockIdx.x * chunk), k1 = min(m, k0 + chunk);
  jump_q(D, Y, r0, k0, k1, [&](int64_t) { return 0.0; }, red);
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) lam[k] = 0.0;
}

}  // namespace tcg
