// pcg.cu — step c (the PCG on lambda) as chain-free GEMV work items in one persistent
// cooperative kernel per implicit-Euler step (four grid barriers per PCG iteration).
//
// Paper: PCG on the interface problem with the Dirichlet preconditioner, the dual
// operator of the two sequential Schur complements; recurrences DESIGN.md R6.
// Setup (chol.cu) leaves X_bb = L_bb^-1, Phi^T = L_pb X_bb (per patch) and the full
// symmetric S_pp^-1 = X_c^T X_c. One PCG iteration is then:
//   P1  p = z + beta p_prev (z = B_D S_bb B_D^T r from P7, on the fly); v_s = B_s^T p;
//       w_s = X_bb v_s, (-g_s) = -Phi^T v_s                           items: patch row blocks
//   PC  Pc = S_pp^-1 G, G = sum_s N_s^T (-g_s)  (= -S_pp^-1 g)        items: coarse row block x column chunk
//   P5  y_s = X_bb^T w_s - Phi_b N_s Pc;  p^T F p = sum_s v_s . y_s   items: patch column blocks
//   P7  alpha = rho / p^T F p; lambda += alpha p; r_new = r - alpha B y;
//       u_s = B_D^T r_new, (S_bb u)_s;  r_new^T z = sum_s u_s . S_bb u_s   items: patch row blocks
// so that every dot product is a sum of per-item partials (no separate jump phase): the
// jump q = B y and z = B_D (S_bb u) are gathered on the fly where they are consumed.
// Partials are summed in one fixed order by every block (bit-identical scalars, deterministic).
#include "common.cuh"
#include "device.h"

namespace tcg {

struct PcgArgs {
  // lambda-space vectors (m)
  double* lam;
  double* r[2];
  double* pk[2];
  // per-patch aug-ordered vectors
  double* XW;    // P1 output: b part w, p part -g
  double* Y;     // P5 output: b part y
  double* PW;    // P7 output: b part S_bb u
  // coarse
  const double* Sinv;  // full symmetric S_pp^-1, Tc x Tc row-major tiles
  double* Ppart;       // Tc x maxch x 64 chunk partials of Pc
  double* Pc;          // materialised coarse solution (standalone kernels)
  int ch;              // tiles per coarse chunk
  int maxch;
  double* partA;       // per-block partials (P5)
  double* partB;       // per-block partials (P7 / prologue)
  double* hist;
  PcgState* st;
  // item lists (sorted by decreasing cost)
  const int2* it_p1;  // (patch, row block of [b;p])
  const int2* it_p5;  // (patch, b column block)
  const int2* it_sy;  // (patch, b row block)
  const int2* it_pc;  // (coarse row block, column chunk)
  int n_p1, n_p5, n_sy, n_pc;
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

// fixed-order block reduction of one value per thread
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

// Coarse solution entry g from the PC chunk partials (fixed order).
__device__ __forceinline__ double pc_get(const PcgArgs& A, int64_t g) {
  const double* p = A.Ppart + ((g >> 6) * A.maxch) * TS + (g & 63);
  double v = 0.0;
  for (int c = 0; c < A.maxch; ++c) v += ldcg(p + (int64_t)c * TS);
  return v;
}

// ---- P1: row GEMV of [X_bb; Phi^T] with v = B_s^T p gathered per b position --------------
// vsrc(b, pos) returns the signed value (B_s^T p)_pos, b = b_off[s] + pos.
template <class Src>
__device__ void p1_item(const DevPlan& D, int s, int I, Src vsrc, double* XW, double* sv) {
  const int Ti = D.Ti[s], Tb = D.Tb[s], nb = D.nb[s];
  const int Jn = (I < Tb) ? I + 1 : Tb;
  const int64_t bo = D.b_off[s];
  for (int e = threadIdx.x; e < Jn * TS; e += blockDim.x) sv[e] = (e < nb) ? vsrc(s, bo + e, e) : 0.0;
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

// ---- PC: Ppart[I][c] = sum_{J in chunk c} Sinv_IJ G_J,  G = sum_csr (src1 - src2) -----------
__device__ void pc_item(const DevPlan& D, const PcgArgs& A, int I, int c, const double* src1, const double* src2,
                        double* sm) {
  const int Tc = D.Tc;
  const int J0 = c * A.ch, J1 = min(Tc, J0 + A.ch);
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
  const double* rowp = A.Sinv + ((int64_t)I * Tc) * TSZ + row0 * TS + 2 * lane;
#pragma unroll 2
  for (int J = J0; J < J1; ++J) {
    const double* t = rowp + (int64_t)J * TSZ;
    const double2 xv = *reinterpret_cast<const double2*>(sm + (J - J0) * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
    for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
  }
  const double sum = warp_reduce8(part);
  if ((lane & 3) == 0) A.Ppart[((int64_t)I * A.maxch + c) * TS + row0 + warp_reduce8_row()] = sum;
  __syncthreads();
}

// ---- P5: column GEMV  y_J = sum_{I>=J} X_IJ^T w_I - sum_{p rows} PhiT_IJ^T (N Pc)_I ---------
// Returns this item's share of p^T F p = v_J . y_J (vsrc gives the lambda values of p).
template <class PcF, class Src>
__device__ double p5_item(const DevPlan& D, int s, int J, const double* W, PcF pc, Src vsrc, double* Y, double* sm,
                          double* red) {
  const int Ti = D.Ti[s], Tb = D.Tb[s], Tp = D.Tp[s], np = D.np[s], nb = D.nb[s];
  const int Tr = Tb + (np > 0 ? Tp : 0);
  double* sw = sm;                    // (Tr - J) * 64
  double* cr = sm + (Tr - J) * TS;    // 8 * 64
  const int* grp = D.p_grp + D.p_off[s];
  const int* bl = D.b_lam + D.b_off[s];
  const double* bs = D.b_sign + D.b_off[s];
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
  cr[warp * TS + 2 * lane] = c0;
  cr[warp * TS + 2 * lane + 1] = c1;
  __syncthreads();
  double contrib = 0.0;
  if (threadIdx.x < TS) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < NTHR / 32; ++w) acc += cr[w * TS + threadIdx.x];
    Y[vo + (int64_t)J * TS + threadIdx.x] = acc;
    const int pos = J * TS + threadIdx.x;
    if (pos < nb) contrib = bs[pos] * vsrc(bl[pos]) * acc;
  }
  return block_sum(contrib, red);
}

// ---- P7: symmetric S_bb apply, one row block I of one patch (packed-lower storage: the
// row's lower tiles as row GEMVs, the tiles below the diagonal as transposed GEMVs).
// u = B_D^T r (weighted gather of usrc). Returns this item's share of u^T S_bb u.
// usrc(s, b, pos) returns (B_D^(s)T r)_pos, b = b_off[s] + pos.
template <class Src>
__device__ double symv_item(const DevPlan& D, const PcgArgs& A, int s, int I, Src usrc, double* sm, double* red) {
  const int Ti = D.Ti[s], Tb = D.Tb[s], nb = D.nb[s];
  double* u = sm;               // Tb*64
  double* cr = u + Tb * TS;     // 8 * 64
  const int64_t bo = D.b_off[s];
  for (int i = threadIdx.x; i < Tb * TS; i += blockDim.x) u[i] = (i < nb) ? usrc(s, bo + i, i) : 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const double* S = D.Sbb + D.sbb_off[s];
  double part[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) part[q] = 0.0;
#pragma unroll 2
  for (int J = 0; J <= I; ++J) {  // row part: S_IJ u_J
    const double* t = S + tri_off(I, J) + row0 * TS + 2 * lane;
    const double2 xv = *reinterpret_cast<const double2*>(u + J * TS + 2 * lane);
    double2 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = ldg2(t + q * TS);
#pragma unroll
    for (int q = 0; q < 8; ++q) part[q] += a[q].x * xv.x + a[q].y * xv.y;
  }
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
    cr[8 * TS + row] = acc;  // staging slot after the 8 warp rows
  }
  __syncthreads();
  double contrib = 0.0;
  if (threadIdx.x < TS) {
    const double v = cr[8 * TS + threadIdx.x];
    A.PW[D.vec_off[s] + (int64_t)(Ti + I) * TS + threadIdx.x] = v;
    contrib = u[I * TS + threadIdx.x] * v;
  }
  return block_sum(contrib, red);
}

// Sum of per-block partials in one fixed order (lane-strided + xor butterfly in warp 0),
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

// Grid barrier for the cooperative (co-resident) launch: one monotonically increasing
// arrival counter (zeroed by the host before the launch); thread 0 of each block arrives
// with a release fence and polls with acquire loads until all blocks of this round arrived.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
    __threadfence();
  }
  __syncthreads();
}

#define TSTAMP(slot) \
  if (A.tstamp && b == 0 && threadIdx.x == 0 && it < 64) A.tstamp[it * 8 + (slot)] = gtimer()

// =======================================================================================
// Persistent cooperative PCG (one launch per implicit-Euler step). Input: r[0] = d,
// lam = 0. Output: lam, history, state. All blocks run the same number of barriers.
// =======================================================================================
__global__ void __launch_bounds__(NTHR, 2) k_pcg(DevPlan D, PcgArgs A) {
  extern __shared__ double sm[];
  __shared__ double red[NTHR];
  const int NB = gridDim.x, b = blockIdx.x;
  const int64_t m = D.m;
  const int64_t chunk = (m + NB - 1) / NB;
  const int64_t k0 = min(m, (int64_t)b * chunk), k1 = min(m, k0 + chunk);
  unsigned int* bar = &A.st->counter[1];
  unsigned int bar_target = 0;
  int it = 0;
  const double* r0 = A.r[0];
  // own/partner form of the jumps (per b position: a_own, a_part, partner index, sign, lambda)
  auto own_idx = [&](int s, int pos) { return D.vec_off[s] + (int64_t)D.Ti[s] * TS + pos; };

  // ---- prologue: u = B_D^T r0, PW = S_bb u, rho0 = r0^T z0 = sum u.S u ----
  {
    double loc = 0.0;
    for (int i = b; i < A.n_sy; i += NB)
      loc += symv_item(D, A, A.it_sy[i].x, A.it_sy[i].y,
                       [&](int, int64_t bb, int) { return D.b_aown[bb] * D.b_sign[bb] * ldcg(r0 + D.b_lam[bb]); },
                       sm, red);
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) A.pk[0][k] = 0.0;
    if (threadIdx.x == 0) A.partB[b] = loc;
  }
  grid_barrier(bar, bar_target);
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
  double rz = rho0;
  for (;;) {
    TSTAMP(0);
    const double* pprev = A.pk[pp];
    double* pcur = A.pk[pp ^ 1];
    // p_k = z_k + beta p_prev,k with z = B_D (S_bb u) from P7; signed value at a b position:
    // sign*z_k = a_own PW[own] + a_part PW[partner]
    auto vnew = [&](int s, int64_t bb, int pos) {
      return D.b_aown[bb] * ldcg(A.PW + own_idx(s, pos)) + D.b_apart[bb] * ldcg(A.PW + D.b_part[bb]) +
             D.b_sign[bb] * beta * ldcg(pprev + D.b_lam[bb]);
    };
    // P1: v = B^T p (on the fly); w = X_bb v, -g = -Phi^T v; owners materialise p
    for (int i = b; i < A.n_p1; i += NB) p1_item(D, A.it_p1[i].x, A.it_p1[i].y, vnew, A.XW, sm);
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x)
      pcur[k] = D.wplus[k] * ldcg(A.PW + D.lam_idx_p[k]) - D.wminus[k] * ldcg(A.PW + D.lam_idx_m[k]) +
                beta * ldcg(pprev + k);
    grid_barrier(bar, bar_target);
    TSTAMP(1);
    // PC: Pc = S_pp^-1 G (chunk partials)
    for (int i = b; i < A.n_pc; i += NB) pc_item(D, A, A.it_pc[i].x, A.it_pc[i].y, A.XW, nullptr, sm);
    grid_barrier(bar, bar_target);
    TSTAMP(2);
    // P5: y = X_bb^T w - Phi_b N Pc ; partial p^T F p
    {
      double loc = 0.0;
      for (int i = b; i < A.n_p5; i += NB)
        loc += p5_item(D, A.it_p5[i].x, A.it_p5[i].y, A.XW, [&](int64_t g) { return pc_get(A, g); },
                       [&](int k) { return ldcg(pcur + k); }, A.Y, sm, red);
      if (threadIdx.x == 0) A.partA[b] = loc;
    }
    grid_barrier(bar, bar_target);
    TSTAMP(3);
    const double pq = sum_partials(A.partA, NB, red);
    if (!(pq > 0.0)) { status = 2; break; }  // lost positive curvature (uniform)
    const double alpha = rho / pq;
    const double* rc = A.r[rp];
    double* rn = A.r[rp ^ 1];
    // u_pos = a_own (sign r_k - alpha sign q_k), sign q_k = Y[own] - Y[partner]
    auto unew = [&](int s, int64_t bb, int pos) {
      return D.b_aown[bb] * (D.b_sign[bb] * ldcg(rc + D.b_lam[bb]) -
                             alpha * (ldcg(A.Y + own_idx(s, pos)) - ldcg(A.Y + D.b_part[bb])));
    };
    // P7: lambda, r updates (owners); S_bb apply of u = B_D^T r_new; partial r_new^T z
    {
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        A.lam[k] += alpha * ldcg(pcur + k);
        rn[k] = ldcg(rc + k) - alpha * (ldcg(A.Y + D.lam_idx_p[k]) - ldcg(A.Y + D.lam_idx_m[k]));
      }
      double loc = 0.0;
      for (int i = b; i < A.n_sy; i += NB) loc += symv_item(D, A, A.it_sy[i].x, A.it_sy[i].y, unew, sm, red);
      if (threadIdx.x == 0) A.partB[b] = loc;
    }
    grid_barrier(bar, bar_target);
    TSTAMP(4);
    rz = sum_partials(A.partB, NB, red);
    ++it;
    const double rel = sqrt(fmax(rz, 0.0) / rho0);
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
  p1_item(D, items[blockIdx.x].x, items[blockIdx.x].y,
          [&](int, int64_t bb, int) { return D.b_sign[bb] * lam[D.b_lam[bb]]; }, XW, sm);
}
__global__ void __launch_bounds__(NTHR) k_pc(DevPlan D, PcgArgs A, const double* src1, const double* src2) {
  extern __shared__ double sm[];
  if (blockIdx.x >= A.n_pc) return;
  pc_item(D, A, A.it_pc[blockIdx.x].x, A.it_pc[blockIdx.x].y, src1, src2, sm);
}
// materialise Pc from the chunk partials
__global__ void k_pc_sum(DevPlan D, PcgArgs A) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < D.nc; g += (int64_t)gridDim.x * blockDim.x)
    A.Pc[g] = pc_get(A, g);
}
__global__ void __launch_bounds__(NTHR) k_p5(DevPlan D, PcgArgs A, const double* W) {
  extern __shared__ double sm[];
  __shared__ double red[NTHR];
  if (blockIdx.x >= A.n_p5) return;
  p5_item(D, A.it_p5[blockIdx.x].x, A.it_p5[blockIdx.x].y, W, [&](int64_t g) { return ldcg(A.Pc + g); },
          [&](int) { return 0.0; }, A.Y, sm, red);
}
// d = B y -> r[0], lam = 0
__global__ void k_dual_rhs(DevPlan D, const double* Y, double* r0, double* lam) {
  const int64_t m = D.m;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    r0[k] = ldcg(Y + D.lam_idx_p[k]) - ldcg(Y + D.lam_idx_m[k]);
    lam[k] = 0.0;
  }
}

}  // namespace tcg
