// solve.cu — step c of the hot path: per implicit-Euler step, the rhs, PCG on the
// multipliers lambda (F-apply, Dirichlet preconditioner, primal coarse solve) and the
// recovery, as batched per-patch kernels that stream the factors from HBM.
//
// Paper: eq. (euler), the 3x3 block system after the e/p/r split,
// "two sequential Schur complements", PCG with the Dirichlet preconditioner
// (P:L170). Algebra, with L the augmented factor of
// [W_rr W_rp; W_pr *] over the r columns (chol.cu):
//   F lam:  v = B^T lam; w_b = L_bb^-1 v; g_s = L_pb w_b (= Phi_b^T v);
//           p = -S_pp^-1 sum N^T g_s; y_b = L_bb^-T (w_b - L_pb^T N p); (F lam)_k = y+ - y-
//   M^-1 r: sum_s B_D^(s) S_bb^(s) B_D^(s)T r   (packed S_bb SYMV)
// Triangular solves use 64x64 diagonal-block inverses so that every tile step is a
// coalesced GEMV (row-major tiles, double2 loads, warp-shuffle reductions).
#include "common.cuh"
#include "device.h"

namespace tcg {

struct FullView {
  const double* A;
  const double* Dinv;
  int subst;  // 1: solve diagonal blocks by substitution with L_II (else multiply by L_II^-1)
  __device__ __forceinline__ const double* tile(int I, int J) const { return A + tri_off(I, J); }
  __device__ __forceinline__ const double* dinv(int I) const { return Dinv + (int64_t)I * TSZ; }
  __device__ __forceinline__ const double* diag(int I) const { return A + tri_off(I, I); }
};

struct LSView {
  const double* L;
  int Tb;
  int subst;  // diagonal tiles hold L_II (subst) or L_II^-1
  __device__ __forceinline__ const double* diag(int I) const { return L + tri_off(I, I); }
  __device__ __forceinline__ const double* tile(int I, int J) const {
    return I < Tb ? L + tri_off(I, J) : L + (tri_tiles(Tb) + (int64_t)(I - Tb) * Tb + J) * TSZ;
  }
  __device__ __forceinline__ const double* dinv(int I) const { return L + tri_off(I, I); }
};

// Diagonal-block substitution (one warp) with the 64x64 factor tile staged in smem.
__device__ void diag_subst(const double* Lg, double* acc, double* dt, bool transpose) {
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) dt[(e / TS) * 65 + (e % TS)] = Lg[e];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double a0 = acc[lane], a1 = acc[lane + 32];
    if (!transpose) {
      for (int j = 0; j < TS; ++j) {
        double aj = __shfl_sync(0xffffffffu, j < 32 ? a0 : a1, j & 31);
        double xj = aj / dt[j * 65 + j];
        if (lane == (j & 31)) { if (j < 32) a0 = xj; else a1 = xj; }
        if (lane > j) a0 -= dt[lane * 65 + j] * xj;
        if (lane + 32 > j) a1 -= dt[(lane + 32) * 65 + j] * xj;
      }
    } else {
      for (int j = TS - 1; j >= 0; --j) {
        double aj = __shfl_sync(0xffffffffu, j < 32 ? a0 : a1, j & 31);
        double xj = aj / dt[j * 65 + j];
        if (lane == (j & 31)) { if (j < 32) a0 = xj; else a1 = xj; }
        if (lane < j) a0 -= dt[j * 65 + lane] * xj;
        if (lane + 32 < j) a1 -= dt[j * 65 + lane + 32] * xj;
      }
    }
    acc[lane] = a0;
    acc[lane + 32] = a1;
  }
  __syncthreads();
}

// Forward substitution over tile rows 0..Trows-1; rows < Tsolve are solved with the
// diagonal inverse, rows >= Tsolve only receive  x_I <- x_I - sum_J L_IJ x_J.
template <class V>
__device__ void tri_fwd(const V& v, double* x, int Trows, int Tsolve, double* acc, double* dt = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = warp * 8;
  for (int I = 0; I < Trows; ++I) {
    double part[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) part[r] = 0.0;
    const int Jmax = min(I, Tsolve);
    for (int J = 0; J < Jmax; ++J) {
      const double* t = v.tile(I, J) + row0 * TS + 2 * lane;
      const double2 xv = *reinterpret_cast<const double2*>(x + J * TS + 2 * lane);
      double2 a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
      for (int r = 0; r < 8; ++r) part[r] += a[r].x * xv.x + a[r].y * xv.y;
    }
    double s = warp_reduce8(part);
    if ((lane & 3) == 0) {
      const int row = row0 + warp_reduce8_row();
      acc[row] = x[I * TS + row] - s;
    }
    __syncthreads();
    if (I < Tsolve && v.subst) {
      diag_subst(v.diag(I), acc, dt, false);
      if (threadIdx.x < TS) x[I * TS + threadIdx.x] = acc[threadIdx.x];
    } else if (I < Tsolve) {
      const double* t = v.dinv(I) + row0 * TS + 2 * lane;
      const double2 av = *reinterpret_cast<const double2*>(acc + 2 * lane);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        double2 a = ldg2(t + r * TS);
        part[r] = a.x * av.x + a.y * av.y;
      }
      s = warp_reduce8(part);
      if ((lane & 3) == 0) x[I * TS + row0 + warp_reduce8_row()] = s;
    } else if (threadIdx.x < TS) {
      x[I * TS + threadIdx.x] = acc[threadIdx.x];
    }
    __syncthreads();
  }
}

// Backward substitution L^T x = rhs over tile columns Tsolve-1..0; tile rows >= Tsolve
// (the primal rows) hold given values that enter as  rhs_J -= sum_I L_IJ^T x_I.
template <class V>
__device__ void tri_bwd(const V& v, double* x, int Trows, int Tsolve, double* red, double* acc, double* dt = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = warp * 8;
  for (int J = Tsolve - 1; J >= 0; --J) {
    double c0 = 0.0, c1 = 0.0;
    for (int I = J + 1; I < Trows; ++I) {
      const double* t = v.tile(I, J) + row0 * TS + 2 * lane;
      double2 a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = ldg2(t + r * TS);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const double xr = x[I * TS + row0 + r];
        c0 += a[r].x * xr;
        c1 += a[r].y * xr;
      }
    }
    red[warp * TS + 2 * lane] = c0;
    red[warp * TS + 2 * lane + 1] = c1;
    __syncthreads();
    if (threadIdx.x < TS) {
      double s = x[J * TS + threadIdx.x];
#pragma unroll
      for (int w = 0; w < NTHR / 32; ++w) s -= red[w * TS + threadIdx.x];
      acc[threadIdx.x] = s;
    }
    __syncthreads();
    if (v.subst) {
      diag_subst(v.diag(J), acc, dt, true);
      if (threadIdx.x < TS) x[J * TS + threadIdx.x] = acc[threadIdx.x];
      __syncthreads();
      continue;
    }
    {
      const double* t = v.dinv(J) + row0 * TS + 2 * lane;
      c0 = c1 = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        double2 a = ldg2(t + r * TS);
        const double xr = acc[row0 + r];
        c0 += a.x * xr;
        c1 += a.y * xr;
      }
      red[warp * TS + 2 * lane] = c0;
      red[warp * TS + 2 * lane + 1] = c1;
    }
    __syncthreads();
    if (threadIdx.x < TS) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NTHR / 32; ++w) s += red[w * TS + threadIdx.x];
      x[J * TS + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------------------
// Full-factor solves (rhs stage, insulator precompute, recovery)
// ----------------------------------------------------------------------------------------

// In place on X (aug order): rows r solved, p rows get x_p - L_pr z_r.
// conductors_only: skip insulator patches (their rhs is phi(t) * XJ).
__global__ void __launch_bounds__(NTHR) k_fwd_full(DevPlan D, double* X, int conductors_only) {
  const int s = blockIdx.x;
  if (conductors_only && D.sigma[s] <= 0.0) return;
  extern __shared__ double sm[];
  double* acc = sm;
  double* x = sm + TS;
  const int T = D.T[s], Tr = D.Ti[s] + D.Tb[s];
  double* Xs = X + D.vec_off[s];
  for (int i = threadIdx.x; i < T * TS; i += blockDim.x) x[i] = Xs[i];
  __syncthreads();
  FullView v{D.A + D.a_off[s], D.Dinv + D.dinv_off[s], D.subst_local};
  tri_fwd(v, x, T, Tr, acc, x + D.maxT * TS);
  for (int i = threadIdx.x; i < T * TS; i += blockDim.x) Xs[i] = x[i];
}

// Recovery: a_r = L^-T (z_r - [0; w_b] - L_pr^T N p), a_p = N p, scattered into the local
// coefficient vectors (eliminated DOFs stay 0).
__global__ void __launch_bounds__(NTHR) k_bwd_full(DevPlan D, const double* __restrict__ X1,
                                                   const double* __restrict__ XW, const double* __restrict__ Pc,
                                                   double* a_loc, int nloc) {
  const int s = blockIdx.x;
  extern __shared__ double sm[];
  double* acc = sm;
  double* red = sm + TS;
  double* x = red + (NTHR / 32) * TS;
  const int Ti = D.Ti[s], Tb = D.Tb[s], T = D.T[s], Tr = Ti + Tb;
  const int64_t vo = D.vec_off[s];
  const int* grp = D.p_grp + D.p_off[s];
  const int np = D.np[s];
  for (int i = threadIdx.x; i < T * TS; i += blockDim.x) {
    double val;
    if (i < Ti * TS) val = X1[vo + i];
    else if (i < Tr * TS) val = X1[vo + i] - XW[vo + i];
    else {
      int t = i - Tr * TS;
      val = (t < np) ? Pc[grp[t]] : 0.0;
    }
    x[i] = val;
  }
  __syncthreads();
  FullView v{D.A + D.a_off[s], D.Dinv + D.dinv_off[s], D.subst_local};
  tri_bwd(v, x, T, Tr, red, acc, x + D.maxT * TS);
  const int* aug = D.aug + D.aug_off[s];
  double* as = a_loc + (int64_t)s * nloc;
  for (int i = threadIdx.x; i < T * TS; i += blockDim.x) {
    int a = aug[i];
    if (a >= 0) as[a] = x[i];
  }
}

// ----------------------------------------------------------------------------------------
// Trailing-block (b,p) solves: the F-apply halves
// ----------------------------------------------------------------------------------------

// XW = forward([v_b; 0]) with v_b = B_s^T lam (signed gather), over LS = [L_bb; L_pb].
__global__ void __launch_bounds__(NTHR) k_fwd_ls(DevPlan D, const double* __restrict__ lam, double* XW,
                                                 const PcgState* st) {
  if (st && st->done) return;
  const int s = blockIdx.x;
  extern __shared__ double sm[];
  double* acc = sm;
  double* x = sm + TS;
  const int Ti = D.Ti[s], Tb = D.Tb[s], Tp = D.Tp[s], nb = D.nb[s];
  const int* bl = D.b_lam + D.b_off[s];
  const double* bs = D.b_sign + D.b_off[s];
  for (int i = threadIdx.x; i < (Tb + Tp) * TS; i += blockDim.x) x[i] = (i < nb) ? bs[i] * lam[bl[i]] : 0.0;
  __syncthreads();
  LSView v{D.LS + D.ls_off[s], Tb, D.subst_local};
  tri_fwd(v, x, Tb + Tp, Tb, acc, x + D.maxTbp * TS);
  double* out = XW + D.vec_off[s] + Ti * TS;
  for (int i = threadIdx.x; i < (Tb + Tp) * TS; i += blockDim.x) out[i] = x[i];
}

// dst_b = L_bb^-T (src_b - L_pb^T N p) with the patch's primal values from Pc.
__global__ void __launch_bounds__(NTHR) k_bwd_ls(DevPlan D, const double* __restrict__ src, const double* __restrict__ Pc,
                                                 double* dst, const PcgState* st) {
  if (st && st->done) return;
  const int s = blockIdx.x;
  extern __shared__ double sm[];
  double* acc = sm;
  double* red = sm + TS;
  double* x = red + (NTHR / 32) * TS;
  const int Ti = D.Ti[s], Tb = D.Tb[s], Tp = D.Tp[s], np = D.np[s];
  const int* grp = D.p_grp + D.p_off[s];
  const double* in = src + D.vec_off[s] + Ti * TS;
  for (int i = threadIdx.x; i < (Tb + Tp) * TS; i += blockDim.x) {
    double val;
    if (i < Tb * TS) val = in[i];
    else {
      int t = i - Tb * TS;
      val = (t < np) ? Pc[grp[t]] : 0.0;
    }
    x[i] = val;
  }
  __syncthreads();
  LSView v{D.LS + D.ls_off[s], Tb, D.subst_local};
  tri_bwd(v, x, Tb + Tp, Tb, red, acc, x + D.maxTbp * TS);
  double* out = dst + D.vec_off[s] + Ti * TS;
  for (int i = threadIdx.x; i < Tb * TS; i += blockDim.x) out[i] = x[i];
}

// ----------------------------------------------------------------------------------------
// Coarse problem: G = sum_s N_s^T (src1_p - src2_p) (fixed CSR order), Pc = S_pp^-1 G.
// One CTA (n_c up to the dynamic shared-memory limit; DESIGN.md §7 lists the multi-CTA
// coarse solve as the next step for cfg4/cfg5).
// ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_coarse_solve(DevPlan D, const double* __restrict__ src1,
                                                       const double* __restrict__ src2, double* Pc,
                                                       const PcgState* st) {
  if (st && st->done) return;
  extern __shared__ double sm[];
  double* acc = sm;
  double* red = sm + TS;
  double* x = red + (NTHR / 32) * TS;
  const int Tc = D.Tc;
  for (int g = threadIdx.x; g < Tc * TS; g += blockDim.x) {
    double val = 0.0;
    if (g < D.nc) {
      for (int e = D.coarse_ptr[g]; e < D.coarse_ptr[g + 1]; ++e) {
        int64_t idx = D.coarse_idx[e];
        val += src2 ? (src1[idx] - src2[idx]) : src1[idx];
      }
    }
    x[g] = val;
  }
  __syncthreads();
  FullView v{D.C, D.Cinv, D.subst_coarse};
  tri_fwd(v, x, Tc, Tc, acc, x + Tc * TS);
  tri_bwd(v, x, Tc, Tc, red, acc, x + Tc * TS);
  for (int g = threadIdx.x; g < D.nc; g += blockDim.x) Pc[g] = x[g];
}

// ----------------------------------------------------------------------------------------
// Preconditioner: PW_b = S_bb (B_D^T r)_b, packed-lower SYMV (diagonal tiles full).
// ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_precond(DevPlan D, const double* __restrict__ r, double* PW,
                                                  const PcgState* st) {
  if (st && st->done) return;
  const int s = blockIdx.x;
  extern __shared__ double sm[];
  const int Ti = D.Ti[s], Tb = D.Tb[s], nb = D.nb[s];
  const int n = Tb * TS;
  double* v = sm;                         // n
  double* outr = v + n;                   // n (row contributions)
  double* colp = outr + n;                // 8 * n (per-warp column contributions)
  const int* bl = D.b_lam + D.b_off[s];
  const double* bs = D.b_sign + D.b_off[s];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double val = 0.0;
    if (i < nb) {
      int k = bl[i];
      double sg = bs[i];
      val = sg * (sg > 0 ? D.wplus[k] : D.wminus[k]) * r[k];
    }
    v[i] = val;
    outr[i] = 0.0;
  }
  for (int i = threadIdx.x; i < 8 * n; i += blockDim.x) colp[i] = 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = warp * 8;
  const double* S = D.Sbb + D.sbb_off[s];
  for (int I = 0; I < Tb; ++I) {
    double part[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) part[q] = 0.0;
    double xr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) xr[q] = v[I * TS + row0 + q];
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
        colp[warp * n + J * TS + 2 * lane] += c0;
        colp[warp * n + J * TS + 2 * lane + 1] += c1;
      }
    }
    double sum = warp_reduce8(part);
    if ((lane & 3) == 0) outr[I * TS + row0 + warp_reduce8_row()] = sum;
  }
  __syncthreads();
  double* out = PW + D.vec_off[s] + Ti * TS;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = outr[i];
#pragma unroll
    for (int w = 0; w < 8; ++w) acc += colp[w * n + i];
    out[i] = acc;
  }
}

// ----------------------------------------------------------------------------------------
// Jump operator + deterministic dot products + PCG scalar logic (Appendix C recurrences).
// ----------------------------------------------------------------------------------------
enum JumpMode { JUMP_D = 0, JUMP_F = 1, JUMP_M0 = 2, JUMP_M = 3, JUMP_PLAIN = 4 };

constexpr int RED_BLOCKS = 148;  // one partial per SM, fixed => deterministic

// out_k = w+ Y[idx+] - w- Y[idx-] (weights only in the preconditioner modes);
// JUMP_D: r = out (dual rhs d), lam = 0.  JUMP_F: q = out, alpha = rho/(pk.q).
// JUMP_M0: z = out, rho0 = rho = r.z (done if 0).  JUMP_M: z = out, rho_new = r.z,
// history, convergence test, beta.
__global__ void __launch_bounds__(256) k_jump(DevPlan D, const double* __restrict__ Y, double* out,
                                              const double* __restrict__ dotv, double* lam, PcgState* st,
                                              double* partial, double* hist, int mode, double rtol, int max_iter) {
  if (mode != JUMP_D && mode != JUMP_PLAIN && st->done) return;
  const int64_t m = D.m;
  const int64_t chunk = (m + RED_BLOCKS - 1) / RED_BLOCKS;
  const int64_t k0 = blockIdx.x * chunk, k1 = min(m, k0 + chunk);
  const bool weighted = (mode == JUMP_M0 || mode == JUMP_M);
  double local = 0.0;
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    double yp = Y[D.lam_idx_p[k]], ym = Y[D.lam_idx_m[k]];
    double val = weighted ? (D.wplus[k] * yp - D.wminus[k] * ym) : (yp - ym);
    out[k] = val;
    if (mode == JUMP_D) lam[k] = 0.0;
    else if (mode != JUMP_PLAIN) local += val * dotv[k];
  }
  __shared__ double sred[256];
  sred[threadIdx.x] = local;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sred[threadIdx.x] += sred[threadIdx.x + o];
    __syncthreads();
  }
  if (mode == JUMP_D || mode == JUMP_PLAIN) return;
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = sred[0];
    __threadfence();
    unsigned int prev = atomicAdd(&st->counter[0], 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double tot = 0.0;
  for (int b = 0; b < (int)gridDim.x; ++b) tot += ((volatile double*)partial)[b];
  st->counter[0] = 0;
  if (mode == JUMP_F) {
    st->pq = tot;
    if (!(tot > 0.0)) {  // loss of positive curvature: stop (reported as non-convergence)
      st->nan = 1;
      st->done = 1;
      st->failed = 1;
      return;
    }
    st->alpha = st->rho / tot;
  } else if (mode == JUMP_M0) {
    st->rho0 = tot;
    st->rho = tot;
    st->iter = 0;
    st->failed = 0;
    st->nan = 0;
    hist[0] = 1.0;
    st->done = (tot == 0.0 || m == 0) ? 1 : 0;
    if (!(tot >= 0.0)) {
      st->nan = 1;
      st->done = 1;
      st->failed = 1;
    }
  } else {  // JUMP_M
    st->rz = tot;
    const int it = st->iter + 1;
    st->iter = it;
    const double rel = sqrt(fmax(tot, 0.0) / st->rho0);
    hist[it] = rel;
    if (rel <= rtol) {
      st->done = 1;
    } else if (it >= max_iter || !(tot == tot)) {
      st->done = 1;
      st->failed = 1;
    } else {
      st->beta = tot / st->rho;
      st->rho = tot;
    }
  }
}

// lam += alpha pk; r -= alpha q
__global__ void k_axpy(double* lam, double* r, const double* __restrict__ pk, const double* __restrict__ q,
                       const PcgState* st, int64_t m) {
  if (st->done) return;
  const double a = st->alpha;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    lam[k] += a * pk[k];
    r[k] -= a * q[k];
  }
}

// pk = z + beta pk (init: pk = z). Runs after the convergence test of JUMP_M.
__global__ void k_xpay(double* pk, const double* __restrict__ z, const PcgState* st, int64_t m, int init) {
  if (st->done) return;
  const double b = init ? 0.0 : st->beta;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    pk[k] = init ? z[k] : z[k] + b * pk[k];
}

// glued readout: out[e] = a_loc[src[e]] (lowest-id owner copy)
__global__ void k_gather_glued(double* out, const double* __restrict__ a_loc, const int64_t* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a_loc[src[i]];
}

// copy helper (aug-ordered vectors)
__global__ void k_copy(double* dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace tcg
