// solve.cu — step c of the hot path, full-factor part: per implicit-Euler step the forward
// solve of the rhs (conductors) and the backward solve of the recovery stream the whole
// augmented factor of every patch (tile-row GEMVs with 64x64 diagonal-block inverses).
// The PCG itself (F-apply, preconditioner, coarse) is in pcg.cu.
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

constexpr int RED_BLOCKS = 148;  // blocks of the lambda-space reductions outside the persistent PCG

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
