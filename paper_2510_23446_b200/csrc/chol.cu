// chol.cu — step b of the hot path: batched right-looking tiled FP64 Cholesky of the
// gauged local matrices W^_rr (augmented with the primal rows) and of the coarse S_pp.
//
// Paper: local solves with W_rr, "two sequential Schur complements", done once
// because the material is linear and dt fixed.
// Layout: tile-packed lower triangle of 64x64 row-major tiles, matrix order
// [i | b | p]. Factoring only the r tile columns (Tfact = Ti + Tb) leaves
//   * the (p,r) block  = W^_pr L_rr^-T    (so Phi = W_rr^-1 W_rp = L_rr^-T L_pr^T),
//   * the (p,p) block  = W^_pp - W^_pr W_rr^-1 W^_rp = S^s (local coarse contribution),
// and the trailing (b,b) block at step k == Ti equals the interface Schur complement
// S_bb = W_bb - W_bi W_ii^-1 W_ib, captured for the Dirichlet preconditioner.
// Kernels per tile step k: capture (if k == Ti), POTRF of tile (k,k) + its triangular
// inverse, TRSM of the tile column below (as a GEMM with the inverse), and the SYRK/GEMM
// trailing update. The GEMMs run on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA).
#include "common.cuh"
#include "device.h"

namespace tcg {

// -------------------------------------------------------------------------------------
// 64x64 tile GEMM on DMMA: C = A B^T (mode 0) or C -= A B^T (mode 1). 128 threads.
// -------------------------------------------------------------------------------------

// ---- cp.async-staged DMMA tile products (two-stage pipeline over a K loop of tiles) -------
// Tiles are copied untransposed (row-major, row stride SPAD, 16-byte cp.async chunks); the
// fragment loads pick the operand orientation: A as [m][k] (AT = false) or as the transpose
// of a [k][m] tile (AT = true); B as [k][n] (BT = false) or as the transpose of [n][k]
// (BT = true). SPAD = 68: every orientation reads conflict-free half-warps.
__device__ __forceinline__ uint32_t cvta_s(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(cvta_s(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void stage_async(const double* __restrict__ g, double* s) {
  for (int c = threadIdx.x; c < TS * (TS / 2); c += blockDim.x) {
    const int r = c >> 5, q = c & 31;
    cp_async16(s + r * SPAD + 2 * q, g + r * TS + 2 * q);
  }
}
__device__ void tile_gemm_nt(const double* A, const double* B, double* C, double* sA, double* sB, int mode) {
  // operands staged with cp.async (no register round trip); the C tile of an update is
  // pulled into L2 meanwhile, so its read-modify-write after the products hits L2
  stage_async(A, sA);
  if (B != A) stage_async(B, sB);
  cp_commit();
  if (mode == 1)
    for (int e = threadIdx.x; e < TSZ / 16; e += blockDim.x) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + 16 * e));
  const double* sBB = (B != A) ? sB : sA;
  cp_wait<0>();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < TS; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sA[(wm + i * 8 + g) * SPAD + k0 + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = sBB[(wn + j * 8 + g) * SPAD + k0 + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  if (C == A) __syncthreads();  // in-place: everyone finished reading sA before C is written
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2* pc = reinterpret_cast<double2*>(C + (wm + i * 8 + g) * TS + wn + j * 8 + 2 * t);
      if (mode == 0) {
        *pc = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        double2 c = *pc;
        c.x -= acc[i][j][0];
        c.y -= acc[i][j][1];
        *pc = c;
      }
    }
}

// -------------------------------------------------------------------------------------
// POTRF of diagonal tile (k,k) fused with its triangular inverse (into the Dinv store).
// One CTA (256 threads) per matrix, the tile and X = L^-1 in shared memory (row stride 65).
// Blocked by 8-column panels (few barriers; the per-column latency chain stays inside one
// warp):
//   panel p (warp 0, lane l = rows c0+l and c0+32+l in registers, shuffles): unblocked
//     Cholesky of the 8 panel columns;
//   trailing update (all threads): W_ic -= sum_{q<8} L_i,c0+q L_c,c0+q for c0+8 <= c <= i;
//   X = L^-1 by right-looking forward elimination of L X = I in the same panels: warp 0
//     finishes the 8 panel rows of X, the trailing phase subtracts their rank-8 contribution
//     from the rows below.
// -------------------------------------------------------------------------------------
constexpr int PS = TS + 1;  // padded shared row stride of the POTRF tiles
#ifdef POTRF_PROBE_ON
__device__ long long g_probe[4096];
#define POTRF_PROBE(slot) if (blockIdx.x == 0 && lane == 0 && p < 2) { asm volatile("" ::: "memory"); g_probe[(8 * p + jj) * 4 + (slot)] = clock64(); }
#else
#define POTRF_PROBE(x)
#endif
__global__ void __launch_bounds__(256) k_potrf(const CholDesc* __restrict__ ds, int k, double* base, double* dinv,
                                               DevError* err, int coarse) {
  const CholDesc d = ds[blockIdx.x];
  if (k >= d.Tfact) return;
  extern __shared__ double psm[];
  double* As = psm;            // 64 x PS
  double* Xs = psm + TS * PS;  // 64 x PS
  __shared__ double dinvd[TS];  // 1 / L_jj
  double* tile = base + d.a_off + tri_off(k, k);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int e = t; e < TSZ; e += blockDim.x) {
    const int i = e >> 6, c = e & 63;
    As[i * PS + c] = (c <= i) ? tile[e] : 0.0;
    Xs[i * PS + c] = (c == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int p = 0; p < 8; ++p) {
    const int c0 = 8 * p;
    if (warp == 0) {
      // lane l owns rows c0+l and c0+32+l of the 8-column panel in registers; column j of L
      // is broadcast by shuffles (fully unrolled: no local memory, no barriers)
      const int r1 = c0 + lane, r2 = c0 + 32 + lane;
      const bool v1 = r1 < TS, v2 = r2 < TS;
      double a1[8], a2[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        a1[q] = v1 ? As[r1 * PS + c0 + q] : 0.0;
        a2[q] = v2 ? As[r2 * PS + c0 + q] : 0.0;
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int j = c0 + jj;
        POTRF_PROBE(0);
        double piv = __shfl_sync(0xffffffffu, a1[jj], jj);
        if (!(piv > 0.0)) {
          if (lane == 0 && atomicCAS(&err->flag, 0, 1) == 0) {
            err->matrix = coarse ? -1 : (int)blockIdx.x;
            err->index = k * TS + j;
            err->value = piv;
          }
          piv = 1.0;
        }
        const double inv = rsqrt(piv);
        POTRF_PROBE(1);
        a1[jj] = (r1 > j) ? a1[jj] * inv : (r1 == j ? piv * inv : a1[jj]);
        a2[jj] *= inv;
        if (lane == 0) dinvd[j] = inv;
        POTRF_PROBE(2);
#pragma unroll
        for (int q = jj + 1; q < 8; ++q) {
          const double lc = __shfl_sync(0xffffffffu, a1[jj], q);  // L[c0+q][j]
          a1[q] = (r1 >= c0 + q) ? a1[q] - a1[jj] * lc : a1[q];
          a2[q] -= a2[jj] * lc;
        }
        POTRF_PROBE(3);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (v1) As[r1 * PS + c0 + q] = (c0 + q <= r1) ? a1[q] : 0.0;
        if (v2) As[r2 * PS + c0 + q] = a2[q];
      }
      __syncwarp();
      // rows c0..c0+7 of X (lane = columns lane, lane+32): X_jc = (X_jc - sum_{c0<=q<j} L_jq X_qc) / L_jj
      double x1[8], x2[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int j = c0 + jj;
        double u1 = Xs[j * PS + lane], u2 = Xs[j * PS + lane + 32];
#pragma unroll
        for (int q = 0; q < jj; ++q) {
          const double l = As[j * PS + c0 + q];
          u1 -= l * x1[q];
          u2 -= l * x2[q];
        }
        x1[jj] = u1 * dinvd[j];
        x2[jj] = u2 * dinvd[j];
        Xs[j * PS + lane] = x1[jj];
        Xs[j * PS + lane + 32] = x2[jj];
      }
    }
    __syncthreads();
    // trailing updates, thread = (column c, every 4th row): W (columns >= c0+8, rows >= c) and
    // X (columns < c0+8, rows >= c0+8): rank-8 with the panel columns / panel rows
    {
      const int c = t & 63, ir = t >> 6;
      if (c < c0 + 8) {
        double xc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xc[q] = Xs[(c0 + q) * PS + c];
        for (int i = c0 + 8 + ir; i < TS; i += 8) {
          const int i2 = i + 4;
          double acc = Xs[i * PS + c], acc2 = (i2 < TS) ? Xs[i2 * PS + c] : 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            acc -= As[i * PS + c0 + q] * xc[q];
            if (i2 < TS) acc2 -= As[i2 * PS + c0 + q] * xc[q];
          }
          Xs[i * PS + c] = acc;
          if (i2 < TS) Xs[i2 * PS + c] = acc2;
        }
      } else {
        double lc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) lc[q] = As[c * PS + c0 + q];
        for (int i = c0 + 8 + ir; i < TS; i += 8) {  // two rows per trip: independent chains
          const int i2 = i + 4;
          double acc = As[i * PS + c], acc2 = (i2 < TS) ? As[i2 * PS + c] : 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            acc -= As[i * PS + c0 + q] * lc[q];
            if (i2 < TS) acc2 -= As[i2 * PS + c0 + q] * lc[q];
          }
          if (i >= c) As[i * PS + c] = acc;
          if (i2 < TS && i2 >= c) As[i2 * PS + c] = acc2;
        }
      }
    }
    __syncthreads();
  }
  double* out = dinv + d.dinv_off + (int64_t)k * TSZ;
  for (int e = t; e < TSZ; e += blockDim.x) {
    const int i = e >> 6, c = e & 63;
    tile[e] = (c <= i) ? As[i * PS + c] : 0.0;
    out[e] = (c <= i) ? Xs[i * PS + c] : 0.0;
  }
}

// A_Ik <- A_Ik L_kk^-T for I in (k, T). grid (maxT-k-1, nmat).
// subst = 0: GEMM with the inverse tile on DMMA; subst = 1: row-wise forward substitution.
__global__ void __launch_bounds__(128) k_trsm(const CholDesc* __restrict__ ds, int k, double* base, const double* dinv,
                                              int subst) {
  const CholDesc d = ds[blockIdx.y];
  const int I = k + 1 + blockIdx.x;
  if (k >= d.Tfact || I >= d.T) return;
  extern __shared__ double smem[];
  double* A = base + d.a_off + tri_off(I, k);
  if (!subst) {
    const double* Li = dinv + d.dinv_off + (int64_t)k * TSZ;
    tile_gemm_nt(A, Li, A, smem, smem + TS * SPAD, 0);
    return;
  }
  double* sA = smem;            // 64 x 65
  double* sL = smem + TS * 65;  // 64 x 65
  const double* L = base + d.a_off + tri_off(k, k);
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) {
    sA[(e / TS) * 65 + (e % TS)] = A[e];
    sL[(e / TS) * 65 + (e % TS)] = L[e];
  }
  __syncthreads();
  if (threadIdx.x < TS) {
    double* a = sA + threadIdx.x * 65;
    for (int j = 0; j < TS; ++j) {
      double v = a[j];
      for (int q = 0; q < j; ++q) v -= sL[j * 65 + q] * a[q];
      a[j] = v / sL[j * 65 + j];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) A[e] = sA[(e / TS) * 65 + (e % TS)];
}

// A_IJ -= L_Ik L_Jk^T for k < J <= I < T. grid (ntri, nmat).
__global__ void __launch_bounds__(128) k_update(const CholDesc* __restrict__ ds, int k, double* base) {
  const CholDesc d = ds[blockIdx.y];
  if (k >= d.Tfact) return;
  const int64_t y = blockIdx.x;
  int Ip = (int)((sqrt(8.0 * (double)y + 1.0) - 1.0) * 0.5);
  while ((int64_t)Ip * (Ip + 1) / 2 > y) --Ip;
  while ((int64_t)(Ip + 1) * (Ip + 2) / 2 <= y) ++Ip;
  const int Jp = (int)(y - (int64_t)Ip * (Ip + 1) / 2);
  const int I = k + 1 + Ip, J = k + 1 + Jp;
  if (I >= d.T) return;
  extern __shared__ double smem[];
  const double* LI = base + d.a_off + tri_off(I, k);
  const double* LJ = base + d.a_off + tri_off(J, k);
  double* C = base + d.a_off + tri_off(I, J);
  tile_gemm_nt(LI, LJ, C, smem, smem + TS * SPAD, 1);
}

// Copy the trailing (b,b) block at step k == Ti: S_bb = W_bb - W_bi W_ii^-1 W_ib.
__global__ void k_capture_sbb(const CholDesc* __restrict__ ds, int k, const double* base, double* sbb) {
  const CholDesc d = ds[blockIdx.y];
  if (d.Ti != k || d.sbb_off < 0) return;
  const int64_t y = blockIdx.x;
  if (y >= tri_tiles(d.Tb)) return;
  int Ip = (int)((sqrt(8.0 * (double)y + 1.0) - 1.0) * 0.5);
  while ((int64_t)Ip * (Ip + 1) / 2 > y) --Ip;
  while ((int64_t)(Ip + 1) * (Ip + 2) / 2 <= y) ++Ip;
  const int Jp = (int)(y - (int64_t)Ip * (Ip + 1) / 2);
  const double* src = base + d.a_off + tri_off(d.Ti + Ip, d.Ti + Jp);
  double* dst = sbb + d.sbb_off + tri_off(Ip, Jp);
  for (int e = threadIdx.x; e < TSZ / 2; e += blockDim.x)
    reinterpret_cast<double2*>(dst)[e] = reinterpret_cast<const double2*>(src)[e];
}

// Coarse assembly S_pp = sum_s N_s^T S^s N_s, S^s = trailing (p,p) block of patch s.
// Patches of one parity colour (ix%2, iy%2, iz%2) share no primal group, so each colour is
// one conflict-free launch; colours run in a fixed order (deterministic sums).
__global__ void k_coarse_scatter(DevPlan D, const int* __restrict__ patches, int npat) {
  const int pi = blockIdx.x;  // grid (npat, chunks): chunk y takes entries y, y + gridDim.y, ...
  if (pi >= npat) return;
  const int s = patches[pi];
  const int Tr = D.Ti[s] + D.Tb[s];
  const int np = D.np[s];
  const int* grp = D.p_grp + D.p_off[s];
  const double* A = D.Ar[D.owner[s]] + D.a_off[s];  // S^s lives on the patch's owner
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < np * np; e += gridDim.y * blockDim.x) {
    const int a = e / np, b = e % np;
    const int ga = grp[a], gb = grp[b];
    if (ga < gb) continue;               // each unordered pair once, into the lower triangle
    if (ga == gb && a != b) continue;    // cannot happen (a group appears once per patch)
    // S^s[a][b] from the stored lower tiles (symmetric)
    int ra = a, rb = b;
    if ((ra >> 6) < (rb >> 6)) { int tmp = ra; ra = rb; rb = tmp; }
    const double v = A[tri_off(Tr + (ra >> 6), Tr + (rb >> 6)) + (ra & 63) * TS + (rb & 63)];
    const int GI = ga >> 6, GJ = gb >> 6;
    double* dst = D.C + tri_off(GI, GJ) + (ga & 63) * TS + (gb & 63);
    *dst += v;
  }
}

// Identity padding of the coarse matrix diagonal beyond n_c.
__global__ void k_coarse_pad(DevPlan D) {
  int64_t g = D.nc + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= (int64_t)D.Tc * TS) return;
  D.C[tri_off(g >> 6, g >> 6) + (g & 63) * TS + (g & 63)] = 1.0;
}

}  // namespace tcg

namespace tcg {

// -------------------------------------------------------------------------------------
// Inverse factors for the chain-free PCG (DESIGN.md §5 "F-apply"):
//   X = L^-1 by blocked inversion  X_II = L_II^-1,  X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ,
//   Phi^T = L_pb X_bb  (= W_pr W_rr^-1 restricted to the b columns).
// All tile products on DMMA. acc[4][4][2] holds a 64x64 tile as in tile_gemm_nt.
// -------------------------------------------------------------------------------------
__device__ __forceinline__ void stage_tile_T(const double* __restrict__ g, double* s) {  // s[n][k] = g[k][n]
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) {
    int k = e / TS, n = e % TS;
    s[n * SPAD + k] = g[e];
  }
}

__device__ __forceinline__ void mma_acc(const double* sA, const double* sB, double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll 4
  for (int k0 = 0; k0 < TS; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sA[(wm + i * 8 + g) * SPAD + k0 + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = sB[(wn + j * 8 + g) * SPAD + k0 + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

__device__ __forceinline__ void acc_zero(double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// write acc (scaled) to a row-major global tile
__device__ __forceinline__ void acc_store(double* C, const double (&acc)[4][4][2], double scale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<double2*>(C + (wm + i * 8 + g) * TS + wn + j * 8 + 2 * t) =
          make_double2(scale * acc[i][j][0], scale * acc[i][j][1]);
}

// write acc into smem as the B operand of a following NN product (sB[n][k] = acc[k][n])
__device__ __forceinline__ void acc_to_smemT(double* sB, const double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = wm + i * 8 + g, n = wn + j * 8 + 2 * t;
      sB[n * SPAD + m] = acc[i][j][0];
      sB[(n + 1) * SPAD + m] = acc[i][j][1];
    }
}

template <bool AT, bool BT>
__device__ __forceinline__ void mma_acc2(const double* sA, const double* sB, double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll 4
  for (int k0 = 0; k0 < TS; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = AT ? sA[(k0 + t) * SPAD + wm + i * 8 + g] : sA[(wm + i * 8 + g) * SPAD + k0 + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = BT ? sB[(wn + j * 8 + g) * SPAD + k0 + t] : sB[(k0 + t) * SPAD + wn + j * 8 + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}
// ---- deep-K tile stream: acc += sum_{q < nk} op(A_q) op(B_q), K split into 32-wide halves,
// 3-stage cp.async pipeline (one __syncthreads pair per half). A stage holds the two operand
// halves in compact layouts: K along the stored tile's rows -> [32][SPAD] (all 64 columns);
// K along its columns -> [64][HPAD]. Fragment reads are conflict-free per half-warp in both
// (row strides 68 and 36 doubles are 4 mod 16 banks). 110.6 KB per CTA: 2 CTAs (8 warps) per
// SM, where the 2-stage full-tile pipeline (139 KB) allowed one.
constexpr int HPAD = 36;
constexpr int HSZ = TS * HPAD;  // >= 32 * SPAD
constexpr int MMA_STG = 2 * HSZ;
constexpr int MMA_SMEM_DOUBLES = 3 * MMA_STG;  // also >= 2 full SPAD tiles (mul_left_store, mirrors)
static_assert(MMA_SMEM_DOUBLES >= 2 * TS * SPAD, "stream buffer must hold two full tiles");
template <bool KROWS>
__device__ __forceinline__ void stage_half(const double* __restrict__ g, double* s, int kh) {
  if (KROWS) {
    for (int c = threadIdx.x; c < 32 * (TS / 2); c += blockDim.x) {
      const int r = c >> 5, q = c & 31;
      cp_async16(s + r * SPAD + 2 * q, g + (kh * 32 + r) * TS + 2 * q);
    }
  } else {
    for (int c = threadIdx.x; c < TS * 16; c += blockDim.x) {
      const int r = c >> 4, q = c & 15;
      cp_async16(s + r * HPAD + 2 * q, g + r * TS + kh * 32 + 2 * q);
    }
  }
}
template <bool AT, bool BT>
__device__ __forceinline__ void mma_acc_h(const double* sA, const double* sB, double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll 4
  for (int k0 = 0; k0 < 32; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = AT ? sA[(k0 + t) * SPAD + wm + i * 8 + g] : sA[(wm + i * 8 + g) * HPAD + k0 + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = BT ? sB[(wn + j * 8 + g) * HPAD + k0 + t] : sB[(k0 + t) * SPAD + wn + j * 8 + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}
template <bool AT, bool BT, class AF, class BF>
__device__ __forceinline__ void mma_stream(AF atile, BF btile, int nk, double* sm, double (&acc)[4][4][2]) {
  if (nk <= 0) return;
  const int ns = 2 * nk;
  auto issue = [&](int s) {
    double* b = sm + (s % 3) * MMA_STG;
    stage_half<AT>(atile(s >> 1), b, s & 1);
    stage_half<!BT>(btile(s >> 1), b + HSZ, s & 1);
  };
  issue(0);
  cp_commit();
  issue(1);
  cp_commit();
  for (int s = 0; s < ns; ++s) {
    if (s + 2 < ns) issue(s + 2);
    cp_commit();
    cp_wait<2>();
    __syncthreads();
    const double* cu = sm + (s % 3) * MMA_STG;
    mma_acc_h<AT, BT>(cu, cu + HSZ, acc);
    __syncthreads();
  }
}
// acc (64x64 row-major [m][n]) into shared memory with row stride SPAD
__device__ __forceinline__ void acc_to_smem(double* s, const double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double* p = s + (wm + i * 8 + g) * SPAD + wn + j * 8 + 2 * t;
      p[0] = acc[i][j][0];
      p[1] = acc[i][j][1];
    }
}
// out = scale * A * T with T = acc (NN), A a row-major global tile; sm: >= 2 tiles
__device__ __forceinline__ void mul_left_store(const double* Ag, const double (&acc)[4][4][2], double scale, double* out,
                                               double* sm) {
  double* sA = sm;
  double* sT = sm + TS * SPAD;
  acc_to_smem(sT, acc);
  stage_async(Ag, sA);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  double acc2[4][4][2];
  acc_zero(acc2);
  mma_acc2<false, false>(sA, sT, acc2);
  acc_store(out, acc2, scale);
}

struct InvDesc {
  int64_t l_off;     // matrix L (tile-packed lower) base offset in Lbase
  int64_t x_off;     // output X base offset (tile-packed lower, T tiles) in Xbase
  int64_t dinv_off;  // diagonal inverses base in Dbase
  int shift;         // L tile (I,J) = tile (shift+I, shift+J); diag inverse index shift+I
  int T;             // tiles to invert
};

// Row I of X = L^-1 for every matrix with T > I. grid (I+1, nmat), 128 threads.
__global__ void __launch_bounds__(128) k_trinv_row(const InvDesc* __restrict__ ds, int I, const double* Lbase,
                                                   double* Xbase, const double* Dbase) {
  const InvDesc d = ds[blockIdx.y];
  const int J = blockIdx.x;
  if (I >= d.T || J > I) return;
  extern __shared__ __align__(16) double smem[];
  const double* Linv = Dbase + d.dinv_off + (int64_t)(d.shift + I) * TSZ;
  double* X = Xbase + d.x_off + tri_off(I, J);
  if (J == I) {
    for (int e = threadIdx.x; e < TSZ / 2; e += blockDim.x)
      reinterpret_cast<double2*>(X)[e] = reinterpret_cast<const double2*>(Linv)[e];
    return;
  }
  double acc[4][4][2];
  acc_zero(acc);
  mma_stream<false, false>([&](int q) { return Lbase + d.l_off + tri_off(d.shift + I, d.shift + J + q); },
                           [&](int q) { return Xbase + d.x_off + tri_off(J + q, J); }, I - J, smem, acc);
  mul_left_store(Linv, acc, -1.0, X, smem);
}

}  // namespace tcg

namespace tcg {

// Full symmetric S_pp^-1 = X_c^T X_c (X_c = L_c^-1 tile-packed lower), stored as Tc x Tc
// row-major 64x64 tiles: tile (I,J) = sum_{K >= max(I,J)} X_KI^T X_KJ. grid (Tc, Tc), 128 thr.
__global__ void __launch_bounds__(128) k_sinv(const double* __restrict__ X, double* Sinv, int Tc) {
  const int I = blockIdx.y, J = blockIdx.x;
  extern __shared__ __align__(16) double smem[];
  double acc[4][4][2];
  acc_zero(acc);
  const int K0 = max(I, J);
  mma_stream<true, false>([&](int q) { return X + tri_off(K0 + q, I); }, [&](int q) { return X + tri_off(K0 + q, J); },
                          Tc - K0, smem, acc);
  acc_store(Sinv + ((int64_t)I * Tc + J) * TSZ, acc, 1.0);
}

// Explicit S_bb^-1 = X_bb^T X_bb (X_bb = L_bb^-1, the trailing (b,b) block of L_rr^-1 in the
// inverse-factor store) per patch, tile-packed lower in the S_bb layout: tile (I,J), I >= J,
// = sum_{K >= I} X_KI^T X_KJ. Diagonal tiles are written full and exactly symmetric (lower
// triangle mirrored). grid (tri_tiles(maxTb), #patches), 128 threads.
__global__ void __launch_bounds__(128) k_sbbinv(DevPlan D, const int* plist, double* SI) {
  const int s = plist[blockIdx.y];
  const int Tb = D.Tb[s], Ti = D.Ti[s];
  const int64_t y = blockIdx.x;
  if (y >= (int64_t)Tb * (Tb + 1) / 2) return;
  int I = (int)((sqrt(8.0 * (double)y + 1.0) - 1.0) * 0.5);
  while ((int64_t)I * (I + 1) / 2 > y) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= y) ++I;
  const int J = (int)(y - (int64_t)I * (I + 1) / 2);
  extern __shared__ __align__(16) double smem[];
  const double* X = D.A + D.a_off[s];
  double acc[4][4][2];
  acc_zero(acc);
  mma_stream<true, false>([&](int q) { return X + tri_off(Ti + I + q, Ti + I); },
                          [&](int q) { return X + tri_off(Ti + I + q, Ti + J); }, Tb - I, smem, acc);
  double* out = SI + D.sbb_off[s] + tri_off(I, J);
  if (I != J) {
    acc_store(out, acc, 1.0);
    return;
  }
  double* st = smem;  // (the pipeline's buffers are free again)
  acc_to_smem(st, acc);
  __syncthreads();
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) {
    const int r = e / TS, c = e % TS;
    out[e] = (c <= r) ? st[r * SPAD + c] : st[c * SPAD + r];
  }
}

// ---- left-looking factorisation (DESIGN.md §5 "Factorisation"): column J of every matrix is
// brought up to date in one pass, A_IJ = W_IJ - sum_{K<J} L_IK L_JK^T for all I >= J, as one
// deep-K DMMA stream per tile (operands read once per column, the tile written once) instead
// of J rank-64 read-modify-writes; potrf + trsm of column J follow. In the b block
// (Ti <= J <= I < Tfact) the partial sum over the i columns gives the interface Schur
// complement S_bb_IJ = W_IJ - sum_{K<Ti} L_IK L_JK^T, written before the stream continues.
// grid (maxT - J, nmat), 128 threads, MMA_SMEM_DOUBLES shared.
__device__ __forceinline__ void acc_sub_store(const double* W, double* out, const double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = (wm + i * 8 + g) * TS + wn + j * 8 + 2 * t;
      const double2 w = *reinterpret_cast<const double2*>(W + o);
      *reinterpret_cast<double2*>(out + o) = make_double2(w.x - acc[i][j][0], w.y - acc[i][j][1]);
    }
}
__global__ void __launch_bounds__(128) k_colupd(const CholDesc* __restrict__ ds, int J, double* base, double* sbb) {
  const CholDesc d = ds[blockIdx.y];
  const int I = J + blockIdx.x;
  if (J >= d.Tfact || I >= d.T) return;
  const bool cap = sbb && d.sbb_off >= 0 && J >= d.Ti && I < d.Tfact;
  if (J == 0 && !cap) return;
  extern __shared__ __align__(16) double smem[];
  double* L = base + d.a_off;
  double* C = L + tri_off(I, J);
  double acc[4][4][2];
  acc_zero(acc);
  const int K1 = cap ? d.Ti : J;
  mma_stream<false, true>([&](int q) { return L + tri_off(I, q); }, [&](int q) { return L + tri_off(J, q); }, K1, smem, acc);
  if (cap) {
    acc_sub_store(C, sbb + d.sbb_off + tri_off(I - d.Ti, J - d.Ti), acc);
    mma_stream<false, true>([&](int q) { return L + tri_off(I, d.Ti + q); }, [&](int q) { return L + tri_off(J, d.Ti + q); },
                            J - d.Ti, smem, acc);
  }
  acc_sub_store(C, C, acc);
}
// after the Tfact columns: the trailing tiles (I, J), Tfact <= J <= I < T (the local coarse
// contribution S^s, or a front's update matrix), A_IJ -= sum_{K<Tfact} L_IK L_JK^T.
// grid (tri_tiles(max T - Tfact), nmat).
__global__ void __launch_bounds__(128) k_tailupd(const CholDesc* __restrict__ ds, double* base) {
  const CholDesc d = ds[blockIdx.y];
  const int Tt = d.T - d.Tfact;
  const int64_t y = blockIdx.x;
  if (y >= (int64_t)Tt * (Tt + 1) / 2 || d.Tfact == 0) return;
  int Ip = (int)((sqrt(8.0 * (double)y + 1.0) - 1.0) * 0.5);
  while ((int64_t)Ip * (Ip + 1) / 2 > y) --Ip;
  while ((int64_t)(Ip + 1) * (Ip + 2) / 2 <= y) ++Ip;
  const int Jp = (int)(y - (int64_t)Ip * (Ip + 1) / 2);
  const int I = d.Tfact + Ip, J = d.Tfact + Jp;
  extern __shared__ __align__(16) double smem[];
  double* L = base + d.a_off;
  double* C = L + tri_off(I, J);
  double acc[4][4][2];
  acc_zero(acc);
  mma_stream<false, true>([&](int q) { return L + tri_off(I, q); }, [&](int q) { return L + tri_off(J, q); }, d.Tfact,
                          smem, acc);
  acc_sub_store(C, C, acc);
}

}  // namespace tcg

namespace tcg {

// In-place inverse of the augmented local factor: row block I of every patch
//   I <  Tr:  X_IJ = L_II^-1                          (J = I)
//             X_IJ = -L_II^-1 sum_{K=J}^{I-1} L_IK X_KJ   (J < I)
//   I >= Tr:  PhiT_IJ = sum_{K=J}^{Tr-1} L_IK X_KJ        (J < Tr; = W_pr W_rr^-1)
// Rows < I already hold X, rows > I still hold L, so row I is computed into a per-patch
// scratch row and copied back (k_xrow_copy) before row I+1. grid (maxTr, P), 128 threads.
__global__ void __launch_bounds__(128) k_xinv_row(DevPlan D, int I, double* scratch, const int64_t* scr_off,
                                                  const int* plist) {
  const int s = plist[blockIdx.y], J = blockIdx.x;
  const int Tr = D.Ti[s] + D.Tb[s], T = D.T[s];
  if (I >= T || J >= Tr || (I < Tr && J > I)) return;
  extern __shared__ __align__(16) double smem[];
  const double* A = D.A + D.a_off[s];
  double* out = scratch + scr_off[s] + (int64_t)J * TSZ;
  if (I < Tr && J == I) {
    const double* Li = D.Dinv + D.dinv_off[s] + (int64_t)I * TSZ;
    for (int e = threadIdx.x; e < TSZ / 2; e += blockDim.x)
      reinterpret_cast<double2*>(out)[e] = reinterpret_cast<const double2*>(Li)[e];
    return;
  }
  const int Kend = (I < Tr) ? I : Tr;
  double acc[4][4][2];
  acc_zero(acc);
  // rows < I already hold X = L^-1, rows >= I still hold L: sum_{K=J}^{Kend-1} L_IK X_KJ
  mma_stream<false, false>([&](int q) { return A + tri_off(I, J + q); }, [&](int q) { return A + tri_off(J + q, J); },
                           Kend - J, smem, acc);
  if (I >= Tr) {
    acc_store(out, acc, 1.0);
    return;
  }
  mul_left_store(D.Dinv + D.dinv_off[s] + (int64_t)I * TSZ, acc, -1.0, out, smem);
}

__global__ void k_xrow_copy(DevPlan D, int I, const double* scratch, const int64_t* scr_off, const int* plist) {
  const int s = plist[blockIdx.y], J = blockIdx.x;
  const int Tr = D.Ti[s] + D.Tb[s], T = D.T[s];
  if (I >= T || J >= Tr || (I < Tr && J > I)) return;
  const double2* src = reinterpret_cast<const double2*>(scratch + scr_off[s] + (int64_t)J * TSZ);
  double2* dst = reinterpret_cast<double2*>(D.A + D.a_off[s] + tri_off(I, J));
  for (int e = threadIdx.x; e < TSZ / 2; e += blockDim.x) dst[e] = src[e];
}

}  // namespace tcg
