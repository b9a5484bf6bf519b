// common.cuh — device helpers shared by the tcg kernels (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tcg {

constexpr int TS = 64;                 // tile edge
constexpr int TSZ = TS * TS;           // doubles per tile
constexpr int NTHR = 256;              // threads of the per-patch solver CTAs (8 warps)
constexpr int SPAD = 68;               // smem row stride (doubles) of staged GEMM tiles

__host__ __device__ inline int64_t tri_tiles(int64_t T) { return T * (T + 1) / 2; }
__host__ __device__ inline int64_t tri_off(int64_t I, int64_t J) { return (I * (I + 1) / 2 + J) * TSZ; }

// Device error record (first failure wins).
struct DevError {
  int flag;        // 0 ok, 1 not SPD
  int matrix;      // patch id, or -1 for the coarse matrix
  int index;       // pivot index within the matrix
  int pad;
  double value;
};

// PCG scalars living on the device (no host round trip inside an iteration).
struct PcgState {
  double rho, rho0, alpha, beta, pq, rz;
  int iter;        // completed iterations (F-applies)
  int done;        // 1 once converged (or max_iter reached); later kernels are no-ops
  int failed;      // 1 if max_iter reached without convergence
  int nan;         // 1 if a NaN/negative curvature guard fired
  int rp;          // buffer holding the final residual (persistent PCG)
  unsigned int counter[4];  // last-block-done counters for deterministic reductions
};

// One work item of the persistent stepper with the scalars of its patch embedded, so that
// an item costs one (shared-memory) load instead of an index -> patch-table chain.
//   P1/P5/SY/FW/BW: s = patch, I = tile row/column block; RHS: I = component (-1 insulator);
//   PC: s = coarse row block, I = column chunk.
struct __align__(16) ItemDesc {
  int s, I;
  int Ti, Tb, Tp, T;
  int nb, np;
  int64_t a_off, vec_off, b_off, p_off, sbb_off;
  int part;  // P5: bit 0: 0 = X_bb^T tiles (-> Y), 1 = Phi_b tiles (-> Y2); bits 4-5: gather code
             // (pcg.cu GAT); coarse items: chunk index
  int bc;    // P1/P5/SY: offset of the patch's b-position records in the block's shared cache (-1: none)
};
// b-position record (shared-memory cache of a block's patches): multiplier k, its sign on
// this side, B_D weights of this side (aown) and of the partner (apart), partner aug index
struct BPos {
  int64_t part;
  int k, pad;
  double aown, apart, sign;
};
// item phases of the stepper; the first NCACHE are the per-iteration ones (shared-memory cache)
// PH_P1 / PH_P5 are the per-iteration F-apply halves; PH_E1 / PH_E5 the same halves in their
// X_bb form for the per-step uses (R4 dual rhs, E1 recovery), which differ from PH_P1 / PH_P5
// when the iteration applies the explicit S_bb^-1 (ItemDesc part bit 3, pcg.cu). PH_P1B holds the
// S_bb^-1 items when they run under the sparse coarse solve's dependency waits (TCG_OVERLAP)
enum { PH_P1 = 0, PH_PC, PH_P5, PH_SY, PH_P1B, PH_FW, PH_FWA, PH_BW, PH_BWC, PH_RHS, PH_E1, PH_E5, NPH };
constexpr int NCACHE = 5;

// Per-matrix descriptor for the batched tiled Cholesky (patches and the coarse matrix).
struct CholDesc {
  int64_t a_off;     // offset (doubles) of the tile-packed lower matrix
  int64_t dinv_off;  // offset (doubles) of the diagonal-inverse tiles (Tfact tiles)
  int64_t sbb_off;   // offset (doubles) of the captured S_bb tiles (-1: none)
  int T;             // tile rows of the matrix
  int Tfact;         // tile columns to factor (remaining r columns)
  int Ti;            // capture S_bb at step k == Ti (before factoring column Ti)
  int Tb;            // tile size of the captured block
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce 8 per-lane partial row sums across a warp. On return, every lane holds the full
// sum for row index ((lane>>4)&1)*4 + ((lane>>3)&1)*2 + ((lane>>2)&1).
__device__ __forceinline__ double warp_reduce8(const double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  double k4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double send = b4 ? v[i] : v[i + 4];
    double keep = b4 ? v[i + 4] : v[i];
    k4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  double k2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    double send = b3 ? k4[i] : k4[i + 2];
    double keep = b3 ? k4[i + 2] : k4[i];
    k2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double send = b2 ? k2[0] : k2[1];
  double keep = b2 ? k2[1] : k2[0];
  double r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  return r;
}
__device__ __forceinline__ int warp_reduce8_row() {
  const int lane = threadIdx.x & 31;
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}

// D(8x8) += A(8x4) * B(4x8) on the FP64 tensor pipe (DMMA). Fragments: a = A[g][t],
// b = B[t][g], d = D[g][2t..2t+1] with g = lane>>2, t = lane&3.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

}  // namespace tcg
