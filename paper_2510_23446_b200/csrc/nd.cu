// nd.cu — sparse (nested-dissection, multifrontal) coarse problem, setup kernels
// (SURVEY §8(f) f1). The frontal matrix of node x (coarse_nd.h) is stored like a patch:
// tile-packed lower 64x64 tiles, order [V_x | B_x]. Partial Cholesky of the V columns
// (run_cholesky with Tfact = T_V) leaves the update matrix U_x = F_BB - L_BV L_BV^T in the
// trailing block; the in-place inverse (k_xinv_row) turns the V columns into
// [L_VV^-1 ; L_BV L_VV^-1], which the stepper applies as GEMVs (forward: node rhs ->
// y_x = L_VV^-1 f_V and the update f_B - L_BV y_x passed to the parent; backward:
// x_V = L_VV^-T y_x - (L_BV L_VV^-1)^T x_B).
// Assembly: S_pp = sum_s N_s^T S^s N_s entries are scattered into the frontal
// of the node that eliminates the first of their two groups (8 parity colours of patches:
// conflict-free, fixed order); children's update matrices are extend-added into the parent
// one child slot per launch (fixed order): deterministic.
#include "common.cuh"
#include "device.h"

namespace tcg {

// identity on the padded diagonal positions of every frontal: V pad [nV, 64 TV) and
// B pad [64 TV + nB, 64 T). One block per node.
__global__ void k_nd_pad(const int* __restrict__ tv, const int* __restrict__ tt, const int* __restrict__ nv,
                         const int* __restrict__ nbv, const int64_t* __restrict__ aoff, double* FR) {
  const int x = blockIdx.x;
  const int TV = tv[x], T = tt[x], nV = nv[x], nB = nbv[x];
  double* F = FR + aoff[x];
  for (int i = threadIdx.x; i < T * TS; i += blockDim.x) {
    const bool pad = (i >= nV && i < TV * TS) || (i >= TV * TS + nB);
    if (pad) F[tri_off(i >> 6, i >> 6) + (i & 63) * TS + (i & 63)] = 1.0;
  }
}

// S^s of patch s (trailing (p,p) block of its factor) into the frontal matrices: map[e] for
// e = a * np + b is the target offset in FR (lower storage) or -1.
__global__ void k_nd_scatter(DevPlan D, const int* __restrict__ patches, int npat, const int64_t* __restrict__ moff,
                             const int64_t* __restrict__ map, double* FR) {
  const int pi = blockIdx.x;
  if (pi >= npat) return;
  const int s = patches[pi];
  const int Tr = D.Ti[s] + D.Tb[s];
  const int np = D.np[s];
  const double* A = D.Ar[D.owner[s]] + D.a_off[s];
  const int64_t* mp = map + moff[s];
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < np * np; e += gridDim.y * blockDim.x) {
    const int64_t t = mp[e];
    if (t < 0) continue;
    int ra = e / np, rb = e % np;
    if ((ra >> 6) < (rb >> 6)) {
      const int tmp = ra;
      ra = rb;
      rb = tmp;
    }
    FR[t] += A[tri_off(Tr + (ra >> 6), Tr + (rb >> 6)) + (ra & 63) * TS + (rb & 63)];
  }
}

// Extend-add of child update matrices into their parents, one child slot per launch.
// ext[xo[c] + i] = parent frontal position of B_c[i]. grid (chunks, nchild).
__global__ void k_nd_extend(const int* __restrict__ kids, int nkids, const int* __restrict__ parent,
                            const int* __restrict__ tv, const int* __restrict__ nbv, const int64_t* __restrict__ aoff,
                            const int64_t* __restrict__ xo, const int* __restrict__ ext, double* FR) {
  const int ci = blockIdx.y;
  if (ci >= nkids) return;
  const int c = kids[ci], p = parent[c];
  const int nB = nbv[c], TVc = tv[c];
  const double* Fc = FR + aoff[c];
  double* Fp = FR + aoff[p];
  const int* ep = ext + xo[c];
  const int64_t npair = (int64_t)nB * (nB + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npair; q += (int64_t)gridDim.x * blockDim.x) {
    // q -> (i, j), j <= i < nB (row-major lower triangle)
    int i = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
    while ((int64_t)i * (i + 1) / 2 > q) --i;
    while ((int64_t)(i + 1) * (i + 2) / 2 <= q) ++i;
    const int j = (int)(q - (int64_t)i * (i + 1) / 2);
    const int ri = TVc * TS + i, rj = TVc * TS + j;  // positions in the child's frontal
    const double v = Fc[tri_off(ri >> 6, rj >> 6) + (ri & 63) * TS + (rj & 63)];
    int pi = ep[i], pj = ep[j];
    if (pi < pj) {
      const int t = pi;
      pi = pj;
      pj = t;
    }
    Fp[tri_off(pi >> 6, pj >> 6) + (pi & 63) * TS + (pj & 63)] += v;
  }
}

}  // namespace tcg
