// assembly.cu — step a of the hot path: per-patch assembly of W^_s = nu_s K_s + (sigma_s/dt) M_s
// and of the load j_S,s, written directly as gauged, permuted, tile-packed dense matrices.
//
// Paper: (K_i)_jk = <nu curl w_k, curl w_j>, (M_C)_jk = <sigma w_k, w_j>, (j_i)_j = <J, w_j>
// (P:L83-87); W = M + dt K, used scaled as W^ = K + M/dt (R7).
// Design (DESIGN.md §5 "assembly"): on an affine box patch the Gauss-quadrature integrals
// factor into 1D integrals, so K and M are sums of Kronecker products of four 1D matrices
// Mb=[int B_i B_j], Md=[int D_i D_j], Kb=[int B_i' B_j'], C=[int D_i B_j'] per direction
// (SURVEY Appendix B). The 1D matrices are computed here by Gauss quadrature (p+1 points
// per element, R8) from Cox-de Boor B-splines and Curry-Schoenberg D-splines
// (R9); every entry of the gauged tile is then generated from them. The padded
// rows/columns of each tile block carry an identity diagonal.
#include "common.cuh"
#include "device.h"

namespace tcg {

// ---------------------------------------------------------------------------------------
// 1D tables
// ---------------------------------------------------------------------------------------

// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on P_q.
__device__ void gauss_legendre(int q, int i, double& x, double& w) {
  double z = cos(M_PI * (i + 0.75) / (q + 0.5));
  double dp = 1.0;
  for (int it = 0; it < 100; ++it) {
    double p0 = 1.0, p1 = 0.0;
    for (int j = 1; j <= q; ++j) {
      double p2 = p1;
      p1 = p0;
      p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
    }
    dp = q * (z * p0 - p1) / (z * z - 1.0);
    double dz = p0 / dp;
    z -= dz;
    if (fabs(dz) < 1e-16) break;
  }
  {  // derivative at the converged node
    double p0 = 1.0, p1 = 0.0;
    for (int j = 1; j <= q; ++j) {
      double p2 = p1;
      p1 = p0;
      p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
    }
    dp = q * (z * p0 - p1) / (z * z - 1.0);
  }
  x = -z;  // ascending order
  w = 2.0 / ((1.0 - z * z) * dp * dp);
}

// All B-splines of degree deg on the open uniform knot vector (p, el, [0,h]) at x, by the
// Cox-de Boor recursion (triangular scheme). Knots t_i, i=0..el+2p. Output nb = el+p-(p-deg).
__device__ void bsplines_at(int p, int el, double h, int deg, double x, double* out /* >= el+2p */) {
  const int nk = el + 2 * p + 1;  // number of knots
  auto knot = [&](int i) -> double {
    if (i <= p) return 0.0;
    if (i >= el + p) return h;
    return h * (double)(i - p) / (double)el;
  };
  // degree 0 on the half-open spans
  for (int i = 0; i < nk - 1; ++i) out[i] = (knot(i) <= x && x < knot(i + 1)) ? 1.0 : 0.0;
  for (int k = 1; k <= deg; ++k) {
    for (int i = 0; i < nk - 1 - k; ++i) {
      double v = 0.0;
      double d1 = knot(i + k) - knot(i);
      if (d1 > 0) v += (x - knot(i)) / d1 * out[i];
      double d2 = knot(i + k + 1) - knot(i + 1);
      if (d2 > 0) v += (knot(i + k + 1) - x) / d2 * out[i + 1];
      out[i] = v;
    }
  }
}

// One block per direction d. Writes Mb, Md, Kb, C, oneD and per-patch-index source
// integrals sD, cB, sB of sin(omega x), cos(omega x) (omega = pi for the BASELINE source and
// the homogeneous MMS, 1 for the paper's solution; see device.h Tables1D for the layout).
__global__ void k_tables1d(Tables1D tb, int p, double omega) {
  const int d = blockIdx.x;
  const int el = tb.el[d], n = el + p, q = p + 1;
  const double h = tb.h[d];
  extern __shared__ double sm[];
  double* gx = sm;                     // q nodes (element-local physical later)
  double* gw = gx + q;                 // q weights
  double* Bv = gw + q;                 // [el*q][n]
  double* Dv = Bv + el * q * n;        // [el*q][n-1]
  double* dBv = Dv + el * q * (n - 1); // [el*q][n]
  double* Xp = dBv + el * q * n;       // [el*q] local x
  double* Wp = Xp + el * q;            // [el*q] weights
  if (threadIdx.x < q) gauss_legendre(q, threadIdx.x, gx[threadIdx.x], gw[threadIdx.x]);
  __syncthreads();
  for (int eg = threadIdx.x; eg < el * q; eg += blockDim.x) {
    int e = eg / q, g = eg % q;
    double a = h * e / el, b = h * (e + 1) / el;
    double x = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
    Xp[eg] = x;
    Wp[eg] = 0.5 * (b - a) * gw[g];
    double tmpB[160], tmpD[160];
    bsplines_at(p, el, h, p, x, tmpB);
    bsplines_at(p, el, h, p - 1, x, tmpD);
    auto knot = [&](int i) -> double {
      if (i <= p) return 0.0;
      if (i >= el + p) return h;
      return h * (double)(i - p) / (double)el;
    };
    // Curry-Schoenberg D_i = p/(t_{i+p+1}-t_{i+1}) B_{i+1,p-1}
    for (int i = 0; i < n - 1; ++i) Dv[eg * (n - 1) + i] = p / (knot(i + p + 1) - knot(i + 1)) * tmpD[i + 1];
    for (int i = 0; i < n; ++i) {
      Bv[eg * n + i] = tmpB[i];
      double dm = (i >= 1) ? Dv[eg * (n - 1) + i - 1] : 0.0;
      double dp = (i <= n - 2) ? Dv[eg * (n - 1) + i] : 0.0;
      dBv[eg * n + i] = dm - dp;  // B_i' = D_{i-1} - D_i
    }
  }
  __syncthreads();
  const int ne = el * q;
  double* Mb = tb.base + tb.off_Mb[d];
  double* Md = tb.base + tb.off_Md[d];
  double* Kb = tb.base + tb.off_Kb[d];
  double* Cm = tb.base + tb.off_C[d];
  double* oneD = tb.base + tb.off_oneD[d];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx % n;
    double sm_b = 0, sk_b = 0;
    for (int eg = 0; eg < ne; ++eg) {
      sm_b += Wp[eg] * Bv[eg * n + i] * Bv[eg * n + j];
      sk_b += Wp[eg] * dBv[eg * n + i] * dBv[eg * n + j];
    }
    Mb[idx] = sm_b;
    Kb[idx] = sk_b;
  }
  for (int idx = threadIdx.x; idx < (n - 1) * (n - 1); idx += blockDim.x) {
    int i = idx / (n - 1), j = idx % (n - 1);
    double s = 0;
    for (int eg = 0; eg < ne; ++eg) s += Wp[eg] * Dv[eg * (n - 1) + i] * Dv[eg * (n - 1) + j];
    Md[idx] = s;
  }
  for (int idx = threadIdx.x; idx < (n - 1) * n; idx += blockDim.x) {
    int i = idx / n, j = idx % n;
    double s = 0;
    for (int eg = 0; eg < ne; ++eg) s += Wp[eg] * Dv[eg * (n - 1) + i] * dBv[eg * n + j];
    Cm[idx] = s;
  }
  for (int i = threadIdx.x; i < n - 1; i += blockDim.x) {
    double s = 0;
    for (int eg = 0; eg < ne; ++eg) s += Wp[eg] * Dv[eg * (n - 1) + i];
    oneD[i] = s;
  }
  // source integrals per patch index along d (physical x = lo + q*h + xloc)
  for (int idx = threadIdx.x; idx < tb.P[d] * n; idx += blockDim.x) {
    int qq = idx / n, i = idx % n;
    double x0 = tb.lo[d] + qq * h;
    double ssD = 0, scB = 0, ssB = 0;
    for (int eg = 0; eg < ne; ++eg) {
      double x = x0 + Xp[eg];
      double sx = sin(omega * x), cx = cos(omega * x);
      if (i < n - 1) ssD += Wp[eg] * sx * Dv[eg * (n - 1) + i];
      scB += Wp[eg] * cx * Bv[eg * n + i];
      ssB += Wp[eg] * sx * Bv[eg * n + i];
    }
    if (i < n - 1) tb.base[tb.off_sD[d] + qq * (n - 1) + i] = ssD;
    tb.base[tb.off_cB[d] + qq * n + i] = scB;
    tb.base[tb.off_sB[d] + qq * n + i] = ssB;
  }
}

// ---------------------------------------------------------------------------------------
// Kronecker entry generator
// ---------------------------------------------------------------------------------------

struct LocalDof {
  int c, i[3];
};

__device__ __forceinline__ LocalDof decode_local(const Geom& G, int a) {
  LocalDof r;
  int c = 0;
  for (;;) {
    int sz = G.cdim[c][0] * G.cdim[c][1] * G.cdim[c][2];
    if (a < sz) break;
    a -= sz;
    ++c;
  }
  r.c = c;
  r.i[0] = a % G.cdim[c][0];
  r.i[1] = (a / G.cdim[c][0]) % G.cdim[c][1];
  r.i[2] = a / (G.cdim[c][0] * G.cdim[c][1]);
  return r;
}

struct T1 {
  const double *Mb, *Md, *Kb, *C;
  int n;
  __device__ double mb(int i, int j) const { return Mb[i * n + j]; }
  __device__ double md(int i, int j) const { return Md[i * (n - 1) + j]; }
  __device__ double kb(int i, int j) const { return Kb[i * n + j]; }
  __device__ double cc(int i, int j) const { return C[i * n + j]; }  // int D_i B_j'
};

// nu-free stiffness K(a,b) and sigma-free mass M(a,b) of the box patch (Appendix B forms).
__device__ void kron_entry(const T1* t, const LocalDof& A, const LocalDof& B, double& K, double& M) {
  const int* a = A.i;
  const int* b = B.i;
  const T1 &X = t[0], &Y = t[1], &Z = t[2];
  K = 0.0;
  M = 0.0;
  if (A.c == B.c) {
    if (A.c == 0) {
      double md = X.md(a[0], b[0]);
      K = md * (Y.mb(a[1], b[1]) * Z.kb(a[2], b[2]) + Y.kb(a[1], b[1]) * Z.mb(a[2], b[2]));
      M = md * Y.mb(a[1], b[1]) * Z.mb(a[2], b[2]);
    } else if (A.c == 1) {
      double md = Y.md(a[1], b[1]);
      K = md * (X.kb(a[0], b[0]) * Z.mb(a[2], b[2]) + X.mb(a[0], b[0]) * Z.kb(a[2], b[2]));
      M = md * X.mb(a[0], b[0]) * Z.mb(a[2], b[2]);
    } else {
      double md = Z.md(a[2], b[2]);
      K = md * (X.mb(a[0], b[0]) * Y.kb(a[1], b[1]) + X.kb(a[0], b[0]) * Y.mb(a[1], b[1]));
      M = md * X.mb(a[0], b[0]) * Y.mb(a[1], b[1]);
    }
    return;
  }
  // off-diagonal component blocks (K only): K_xy = -C (x) C^T (x) Mb etc.
  if (A.c == 0 && B.c == 1) K = -X.cc(a[0], b[0]) * Y.cc(b[1], a[1]) * Z.mb(a[2], b[2]);
  else if (A.c == 1 && B.c == 0) K = -X.cc(b[0], a[0]) * Y.cc(a[1], b[1]) * Z.mb(b[2], a[2]);
  else if (A.c == 0 && B.c == 2) K = -X.cc(a[0], b[0]) * Y.mb(a[1], b[1]) * Z.cc(b[2], a[2]);
  else if (A.c == 2 && B.c == 0) K = -X.cc(b[0], a[0]) * Y.mb(b[1], a[1]) * Z.cc(a[2], b[2]);
  else if (A.c == 1 && B.c == 2) K = -X.mb(a[0], b[0]) * Y.cc(a[1], b[1]) * Z.cc(b[2], a[2]);
  else /* 2,1 */ K = -X.mb(b[0], a[0]) * Y.cc(b[1], a[1]) * Z.cc(a[2], b[2]);
}

__device__ __forceinline__ int find_patch(const int64_t* start, int P, int64_t x) {
  int lo = 0, hi = P;  // start[lo] <= x < start[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (start[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// One CTA per 64x64 tile of the tile-packed lower augmented matrices [i|b|p] of the
// launching rank's patches (plist, tile prefix tstart over plist).
__global__ void __launch_bounds__(256) k_assemble(DevPlan D, Tables1D tb, Geom G, double inv_dt, const int* plist,
                                                  const int64_t* tstart, int nlist) {
  const int64_t tile = blockIdx.x;
  const int li = find_patch(tstart, nlist, tile);
  const int s = plist[li];
  const int64_t tl = tile - tstart[li];
  int I = (int)((sqrt(8.0 * (double)tl + 1.0) - 1.0) * 0.5);
  while ((int64_t)I * (I + 1) / 2 > tl) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tl) ++I;
  const int J = (int)(tl - (int64_t)I * (I + 1) / 2);
  __shared__ T1 t[3];
  if (threadIdx.x < 3) {
    int d = threadIdx.x;
    t[d].Mb = tb.base + tb.off_Mb[d];
    t[d].Md = tb.base + tb.off_Md[d];
    t[d].Kb = tb.base + tb.off_Kb[d];
    t[d].C = tb.base + tb.off_C[d];
    t[d].n = tb.el[d] + G.p;
  }
  __syncthreads();
  const double nu = D.nu[s], sg = D.sigma[s] * inv_dt;
  const int* aug = D.aug + D.aug_off[s];
  double* out = D.A + D.a_off[s] + tri_off(I, J);
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) {
    const int r = e / TS, c = e % TS;
    const int ga = aug[I * TS + r], gb = aug[J * TS + c];
    double v;
    if (ga < 0 || gb < 0) {
      v = (I == J && r == c) ? 1.0 : 0.0;
    } else {
      LocalDof A = decode_local(G, ga), B = decode_local(G, gb);
      double K, M;
      kron_entry(t, A, B, K, M);
      v = nu * K + sg * M;
    }
    out[e] = v;
  }
}

// rho-scaling weights (R5): for multiplier k joining s+ and s-,
// w+ = rho(s-)/(rho(s+)+rho(s-)), w- = rho(s+)/(rho(s+)+rho(s-)), rho = diagonal of W^.
// k_rho_capture copies the two diagonal entries from the assembled tiles into rho[2k], rho[2k+1]
// (only the sides whose patch has only[s] != 0, if only is given: the Newton re-assembly of the
// nonlinear patches, nonlinear.cu); k_rho_weights forms the weights from them.
__global__ void k_rho_capture(DevPlan D, double* rho, const unsigned char* only) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= D.m) return;
  for (int side = 0; side < 2; ++side) {
    int s = side == 0 ? D.lam_patch_p[k] : D.lam_patch_m[k];
    if (only && !only[s]) continue;
    int pos = D.Ti[s] * TS + (side == 0 ? D.lam_pos_p[k] : D.lam_pos_m[k]);
    int Itile = pos / TS, rr = pos % TS;
    rho[2 * k + side] = D.Ar[D.owner[s]][D.a_off[s] + tri_off(Itile, Itile) + rr * TS + rr];
  }
}

__global__ void k_rho_weights(DevPlan D, int scaling, const double* rho) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= D.m) return;
  if (scaling == 0) {
    D.wplus[k] = 1.0;
    D.wminus[k] = 1.0;
    return;
  }
  const double rp = rho[2 * k], rm = rho[2 * k + 1];
  D.wplus[k] = rm / (rp + rm);
  D.wminus[k] = rp / (rp + rm);
}

// Per b position: a_own = weight of this side, a_part = -(weight of the other side), so that
// sign * (w+ y[+] - w- y[-]) = a_own y[own] + a_part y[partner].
__global__ void k_btables(DevPlan D, int64_t nbtot) {
  int64_t bb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (bb >= nbtot) return;
  const int k = D.b_lam[bb];
  const bool plus = D.b_sign[bb] > 0;
  D.b_aown[bb] = plus ? D.wplus[k] : D.wminus[k];
  D.b_apart[bb] = plus ? -D.wminus[k] : -D.wplus[k];
}

// Spatial load j_S,s = <S, w> in aug order (r and p positions; padding 0), from the
// separable 1D source integrals. kind 1: S = (pi sx cy sz, -pi cx sy sz, 0);
// kind 2: S = (sy sz, sx sz, sx sy); kind 3 (tables with omega = 1): S = (sx cy cz, -2 cx sy cz, cx cy sz).
__device__ double load_entry(const Tables1D& tb, const Geom& G, int kind, int pidx[3], const LocalDof& A) {
  if (kind == 0) return 0.0;
  const int* i = A.i;
  auto sD = [&](int d, int ii) { return tb.base[tb.off_sD[d] + pidx[d] * (tb.el[d] + G.p - 1) + ii]; };
  auto cB = [&](int d, int ii) { return tb.base[tb.off_cB[d] + pidx[d] * (tb.el[d] + G.p) + ii]; };
  auto sB = [&](int d, int ii) { return tb.base[tb.off_sB[d] + pidx[d] * (tb.el[d] + G.p) + ii]; };
  auto oD = [&](int d, int ii) { return tb.base[tb.off_oneD[d] + ii]; };
  if (kind == 1) {
    if (A.c == 0) return M_PI * sD(0, i[0]) * cB(1, i[1]) * sB(2, i[2]);
    if (A.c == 1) return -M_PI * cB(0, i[0]) * sD(1, i[1]) * sB(2, i[2]);
    return 0.0;
  }
  if (kind == 3) {
    if (A.c == 0) return sD(0, i[0]) * cB(1, i[1]) * cB(2, i[2]);
    if (A.c == 1) return -2.0 * cB(0, i[0]) * sD(1, i[1]) * cB(2, i[2]);
    return cB(0, i[0]) * cB(1, i[1]) * sD(2, i[2]);
  }
  if (A.c == 0) return oD(0, i[0]) * sB(1, i[1]) * sB(2, i[2]);
  if (A.c == 1) return sB(0, i[0]) * oD(1, i[1]) * sB(2, i[2]);
  return sB(0, i[0]) * sB(1, i[1]) * oD(2, i[2]);
}

// One CTA per owned patch: JS[vec_off[s] + pos] for every aug position.
__global__ void k_load_vector(DevPlan D, Tables1D tb, Geom G, int kind, double* JS, const int* plist) {
  const int s = plist[blockIdx.x];
  int pidx[3] = {s % G.P[0], (s / G.P[0]) % G.P[1], s / (G.P[0] * G.P[1])};
  const int* aug = D.aug + D.aug_off[s];
  const int R = D.T[s] * TS;
  for (int pos = threadIdx.x; pos < R; pos += blockDim.x) {
    int a = aug[pos];
    JS[D.vec_off[s] + pos] = (a < 0) ? 0.0 : load_entry(tb, G, kind, pidx, decode_local(G, a));
  }
}

}  // namespace tcg
