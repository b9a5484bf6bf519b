// nonlinear.cu — SURVEY §8(f) f4: nonlinear reluctivity nu(|B|) with Newton's method per
// implicit-Euler step (R25). Included by capi.cu after assembly.cu.
//
// Paper: "nonlinear behavior can be modeled as a simple extension" (§2); no law is
// given. Reading R25: Brauer law nu(b2) = k1 exp(k2 b2) + k3 (b2 = |B|^2) on the patches with
// nonzero parameters; the Newton iterate of one step solves
//     J(a_k) a_{k+1} = (Kt(a_k) - K(a_k)) a_k + (sigma/dt) M a^l + j^(l+1),
//     J = Kt + (sigma/dt) M,  Kt_jk = < (nu I + 2 nu' B B^T) curl w_k, curl w_j >,
// with the linear method's IETI-DP solve (the stepper's right-hand side gains the vector
// g = (Kt - K) a_k, DESIGN.md §5 "Newton"). Unlike the linear assembly (Kronecker products of
// 1D matrices, assembly.cu), the tangent matrix has a point-dependent 3x3 coefficient, so it is
// integrated entry by entry over the Gauss points of the two functions' common support:
//   k_nl_tab1d    1D tables at the Gauss points: weight, active B, D, B' values per direction
//   k_nl_quad     per Gauss point of every nonlinear patch: B = curl A_h, nu, nu',
//                 Nw = w (nu I + 2 nu' B B^T) (6 entries) and gq = w 2 nu' |B|^2 B (3 entries)
//   k_nl_g        g_a = sum_q gq(q) . curl w_a(q)  (= ((Kt - K) a)_a), scattered to aug order
//   k_nl_assemble the gauged, permuted tile-packed J of the nonlinear patches (padding
//                 rows/columns identity), overwriting k_assemble's linear tiles
//   k_nl_norms    per-block partial sums of |a - a_k|^2 and |a|^2 (Newton stopping rule)
// Quadrature as the linear assembly: p+1 Gauss points per direction per element (R8).
#include "common.cuh"
#include "device.h"

namespace tcg {

constexpr int NL_MAXP = 7;  // p + 1 <= 8 Gauss points (gauss_legendre)
constexpr int NL_NORM_BLOCKS = 148;

struct NlTab {
  const double* base;  // per direction d: nq[d] points x stride, from off[d]
  int64_t off[3];
  int nq[3];           // Gauss points per direction over the patch: el[d] * (p + 1)
  int stride;          // 1 + 3 (p + 1): weight, B[p+1], D[p+1] (p used), dB[p+1]
};

// one block per direction: the 1D Gauss-point tables of the patch box (all patches of a
// config share the shape; local coordinates [0, h_d])
__global__ void k_nl_tab1d(double* tab, NlTab T, Tables1D tb, int p) {
  const int d = blockIdx.x;
  const int q = p + 1, el = tb.el[d];
  const double h = tb.h[d];
  const int n = el + p;
  for (int qd = threadIdx.x; qd < T.nq[d]; qd += blockDim.x) {
    const int e = qd / q, g = qd % q;
    double gx, gw;
    gauss_legendre(q, g, gx, gw);
    const double a0 = h * e / el, b0 = h * (e + 1) / el;
    const double xl = 0.5 * (a0 + b0) + 0.5 * (b0 - a0) * gx;
    double tB[160], tD[160];
    bsplines_at(p, el, h, p, xl, tB);
    bsplines_at(p, el, h, p - 1, xl, tD);
    auto knot = [&](int i) -> double { return i <= p ? 0.0 : (i >= el + p ? h : h * (double)(i - p) / el); };
    double* o = tab + T.off[d] + (int64_t)qd * T.stride;
    o[0] = 0.5 * (b0 - a0) * gw;
    for (int k = 0; k <= p; ++k) {
      const int i = e + k;
      const double dm = (i >= 1) ? p / (knot(i + p) - knot(i)) * tD[i] : 0.0;                // D_{i-1}
      const double dp = (i <= n - 2) ? p / (knot(i + p + 1) - knot(i + 1)) * tD[i + 1] : 0.0;  // D_i
      o[1 + k] = tB[i];
      o[1 + q + k] = (k < p) ? dp : 0.0;
      o[1 + 2 * q + k] = dm - dp;
    }
  }
}

// 1D factor of kind (0 B, 1 D, 2 B') of function index i along d at point qd (0 off support)
__device__ __forceinline__ double nl_f1(const double* tab, const NlTab& T, int d, int kind, int i, int qd, int p) {
  const int q = p + 1;
  const int k = i - qd / q;
  if (k < 0 || k > (kind == 1 ? p - 1 : p)) return 0.0;
  return tab[T.off[d] + (int64_t)qd * T.stride + 1 + kind * q + k];
}

// Gauss-point range [lo, hi) along d of the support of index i (D-spline if dspl)
__device__ __forceinline__ void nl_support(int i, bool dspl, int p, int el, int& lo, int& hi) {
  const int e0 = max(0, dspl ? i - p + 1 : i - p), e1 = min(el - 1, i);
  lo = e0 * (p + 1);
  hi = (e1 + 1) * (p + 1);
}

// the two nonzero curl components of w_a, a = (c, i, j, k): component r[t], sign sg[t],
// kinds per direction kd[t][3] (0 B, 1 D, 2 B')
struct CurlTerms {
  int r[2];
  double sg[2];
  int kd[2][3];
};
__device__ __forceinline__ CurlTerms curl_terms(int c) {
  CurlTerms C;
  if (c == 0) {         // curl(D B B e_x) = (0, D B B', -D B' B)
    C.r[0] = 1; C.sg[0] = 1.0;  C.kd[0][0] = 1; C.kd[0][1] = 0; C.kd[0][2] = 2;
    C.r[1] = 2; C.sg[1] = -1.0; C.kd[1][0] = 1; C.kd[1][1] = 2; C.kd[1][2] = 0;
  } else if (c == 1) {  // curl(B D B e_y) = (-B D B', 0, B' D B)
    C.r[0] = 0; C.sg[0] = -1.0; C.kd[0][0] = 0; C.kd[0][1] = 1; C.kd[0][2] = 2;
    C.r[1] = 2; C.sg[1] = 1.0;  C.kd[1][0] = 2; C.kd[1][1] = 1; C.kd[1][2] = 0;
  } else {              // curl(B B D e_z) = (B B' D, -B' B D, 0)
    C.r[0] = 0; C.sg[0] = 1.0;  C.kd[0][0] = 0; C.kd[0][1] = 2; C.kd[0][2] = 1;
    C.r[1] = 1; C.sg[1] = -1.0; C.kd[1][0] = 2; C.kd[1][1] = 0; C.kd[1][2] = 1;
  }
  return C;
}

// index of the symmetric 3x3 entry (r, r') in the stored order 00 11 22 01 02 12
__device__ __forceinline__ int sym6(int r, int rr) {
  if (r == rr) return r;
  const int lo = min(r, rr), hi = max(r, rr);
  return lo == 0 ? (hi == 1 ? 3 : 4) : 5;
}

// Gauss-point coefficients of every nonlinear patch of the launching rank (grid.x = patches of
// nlist, grid.y * blockDim.x threads stride the points). Q layout per patch li: 9 planes of
// nqp doubles (Nw 00 11 22 01 02 12, gq x y z).
__global__ void __launch_bounds__(256) k_nl_quad(Geom G, NlTab T, const int* nlist, const double* __restrict__ a_loc,
                                                 const double* __restrict__ nlk, double* Q) {
  const int li = blockIdx.x, s = nlist[li];
  const int p = G.p, q = p + 1;
  const int nqx = T.nq[0], nqy = T.nq[1], nqz = T.nq[2];
  const int64_t nqp = (int64_t)nqx * nqy * nqz;
  const double* as = a_loc + (int64_t)s * G.nloc;
  const double k1 = nlk[3 * s], k2 = nlk[3 * s + 1], k3 = nlk[3 * s + 2];
  int off[3];
  off[0] = 0;
  off[1] = G.cdim[0][0] * G.cdim[0][1] * G.cdim[0][2];
  off[2] = off[1] + G.cdim[1][0] * G.cdim[1][1] * G.cdim[1][2];
  double* Qs = Q + (int64_t)li * 9 * nqp;
  for (int64_t w = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; w < nqp; w += (int64_t)gridDim.y * blockDim.x) {
    const int qx = (int)(w % nqx), qy = (int)((w / nqx) % nqy), qz = (int)(w / ((int64_t)nqx * nqy));
    const int e3[3] = {qx / q, qy / q, qz / q};
    const int qd[3] = {qx, qy, qz};
    const double* row[3];
    for (int d = 0; d < 3; ++d) row[d] = T.base + T.off[d] + (int64_t)qd[d] * T.stride;
    const double wt = row[0][0] * row[1][0] * row[2][0];
    double Bq[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < 3; ++c) {
      const int nk = (c == 2) ? p : q, nj = (c == 1) ? p : q, ni = (c == 0) ? p : q;
      const CurlTerms C = curl_terms(c);
      for (int kk = 0; kk < nk; ++kk)
        for (int jj = 0; jj < nj; ++jj)
          for (int ii = 0; ii < ni; ++ii) {
            const int i = e3[0] + ii, j = e3[1] + jj, k = e3[2] + kk;
            const double cf = as[off[c] + i + G.cdim[c][0] * (j + G.cdim[c][1] * k)];
            const int lk[3] = {ii, jj, kk};
            for (int t = 0; t < 2; ++t) {
              double v = C.sg[t];
              for (int d = 0; d < 3; ++d) v *= row[d][1 + C.kd[t][d] * q + lk[d]];
              Bq[C.r[t]] += cf * v;
            }
          }
    }
    const double b2 = Bq[0] * Bq[0] + Bq[1] * Bq[1] + Bq[2] * Bq[2];
    const double ex = exp(k2 * b2);
    const double nu = k1 * ex + k3, dnu2 = 2.0 * k1 * k2 * ex;  // nu, 2 dnu/d(b2)
    Qs[0 * nqp + w] = wt * (nu + dnu2 * Bq[0] * Bq[0]);
    Qs[1 * nqp + w] = wt * (nu + dnu2 * Bq[1] * Bq[1]);
    Qs[2 * nqp + w] = wt * (nu + dnu2 * Bq[2] * Bq[2]);
    Qs[3 * nqp + w] = wt * dnu2 * Bq[0] * Bq[1];
    Qs[4 * nqp + w] = wt * dnu2 * Bq[0] * Bq[2];
    Qs[5 * nqp + w] = wt * dnu2 * Bq[1] * Bq[2];
    Qs[6 * nqp + w] = wt * dnu2 * b2 * Bq[0];
    Qs[7 * nqp + w] = wt * dnu2 * b2 * Bq[1];
    Qs[8 * nqp + w] = wt * dnu2 * b2 * Bq[2];
  }
}

// g_a = sum_q gq(q) . curl w_a(q) for every local DOF of the nonlinear patches, written at
// the DOF's aug position (E DOFs dropped); grid.x = patches, threads stride the DOFs.
__global__ void __launch_bounds__(256) k_nl_g(DevPlan D, Geom G, NlTab T, const int* nlist, const double* __restrict__ Q,
                                              double* gvec) {
  extern __shared__ double tabs[];
  const int li = blockIdx.x, s = nlist[li];
  const int p = G.p;
  const int64_t tsz = T.off[2] + (int64_t)T.nq[2] * T.stride;
  for (int64_t i = threadIdx.x; i < tsz; i += blockDim.x) tabs[i] = T.base[i];
  __syncthreads();
  const int nqx = T.nq[0], nqy = T.nq[1];
  const int64_t nqp = (int64_t)nqx * nqy * T.nq[2];
  const double* Qs = Q + (int64_t)li * 9 * nqp;
  const int* l2a = D.loc2aug + (int64_t)s * G.nloc;
  double* gs = gvec + D.vec_off[s];
  for (int a = blockIdx.y * blockDim.x + threadIdx.x; a < G.nloc; a += gridDim.y * blockDim.x) {
    const int pos = l2a[a];
    if (pos < 0) continue;
    const LocalDof A = decode_local(G, a);
    const CurlTerms C = curl_terms(A.c);
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) nl_support(A.i[d], d == A.c, p, G.el[d], lo[d], hi[d]);
    double acc = 0.0;
    for (int qz = lo[2]; qz < hi[2]; ++qz)
      for (int qy = lo[1]; qy < hi[1]; ++qy) {
        double yz[2];
        for (int t = 0; t < 2; ++t)
          yz[t] = C.sg[t] * nl_f1(tabs, T, 1, C.kd[t][1], A.i[1], qy, p) * nl_f1(tabs, T, 2, C.kd[t][2], A.i[2], qz, p);
        for (int qx = lo[0]; qx < hi[0]; ++qx) {
          const int64_t w = qx + (int64_t)nqx * (qy + (int64_t)nqy * qz);
          for (int t = 0; t < 2; ++t)
            acc += yz[t] * nl_f1(tabs, T, 0, C.kd[t][0], A.i[0], qx, p) * Qs[(6 + C.r[t]) * nqp + w];
        }
      }
    gs[pos] = acc;
  }
}

// One CTA per 64x64 tile of the nonlinear patches' tile-packed J = Kt + (sigma/dt) M (the
// rank's nonlinear list nlist, tile prefix tstart over it); same layout and padding as
// k_assemble. Kt entry (a, b): sum over the Gauss points of the elements both functions are
// active on of curl w_a^T Nw curl w_b (each curl has two nonzero components, each a product
// of three 1D factors). Loops run element by element (the active-function offset i - e is
// fixed per element, no division or support test per point), Q = p + 1 points unrolled.
template <int P>
__global__ void __launch_bounds__(256) k_nl_assemble(DevPlan D, Tables1D tb, Geom G, NlTab T, double inv_dt,
                                                     const int* nlist, const int64_t* tstart, int nnl,
                                                     const double* __restrict__ Q) {
  constexpr int NQ = P + 1;
  extern __shared__ double tabs[];
  const int64_t tile = blockIdx.x;
  const int li = find_patch(tstart, nnl, tile);
  const int s = nlist[li];
  const int64_t tl = tile - tstart[li];
  int I = (int)((sqrt(8.0 * (double)tl + 1.0) - 1.0) * 0.5);
  while ((int64_t)I * (I + 1) / 2 > tl) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tl) ++I;
  const int J = (int)(tl - (int64_t)I * (I + 1) / 2);
  __shared__ T1 t1[3];
  if (threadIdx.x < 3) {
    const int d = threadIdx.x;
    t1[d].Mb = tb.base + tb.off_Mb[d];
    t1[d].Md = tb.base + tb.off_Md[d];
    t1[d].Kb = tb.base + tb.off_Kb[d];
    t1[d].C = tb.base + tb.off_C[d];
    t1[d].n = tb.el[d] + G.p;
  }
  const int64_t tsz = T.off[2] + (int64_t)T.nq[2] * T.stride;
  for (int64_t i = threadIdx.x; i < tsz; i += blockDim.x) tabs[i] = T.base[i];
  __syncthreads();
  const int nqx = T.nq[0], nqy = T.nq[1];
  const int64_t nqp = (int64_t)nqx * nqy * T.nq[2];
  const int st = T.stride;
  const double* Qs = Q + (int64_t)li * 9 * nqp;
  const double sg = D.sigma[s] * inv_dt;
  const int* aug = D.aug + D.aug_off[s];
  double* out = D.A + D.a_off[s] + tri_off(I, J);
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) {
    const int r = e / TS, c = e % TS;
    const int ga = aug[I * TS + r], gb = aug[J * TS + c];
    double v;
    if (ga < 0 || gb < 0) {
      v = (I == J && r == c) ? 1.0 : 0.0;
    } else {
      const LocalDof A = decode_local(G, ga), B = decode_local(G, gb);
      double Kl, M;
      kron_entry(t1, A, B, Kl, M);
      int e0[3], e1[3];
      bool empty = false;
      for (int d = 0; d < 3; ++d) {
        const int a0 = max(0, A.i[d] - (d == A.c ? P - 1 : P)), b0 = max(0, B.i[d] - (d == B.c ? P - 1 : P));
        e0[d] = max(a0, b0);
        e1[d] = min(min(A.i[d], B.i[d]), G.el[d] - 1);
        empty |= e0[d] > e1[d];
      }
      double K = 0.0;
      if (!empty) {
        const CurlTerms CA = curl_terms(A.c), CB = curl_terms(B.c);
        const double* Nq[2][2];
        for (int t = 0; t < 2; ++t)
          for (int u = 0; u < 2; ++u) Nq[t][u] = Qs + sym6(CA.r[t], CB.r[u]) * nqp;
        // table column of each term's factor along d: 1 + kind * NQ (+ active offset per element)
        int ka[2][3], kb[2][3];
        for (int t = 0; t < 2; ++t)
          for (int d = 0; d < 3; ++d) {
            ka[t][d] = 1 + CA.kd[t][d] * NQ;
            kb[t][d] = 1 + CB.kd[t][d] * NQ;
          }
        for (int ez = e0[2]; ez <= e1[2]; ++ez) {
          const int oaz = A.i[2] - ez, obz = B.i[2] - ez;
#pragma unroll
          for (int gz = 0; gz < NQ; ++gz) {
            const int qz = ez * NQ + gz;
            const double* rz = tabs + T.off[2] + (int64_t)qz * st;
            double za[2], zb[2];
            for (int t = 0; t < 2; ++t) {
              za[t] = CA.sg[t] * rz[ka[t][2] + oaz];
              zb[t] = CB.sg[t] * rz[kb[t][2] + obz];
            }
            for (int ey = e0[1]; ey <= e1[1]; ++ey) {
              const int oay = A.i[1] - ey, oby = B.i[1] - ey;
#pragma unroll
              for (int gy = 0; gy < NQ; ++gy) {
                const int qy = ey * NQ + gy;
                const double* ry = tabs + T.off[1] + (int64_t)qy * st;
                double ya[2], yb[2];
                for (int t = 0; t < 2; ++t) {
                  ya[t] = za[t] * ry[ka[t][1] + oay];
                  yb[t] = zb[t] * ry[kb[t][1] + oby];
                }
                const int64_t wrow = (int64_t)nqx * (qy + (int64_t)nqy * qz);
                for (int ex = e0[0]; ex <= e1[0]; ++ex) {
                  const int oax = A.i[0] - ex, obx = B.i[0] - ex;
#pragma unroll
                  for (int gx = 0; gx < NQ; ++gx) {
                    const int qx = ex * NQ + gx;
                    const double* rx = tabs + T.off[0] + (int64_t)qx * st;
                    const double fa0 = ya[0] * rx[ka[0][0] + oax], fa1 = ya[1] * rx[ka[1][0] + oax];
                    const double fb0 = yb[0] * rx[kb[0][0] + obx], fb1 = yb[1] * rx[kb[1][0] + obx];
                    const int64_t w = wrow + qx;
                    K += fa0 * (__ldg(Nq[0][0] + w) * fb0 + __ldg(Nq[0][1] + w) * fb1) +
                         fa1 * (__ldg(Nq[1][0] + w) * fb0 + __ldg(Nq[1][1] + w) * fb1);
                  }
                }
              }
            }
          }
        }
      }
      v = K + sg * M;
    }
    out[e] = v;
  }
}

// ---- element matrices (p <= 3): one CTA per element of a nonlinear patch computes the
// element tangent matrix Ke[a][b] = sum_q curl w_a^T Nw curl w_b over the element's (p+1)^3
// Gauss points with the functions' curl values and Nw staged in shared memory (lower triangle,
// local function order: component-major, then kk, jj, ii of the active functions); the tile
// kernel then sums Ke over the elements of each entry's common support (fixed element order).
template <int P>
struct NlElem {
  static constexpr int NQ = P + 1, NQ3 = NQ * NQ * NQ;
  static constexpr int NF1 = P * (P + 1) * (P + 1), NF = 3 * NF1;
  static constexpr size_t smem = sizeof(double) * ((size_t)NF * NQ3 * 2 + 6 * NQ3);
  // local index of a function (component c, element offsets oi, oj, ok along x, y, z)
  __device__ static int loc(int c, int oi, int oj, int ok) {
    const int n0 = (c == 0) ? P : P + 1, n1 = (c == 1) ? P : P + 1;
    return c * NF1 + oi + n0 * (oj + n1 * ok);
  }
};
template <int P>
__global__ void __launch_bounds__(256) k_nl_elem(Geom G, NlTab T, const int* nlist, const double* __restrict__ Q,
                                                 double* Kel) {
  using E = NlElem<P>;
  constexpr int NQ = E::NQ, NQ3 = E::NQ3, NF1 = E::NF1, NF = E::NF;
  extern __shared__ double sm[];
  double* Cv = sm;               // [NF][NQ3][2]: the two nonzero curl terms (signs included)
  double* Ns = sm + NF * NQ3 * 2;  // [6][NQ3]
  const int li = blockIdx.y;
  const int e = blockIdx.x, ne = G.el[0] * G.el[1] * G.el[2];
  const int ex = e % G.el[0], ey = (e / G.el[0]) % G.el[1], ez = e / (G.el[0] * G.el[1]);
  const int nqx = T.nq[0], nqy = T.nq[1];
  const int64_t nqp = (int64_t)nqx * nqy * T.nq[2];
  const double* Qs = Q + (int64_t)li * 9 * nqp;
  for (int i = threadIdx.x; i < 6 * NQ3; i += blockDim.x) {
    const int comp = i / NQ3, q = i % NQ3;
    const int gx = q % NQ, gy = (q / NQ) % NQ, gz = q / (NQ * NQ);
    const int64_t w = (ex * NQ + gx) + (int64_t)nqx * ((ey * NQ + gy) + (int64_t)nqy * (ez * NQ + gz));
    Ns[i] = Qs[comp * nqp + w];
  }
  for (int i = threadIdx.x; i < NF * NQ3; i += blockDim.x) {
    const int f = i / NQ3, q = i % NQ3;
    const int c = f / NF1, lf = f % NF1;
    const int n0 = (c == 0) ? P : P + 1, n1 = (c == 1) ? P : P + 1;
    const int oi = lf % n0, oj = (lf / n0) % n1, ok = lf / (n0 * n1);
    const int gx = q % NQ, gy = (q / NQ) % NQ, gz = q / (NQ * NQ);
    const double* rx = T.base + T.off[0] + (int64_t)(ex * NQ + gx) * T.stride + 1;
    const double* ry = T.base + T.off[1] + (int64_t)(ey * NQ + gy) * T.stride + 1;
    const double* rz = T.base + T.off[2] + (int64_t)(ez * NQ + gz) * T.stride + 1;
    const CurlTerms C = curl_terms(c);
    for (int t = 0; t < 2; ++t)
      Cv[(f * NQ3 + q) * 2 + t] = C.sg[t] * rx[C.kd[t][0] * NQ + oi] * ry[C.kd[t][1] * NQ + oj] * rz[C.kd[t][2] * NQ + ok];
  }
  __syncthreads();
  double* K = Kel + ((int64_t)li * ne + e) * NF * NF;
  for (int idx = threadIdx.x; idx < NF * NF; idx += blockDim.x) {
    const int a = idx / NF, b = idx % NF;
    if (b > a) continue;
    const CurlTerms CA = curl_terms(a / NF1), CB = curl_terms(b / NF1);
    const double* n00 = Ns + sym6(CA.r[0], CB.r[0]) * NQ3;
    const double* n01 = Ns + sym6(CA.r[0], CB.r[1]) * NQ3;
    const double* n10 = Ns + sym6(CA.r[1], CB.r[0]) * NQ3;
    const double* n11 = Ns + sym6(CA.r[1], CB.r[1]) * NQ3;
    const double* ca = Cv + a * NQ3 * 2;
    const double* cb = Cv + b * NQ3 * 2;
    double acc = 0.0;
#pragma unroll 4
    for (int q = 0; q < NQ3; ++q) {
      const double a0 = ca[2 * q], a1 = ca[2 * q + 1], b0 = cb[2 * q], b1 = cb[2 * q + 1];
      acc += a0 * (n00[q] * b0 + n01[q] * b1) + a1 * (n10[q] * b0 + n11[q] * b1);
    }
    K[a * NF + b] = acc;
  }
}

// the tile-packed J of the nonlinear patches from the element matrices: entry (a, b) = sum over
// the elements both functions are active on (z, y, x order) of Ke + (sigma/dt) M_ab
template <int P>
__global__ void __launch_bounds__(256) k_nl_gather(DevPlan D, Tables1D tb, Geom G, double inv_dt, const int* nlist,
                                                   const int64_t* tstart, int nnl, const double* __restrict__ Kel) {
  using E = NlElem<P>;
  constexpr int NF = E::NF;
  const int64_t tile = blockIdx.x;
  const int li = find_patch(tstart, nnl, tile);
  const int s = nlist[li];
  const int64_t tl = tile - tstart[li];
  int I = (int)((sqrt(8.0 * (double)tl + 1.0) - 1.0) * 0.5);
  while ((int64_t)I * (I + 1) / 2 > tl) --I;
  while ((int64_t)(I + 1) * (I + 2) / 2 <= tl) ++I;
  const int J = (int)(tl - (int64_t)I * (I + 1) / 2);
  __shared__ T1 t1[3];
  if (threadIdx.x < 3) {
    const int d = threadIdx.x;
    t1[d].Mb = tb.base + tb.off_Mb[d];
    t1[d].Md = tb.base + tb.off_Md[d];
    t1[d].Kb = tb.base + tb.off_Kb[d];
    t1[d].C = tb.base + tb.off_C[d];
    t1[d].n = tb.el[d] + G.p;
  }
  __syncthreads();
  const int ne = G.el[0] * G.el[1] * G.el[2];
  const double* Ks = Kel + (int64_t)li * ne * NF * NF;
  const double sg = D.sigma[s] * inv_dt;
  const int* aug = D.aug + D.aug_off[s];
  double* out = D.A + D.a_off[s] + tri_off(I, J);
  for (int e = threadIdx.x; e < TSZ; e += blockDim.x) {
    const int r = e / TS, c = e % TS;
    const int ga = aug[I * TS + r], gb = aug[J * TS + c];
    double v;
    if (ga < 0 || gb < 0) {
      v = (I == J && r == c) ? 1.0 : 0.0;
    } else {
      const LocalDof A = decode_local(G, ga), B = decode_local(G, gb);
      double Kl, M;
      kron_entry(t1, A, B, Kl, M);
      int e0[3], e1[3];
      bool empty = false;
      for (int d = 0; d < 3; ++d) {
        const int a0 = max(0, A.i[d] - (d == A.c ? P - 1 : P)), b0 = max(0, B.i[d] - (d == B.c ? P - 1 : P));
        e0[d] = max(a0, b0);
        e1[d] = min(min(A.i[d], B.i[d]), G.el[d] - 1);
        empty |= e0[d] > e1[d];
      }
      double K = 0.0;
      if (!empty)
        for (int ez = e0[2]; ez <= e1[2]; ++ez)
          for (int ey = e0[1]; ey <= e1[1]; ++ey)
            for (int ex = e0[0]; ex <= e1[0]; ++ex) {
              const int la = E::loc(A.c, A.i[0] - ex, A.i[1] - ey, A.i[2] - ez);
              const int lb = E::loc(B.c, B.i[0] - ex, B.i[1] - ey, B.i[2] - ez);
              const int el = ex + G.el[0] * (ey + G.el[1] * ez);
              K += __ldg(Ks + (int64_t)el * NF * NF + (int64_t)max(la, lb) * NF + min(la, lb));
            }
      v = K + sg * M;
    }
    out[e] = v;
  }
}

// host-side dispatch on the spline degree (the Gauss-point loops unroll)
// p <= 3: element matrices (Kel: nnl x elements x NF^2 doubles) then the tile gather; else the
// per-entry Gauss-point kernel
inline size_t nl_elem_doubles(int p, int nel) {
  if (p < 1 || p > 3) return 0;
  const size_t nf = 3 * (size_t)p * (p + 1) * (p + 1);
  return (size_t)nel * nf * nf;
}
inline void launch_nl_assemble(int p, unsigned grid, size_t smem, cudaStream_t st, const DevPlan& D, const Tables1D& tb,
                               const Geom& G, const NlTab& T, double inv_dt, const int* nlist, const int64_t* tstart,
                               int nnl, const double* Q, double* Kel = nullptr) {
  if (Kel && p >= 1 && p <= 3) {
    const unsigned ne = (unsigned)(G.el[0] * G.el[1] * G.el[2]);
    switch (p) {
#define NLE(PP)                                                                                  \
  case PP:                                                                                       \
    k_nl_elem<PP><<<dim3(ne, (unsigned)nnl), 256, NlElem<PP>::smem, st>>>(G, T, nlist, Q, Kel);  \
    k_nl_gather<PP><<<grid, 256, 0, st>>>(D, tb, G, inv_dt, nlist, tstart, nnl, Kel);            \
    break;
      NLE(1) NLE(2) NLE(3)
#undef NLE
      default: break;
    }
    return;
  }
  switch (p) {
#define NLA(PP) \
  case PP: k_nl_assemble<PP><<<grid, 256, smem, st>>>(D, tb, G, T, inv_dt, nlist, tstart, nnl, Q); break;
    NLA(1) NLA(2) NLA(3) NLA(4) NLA(5) NLA(6) NLA(7)
#undef NLA
    default: break;
  }
}
inline cudaError_t nl_assemble_smem(size_t smem) {
  const void* fs[7] = {(const void*)k_nl_assemble<1>, (const void*)k_nl_assemble<2>, (const void*)k_nl_assemble<3>,
                       (const void*)k_nl_assemble<4>, (const void*)k_nl_assemble<5>, (const void*)k_nl_assemble<6>,
                       (const void*)k_nl_assemble<7>};
  for (const void* f : fs) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const void* ef[3] = {(const void*)k_nl_elem<1>, (const void*)k_nl_elem<2>, (const void*)k_nl_elem<3>};
  const size_t es[3] = {NlElem<1>::smem, NlElem<2>::smem, NlElem<3>::smem};
  for (int i = 0; i < 3; ++i) {
    cudaError_t e = cudaFuncSetAttribute(ef[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)es[i]);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// per-block partial sums (fixed order) of |a - a_k|^2 and |a|^2 over the owned patches'
// local vectors (global layout npatch x nloc)
__global__ void __launch_bounds__(256) k_nl_norms(const double* __restrict__ a, const double* __restrict__ ak,
                                                  const int* owner, int me, int nloc, int64_t n, double* part) {
  __shared__ double s0[256], s1[256];
  double x0 = 0.0, x1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (owner[i / nloc] != me) continue;
    const double d = a[i] - ak[i];
    x0 += d * d;
    x1 += a[i] * a[i];
  }
  s0[threadIdx.x] = x0;
  s1[threadIdx.x] = x1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0[0];
    part[2 * blockIdx.x + 1] = s1[0];
  }
}

}  // namespace tcg
