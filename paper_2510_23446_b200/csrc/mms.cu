// mms.cu — the paper's own experiment on the GPU (§4).
//
// Prescribed solution A = amp e^-t S(x), S = (sin x cos y cos z, -2 cos x sin y cos z,
// cos x cos y sin z), so B = curl A = amp e^-t (-3 cos x sin y sin z, 0,
// 3 sin x sin y cos z), E_C = -dA/dt = A, and J = nu curl curl A + sigma dA/dt =
// amp e^-t (3 nu - sigma) S (curl curl S = 3 S). "Homogenized boundary, source and initial
// terms" (R21): the Dirichlet DOFs a_D(t) = amp e^-t (Pi_h S)_D and the
// initial coefficients a(0) = amp Pi_h S, Pi_h the commuting spline projection (Greville
// interpolation in the B-spline directions, histopolation on the Greville intervals in the
// D-spline direction). S is separable, so Pi_h S is a product of 1D projections: per
// direction and patch index, c_cos = I^-1 [cos(xi_i)] (B coefficients) and
// c_sin = H^-1 [int_{xi_a}^{xi_a+1} sin] (D coefficients).
// The lifting enters the right-hand side as f_r - W_rD a_D, f_p - W_pD a_D; since
// a_D(t) = e^-t a_D(0) and J ~ e^-t, both fold into the load template
//   JS_s = (3 nu_s - sigma_s) j_S,s - W^_s,(r,p)D (Pi_h S)_D,   phi(t) = amp e^-t,
// and the stepper writes a_D(t) into the local coefficients after every step (mass term of
// the next step, output). Errors per step by (p+1)-point Gauss quadrature:
//   e_B = ||B(t) - curl A_h||^2_{L2(Omega)},  e_E = ||E_C(t) + (A_h - A_h,prev)/dt||^2_{L2(Omega_C)},
// eps_B^2 = max e_B + dt sum e_B, eps_E^2 = dt sum e_E (running max / sums on the device).
#include "common.cuh"
#include "device.h"

namespace tcg {

constexpr int kProjMaxN = 72;  // B-splines per patch and direction supported by k_proj1d

// Greville abscissa i of the degree-p B-splines on the patch knot vector (local [0, h]).
__device__ double greville_local(int p, int el, double h, int i) {
  double s = 0.0;
  for (int q = i + 1; q <= i + p; ++q) s += (q <= p) ? 0.0 : (q >= el + p ? h : h * (double)(q - p) / (double)el);
  return s / p;
}

// Dense solve A x = b (n x n, row stride n) by Gaussian elimination without pivoting (the
// B-spline collocation and histopolation matrices are totally positive: no pivoting needed).
__device__ void solve_np(double* A, double* b, int n) {
  for (int k = 0; k < n; ++k) {
    const double piv = A[k * n + k];
    for (int i = k + 1; i < n; ++i) {
      const double f = A[i * n + k] / piv;
      if (f == 0.0) continue;
      for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double v = b[i];
    for (int j = i + 1; j < n; ++j) v -= A[i * n + j] * b[j];
    b[i] = v / A[i * n + i];
  }
}

// One block (thread 0 does the arithmetic) per (direction d, patch index q): the 1D
// projection coefficients of cos (Greville interpolation, n values) and of sin
// (histopolation, n-1 values) on the patch's knot vector. out[off_cos[d] + q*n + i],
// out[off_sin[d] + q*(n-1) + i].
__global__ void k_proj1d(Tables1D tb, int p, const int64_t* __restrict__ off_cos, const int64_t* __restrict__ off_sin,
                         double* out) {
  const int d = blockIdx.y, q = blockIdx.x;
  if (q >= tb.P[d] || threadIdx.x != 0) return;
  const int el = tb.el[d], n = el + p;
  const double h = tb.h[d], x0 = tb.lo[d] + q * h;
  extern __shared__ double sm[];
  double* Amat = sm;            // n x n
  double* rhs = Amat + n * n;   // n
  double tmp[160];
  // Greville interpolation of cos: I[i][j] = B_j(xi_i), rhs_i = cos(x0 + xi_i)
  for (int i = 0; i < n; ++i) {
    const double xi = greville_local(p, el, h, i);
    if (xi >= h) {
      for (int j = 0; j < n; ++j) tmp[j] = (j == n - 1) ? 1.0 : 0.0;  // closed right end
    } else {
      bsplines_at(p, el, h, p, xi, tmp);
    }
    for (int j = 0; j < n; ++j) Amat[i * n + j] = tmp[j];
    rhs[i] = cos(x0 + xi);
  }
  solve_np(Amat, rhs, n);
  for (int i = 0; i < n; ++i) out[off_cos[d] + (int64_t)q * n + i] = rhs[i];
  // histopolation of sin: H[a][j] = int_{xi_a}^{xi_a+1} D_j, rhs_a = int sin(x0 + x), both by
  // (p+3)-point Gauss on every knot span inside the interval
  const int m = n - 1, nq = p + 3;
  double gx[8], gw[8];
  for (int g = 0; g < nq; ++g) gauss_legendre(nq, g, gx[g], gw[g]);
  for (int a = 0; a < m; ++a) {
    for (int j = 0; j < m; ++j) Amat[a * m + j] = 0.0;
    rhs[a] = 0.0;
    const double lo = greville_local(p, el, h, a), hi = greville_local(p, el, h, a + 1);
    // cut points: the interval ends and the interior knots between them
    double cuts[170];
    int nc = 0;
    cuts[nc++] = lo;
    for (int e = 1; e < el; ++e) {
      const double k = h * (double)e / (double)el;
      if (k > lo && k < hi) cuts[nc++] = k;
    }
    cuts[nc++] = hi;
    for (int c = 0; c + 1 < nc; ++c) {
      const double u = cuts[c], v = cuts[c + 1];
      for (int g = 0; g < nq; ++g) {
        const double x = 0.5 * (u + v) + 0.5 * (v - u) * gx[g], w = 0.5 * (v - u) * gw[g];
        bsplines_at(p, el, h, p - 1, x, tmp);
        for (int j = 0; j < m; ++j) {
          const double tj1 = (j + 1 <= p) ? 0.0 : (j + 1 >= el + p ? h : h * (double)(j + 1 - p) / el);
          const double tjp = (j + p + 1 <= p) ? 0.0 : (j + p + 1 >= el + p ? h : h * (double)(j + p + 1 - p) / el);
          Amat[a * m + j] += w * (p / (tjp - tj1)) * tmp[j + 1];  // Curry-Schoenberg D_j
        }
        rhs[a] += w * sin(x0 + x);
      }
    }
  }
  solve_np(Amat, rhs, m);
  for (int i = 0; i < m; ++i) out[off_sin[d] + (int64_t)q * m + i] = rhs[i];
}

struct ProjTables {
  const double* base;
  int64_t off_cos[3], off_sin[3];
  int n[3];
};

// (Pi_h S) at local DOF A of the patch with indices pidx (product of 1D coefficients)
__device__ __forceinline__ double proj_entry(const ProjTables& pt, const int pidx[3], const LocalDof& A) {
  auto cB = [&](int d, int i) { return pt.base[pt.off_cos[d] + (int64_t)pidx[d] * pt.n[d] + i]; };
  auto sD = [&](int d, int i) { return pt.base[pt.off_sin[d] + (int64_t)pidx[d] * (pt.n[d] - 1) + i]; };
  if (A.c == 0) return sD(0, A.i[0]) * cB(1, A.i[1]) * cB(2, A.i[2]);
  if (A.c == 1) return -2.0 * cB(0, A.i[0]) * sD(1, A.i[1]) * cB(2, A.i[2]);
  return cB(0, A.i[0]) * cB(1, A.i[1]) * sD(2, A.i[2]);
}

// Per owned patch: a_loc = amp Pi_h S (initial condition of the conductors) and the Dirichlet
// template aD0[q] = (Pi_h S) at the q-th Dirichlet DOF (dlist: s * nloc + a).
__global__ void k_mms_init(DevPlan D, Geom G, ProjTables pt, double amp, const int* plist, double* a_loc,
                           const int64_t* __restrict__ dlist, const int64_t* __restrict__ doff, double* aD0) {
  const int s = plist[blockIdx.x];
  const int pidx[3] = {s % G.P[0], (s / G.P[0]) % G.P[1], s / (G.P[0] * G.P[1])};
  // conductors start from amp Pi_h S; an insulator (no mass term, sigma = 0) has no memory and
  // its gauge (tree) DOFs stay 0, as every step's recovery leaves them
  const bool cond = D.sigma[s] > 0.0;
  for (int a = threadIdx.x; a < G.nloc; a += blockDim.x)
    a_loc[(int64_t)s * G.nloc + a] = cond ? amp * proj_entry(pt, pidx, decode_local(G, a)) : 0.0;
  for (int64_t q = doff[s] + threadIdx.x; q < doff[s + 1]; q += blockDim.x)
    aD0[q] = proj_entry(pt, pidx, decode_local(G, (int)(dlist[q] - (int64_t)s * G.nloc)));
}

// Per owned patch, every aug position (r and p rows): JS = (3 nu - sigma) j_S - sum_{b in D}
// W^(a, b) (Pi_h S)_b, W^ = nu K + sigma/dt M from the Kronecker entries (the lifting folded
// into the load template; the stepper multiplies it by phi(t) = amp e^-t).
__global__ void k_mms_load(DevPlan D, Tables1D tb, Geom G, double inv_dt, const int* plist,
                           const int64_t* __restrict__ dlist, const int64_t* __restrict__ doff,
                           const double* __restrict__ aD0, double* JS) {
  const int s = plist[blockIdx.x];
  __shared__ T1 t[3];
  if (threadIdx.x < 3) {
    const int d = threadIdx.x;
    t[d].Mb = tb.base + tb.off_Mb[d];
    t[d].Md = tb.base + tb.off_Md[d];
    t[d].Kb = tb.base + tb.off_Kb[d];
    t[d].C = tb.base + tb.off_C[d];
    t[d].n = tb.el[d] + G.p;
  }
  __syncthreads();
  int pidx[3] = {s % G.P[0], (s / G.P[0]) % G.P[1], s / (G.P[0] * G.P[1])};
  const double nu = D.nu[s], sg = D.sigma[s] * inv_dt;
  const int* aug = D.aug + D.aug_off[s];
  const int R = D.T[s] * TS;
  for (int pos = threadIdx.x; pos < R; pos += blockDim.x) {
    const int a = aug[pos];
    if (a < 0) {
      JS[D.vec_off[s] + pos] = 0.0;
      continue;
    }
    const LocalDof A = decode_local(G, a);
    double h = 0.0;
    for (int64_t q = doff[s]; q < doff[s + 1]; ++q) {
      const LocalDof B = decode_local(G, (int)(dlist[q] - (int64_t)s * G.nloc));
      // the 1D factors vanish unless the supports overlap (|i_a - i_b| <= p per direction)
      if (abs(A.i[0] - B.i[0]) > G.p || abs(A.i[1] - B.i[1]) > G.p || abs(A.i[2] - B.i[2]) > G.p) continue;
      double K, M;
      kron_entry(t, A, B, K, M);
      h += (nu * K + sg * M) * aD0[q];
    }
    JS[D.vec_off[s] + pos] = (3.0 * nu - D.sigma[s]) * load_entry(tb, G, 3, pidx, A) - h;
  }
}

// ---- error norms ----------------------------------------------------------
// grid (owned patches, elements along z); every thread takes (ex, ey, Gauss point) tuples
// of its z layer. part[2 * block] = e_B share, part[2 * block + 1] = e_E share.
__global__ void __launch_bounds__(256) k_mms_errors(DevPlan D, Geom G, Tables1D tb, double t, double dt, double amp,
                                                    const int* plist, const double* __restrict__ a_loc,
                                                    const double* __restrict__ a_prev, double* part) {
  const int s = plist[blockIdx.x], ez = blockIdx.y;
  const int p = G.p, q = p + 1;
  const int pidx[3] = {s % G.P[0], (s / G.P[0]) % G.P[1], s / (G.P[0] * G.P[1])};
  const bool cond = D.sigma[s] > 0.0;
  const double* as = a_loc + (int64_t)s * G.nloc;
  const double* ao = a_prev + (int64_t)s * G.nloc;
  __shared__ double red[256];
  double gx[8], gw[8];
  for (int g = 0; g < q; ++g) gauss_legendre(q, g, gx[g], gw[g]);
  double eB = 0.0, eE = 0.0;
  const int npt = G.el[0] * G.el[1] * q * q * q;
  const double et = amp * exp(-t);
  int off[3];
  off[0] = 0;
  off[1] = G.cdim[0][0] * G.cdim[0][1] * G.cdim[0][2];
  off[2] = off[1] + G.cdim[1][0] * G.cdim[1][1] * G.cdim[1][2];
  for (int w = threadIdx.x; w < npt; w += blockDim.x) {
    int r = w;
    const int gxi = r % q; r /= q;
    const int gyi = r % q; r /= q;
    const int gzi = r % q; r /= q;
    const int ex = r % G.el[0], ey = r / G.el[0];
    const int e3[3] = {ex, ey, ez};
    const int gi[3] = {gxi, gyi, gzi};
    double x[3], wt = 1.0;
    double Bv[3][8], Dv[3][8], dB[3][8];  // active functions: B e..e+p, D e..e+p-1
    for (int d = 0; d < 3; ++d) {
      const int el = tb.el[d];
      const double h = tb.h[d];
      const double a0 = h * e3[d] / el, b0 = h * (e3[d] + 1) / el;
      const double xl = 0.5 * (a0 + b0) + 0.5 * (b0 - a0) * gx[gi[d]];
      wt *= 0.5 * (b0 - a0) * gw[gi[d]];
      x[d] = tb.lo[d] + pidx[d] * h + xl;
      double tB[160], tD[160];
      bsplines_at(p, el, h, p, xl, tB);
      bsplines_at(p, el, h, p - 1, xl, tD);
      auto knot = [&](int i) -> double { return i <= p ? 0.0 : (i >= el + p ? h : h * (double)(i - p) / el); };
      const int n = el + p;
      for (int k = 0; k <= p; ++k) {
        const int i = e3[d] + k;
        Bv[d][k] = tB[i];
        const double dm = (i >= 1) ? p / (knot(i + p) - knot(i)) * tD[i] : 0.0;            // D_{i-1}
        const double dp = (i <= n - 2) ? p / (knot(i + p + 1) - knot(i + 1)) * tD[i + 1] : 0.0;  // D_i
        dB[d][k] = dm - dp;
        if (k < p) Dv[d][k] = dp;
      }
    }
    // A_h and curl A_h: component c, active indices (D along c, B elsewhere)
    double Ah[3] = {0, 0, 0}, Ao[3] = {0, 0, 0}, Ch[3] = {0, 0, 0};
    for (int c = 0; c < 3; ++c) {
      const int nk = (c == 2) ? p : p + 1, nj = (c == 1) ? p : p + 1, ni = (c == 0) ? p : p + 1;
      for (int kk = 0; kk < nk; ++kk)
        for (int jj = 0; jj < nj; ++jj)
          for (int ii = 0; ii < ni; ++ii) {
            const int i = ex + ii, j = ey + jj, k = ez + kk;
            const int loc = off[c] + i + G.cdim[c][0] * (j + G.cdim[c][1] * k);
            const double cf = as[loc], co = ao[loc];
            const double fx = (c == 0) ? Dv[0][ii] : Bv[0][ii];
            const double fy = (c == 1) ? Dv[1][jj] : Bv[1][jj];
            const double fz = (c == 2) ? Dv[2][kk] : Bv[2][kk];
            const double v = fx * fy * fz;
            Ah[c] += cf * v;
            Ao[c] += co * v;
            if (c == 0) {  // curl (w_x) = (0, d/dz, -d/dy)
              Ch[1] += cf * fx * fy * dB[2][kk];
              Ch[2] -= cf * fx * dB[1][jj] * fz;
            } else if (c == 1) {  // curl (w_y) = (-d/dz, 0, d/dx)
              Ch[0] -= cf * fx * fy * dB[2][kk];
              Ch[2] += cf * dB[0][ii] * fy * fz;
            } else {  // curl (w_z) = (d/dy, -d/dx, 0)
              Ch[0] += cf * fx * dB[1][jj] * fz;
              Ch[1] -= cf * dB[0][ii] * fy * fz;
            }
          }
    }
    const double sx = sin(x[0]), sy = sin(x[1]), sz = sin(x[2]);
    const double cx = cos(x[0]), cy = cos(x[1]), cz = cos(x[2]);
    const double Be[3] = {-3.0 * et * cx * sy * sz, 0.0, 3.0 * et * sx * sy * cz};
    for (int c = 0; c < 3; ++c) eB += wt * (Be[c] - Ch[c]) * (Be[c] - Ch[c]);
    if (cond) {
      const double Ee[3] = {et * sx * cy * cz, -2.0 * et * cx * sy * cz, et * cx * cy * sz};
      for (int c = 0; c < 3; ++c) {
        const double v = Ee[c] + (Ah[c] - Ao[c]) / dt;
        eE += wt * v * v;
      }
    }
  }
  const double sB = block_sum(eB, red);
  const double sE = block_sum(eE, red);
  if (threadIdx.x == 0) {
    part[2 * ((int64_t)blockIdx.x * gridDim.y + blockIdx.y)] = sB;
    part[2 * ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) + 1] = sE;
  }
}

// One thread: this step's e_B, e_E as the fixed-order sum of the block partials; running
// max / dt-sums (acc[0] = max e_B, acc[1] = sum e_B, acc[2] = sum e_E), per-step values.
__global__ void k_mms_accumulate(const double* part, int nblocks, double dt, double* acc, double* per_step, int step) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double eB = 0.0, eE = 0.0;
  for (int b = 0; b < nblocks; ++b) {
    eB += part[2 * b];
    eE += part[2 * b + 1];
  }
  acc[0] = fmax(acc[0], eB);
  acc[1] += dt * eB;
  acc[2] += dt * eE;
  acc[3] = sqrt(acc[0] + acc[1]);  // eps_B
  acc[4] = sqrt(acc[2]);           // eps_E
  per_step[2 * step] = eB;
  per_step[2 * step + 1] = eE;
}

}  // namespace tcg
