#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
// plan.cpp — host planning: glued topology, ranked-Kruskal tree, partition, numbering.
// See plan.h for the paper passages and DESIGN.md readings followed.
#include "plan.h"

#include <algorithm>
#include <numeric>
#include <sstream>

namespace tcg {

void Plan::edge_coords(int64_t e, int& c, int64_t& i, int64_t& j, int64_t& k) const {
  c = e < eoff[1] ? 0 : (e < eoff[2] ? 1 : 2);
  int64_t r = e - eoff[c];
  i = r % edim[c][0];
  j = (r / edim[c][0]) % edim[c][1];
  k = r / (edim[c][0] * edim[c][1]);
}

int Plan::local_id(int c, int i, int j, int k) const {
  int off = 0;
  for (int cc = 0; cc < c; ++cc) off += comp_dim(cc, 0) * comp_dim(cc, 1) * comp_dim(cc, 2);
  return off + i + comp_dim(c, 0) * (j + comp_dim(c, 1) * k);
}

void Plan::local_coords(int a, int& c, int& i, int& j, int& k) const {
  c = 0;
  for (;;) {
    int sz = comp_dim(c, 0) * comp_dim(c, 1) * comp_dim(c, 2);
    if (a < sz) break;
    a -= sz;
    ++c;
  }
  i = a % comp_dim(c, 0);
  j = (a / comp_dim(c, 0)) % comp_dim(c, 1);
  k = a / (comp_dim(c, 0) * comp_dim(c, 1));
}

int64_t Plan::local_to_global(int s, int a) const {
  int c, i, j, k;
  local_coords(a, c, i, j, k);
  int ix = s % P[0], iy = (s / P[0]) % P[1], iz = s / (P[0] * P[1]);
  return edge_id(c, (int64_t)ix * (n[0] - 1) + i, (int64_t)iy * (n[1] - 1) + j, (int64_t)iz * (n[2] - 1) + k);
}

// Owning patches of a glued edge: along the edge direction the patch is unique; along a
// transverse direction a coordinate on an interior patch-boundary layer has two patches.
void Plan::owners(int64_t e, int* out, int& cnt) const {
  int c;
  int64_t x[3];
  edge_coords(e, c, x[0], x[1], x[2]);
  int cand[3][2], nc_[3];
  for (int d = 0; d < 3; ++d) {
    int64_t h = n[d] - 1;
    if (d == c) {
      cand[d][0] = (int)(x[d] / h);
      nc_[d] = 1;
    } else if (x[d] % h == 0) {
      int q = (int)(x[d] / h);
      nc_[d] = 0;
      if (q - 1 >= 0) cand[d][nc_[d]++] = q - 1;
      if (q < P[d]) cand[d][nc_[d]++] = q;
    } else {
      cand[d][0] = (int)(x[d] / h);
      nc_[d] = 1;
    }
  }
  cnt = 0;
  for (int a = 0; a < nc_[2]; ++a)
    for (int b = 0; b < nc_[1]; ++b)
      for (int q = 0; q < nc_[0]; ++q) out[cnt++] = cand[0][q] + P[0] * (cand[1][b] + P[1] * cand[2][a]);
  std::sort(out, out + cnt);
}

namespace {
struct DSU {
  std::vector<int64_t> parent;
  explicit DSU(int64_t nv) : parent(nv) { std::iota(parent.begin(), parent.end(), 0); }
  int64_t find(int64_t a) {
    while (parent[a] != a) {
      parent[a] = parent[parent[a]];
      a = parent[a];
    }
    return a;
  }
  bool unite(int64_t a, int64_t b) {
    a = find(a);
    b = find(b);
    if (a == b) return false;
    if (a < b) std::swap(a, b);
    parent[a] = b;
    return true;
  }
};
int ceil_tiles(int v) { return (v + TILE - 1) / TILE; }
}  // namespace

std::string Plan::build() {
  std::ostringstream err;
  const bool tm = getenv("TCG_HOST_TIMING") && atoi(getenv("TCG_HOST_TIMING")) != 0;
  auto tlast = std::chrono::steady_clock::now();
  std::string tline;
#define PMARK(w)                                                                                       \
  if (tm) {                                                                                            \
    const auto t_ = std::chrono::steady_clock::now();                                                  \
    tline += std::string(" ") + (w) + " " + std::to_string(std::chrono::duration<double, std::milli>(t_ - tlast).count()); \
    tlast = t_;                                                                                        \
  }
  if (p < 1) return "degree p must be >= 1";
  for (int d = 0; d < 3; ++d) {
    if (P[d] < 1 || el[d] < 1) return "patch and element counts must be >= 1";
    if (!(lo[d] < hi[d])) return "degenerate box";
    n[d] = el[d] + p;
    N[d] = (int64_t)P[d] * (n[d] - 1) + 1;
  }
  npatch = P[0] * P[1] * P[2];
  if ((int)sigma.size() != npatch || (int)nu.size() != npatch) return "materials not set for every patch";
  for (int s = 0; s < npatch; ++s) {
    if (!(sigma[s] >= 0)) return "sigma must be >= 0";
    if (!(nu[s] > 0)) return "nu must be > 0";
  }
  nloc = 0;
  for (int c = 0; c < 3; ++c) nloc += comp_dim(c, 0) * comp_dim(c, 1) * comp_dim(c, 2);
  nverts = N[0] * N[1] * N[2];
  int64_t off = 0;
  for (int c = 0; c < 3; ++c) {
    for (int d = 0; d < 3; ++d) edim[c][d] = N[d] - (c == d ? 1 : 0);
    eoff[c] = off;
    off += edim[c][0] * edim[c][1] * edim[c][2];
  }
  eoff[3] = off;
  nedges = off;

  PMARK("head");
  // ---- classes and regions (R3) ----
  cls.assign(nedges, CLS_I);
  region.assign(nedges, 0);
  std::vector<uint8_t> nown(nedges, 0);
  // per direction and vertex coordinate x: patch-layer / boundary flags and the (one or two)
  // patch indices whose closure contains the layer x (transverse), or the patch holding the
  // edge [x, x+1] (along the edge); the edge loops below run in edge-id order
  std::vector<int> t_first[3], t_cnt[3], a_patch[3];
  std::vector<uint8_t> t_bnd[3], t_lay[3];
  for (int d = 0; d < 3; ++d) {
    const int64_t h = n[d] - 1;
    t_first[d].resize(N[d]);
    t_cnt[d].resize(N[d]);
    t_bnd[d].resize(N[d]);
    t_lay[d].resize(N[d]);
    a_patch[d].resize(N[d]);
    for (int64_t x = 0; x < N[d]; ++x) {
      t_bnd[d][x] = (x == 0 || x == N[d] - 1);
      t_lay[d][x] = !t_bnd[d][x] && (x % h == 0);
      if (x % h == 0) {
        const int q = (int)(x / h);
        t_first[d][x] = q - 1 >= 0 ? q - 1 : q;
        t_cnt[d][x] = (q - 1 >= 0) + (q < P[d]);
      } else {
        t_first[d][x] = (int)(x / h);
        t_cnt[d][x] = 1;
      }
      a_patch[d][x] = (int)std::min<int64_t>(x / h, P[d] - 1);
    }
  }
  std::vector<uint8_t> sflag(npatch);
  for (int s = 0; s < npatch; ++s) sflag[s] = (sigma[s] > 0) ? 1 : 2;
  {
    int64_t e = 0;
    for (int c = 0; c < 3; ++c)
      for (int64_t k = 0; k < edim[c][2]; ++k)
        for (int64_t j = 0; j < edim[c][1]; ++j)
          for (int64_t i = 0; i < edim[c][0]; ++i, ++e) {
            const int64_t x[3] = {i, j, k};
            bool bnd = false;
            int nlay = 0;
            int f[3], cn[3];
            for (int d = 0; d < 3; ++d) {
              if (d == c) {
                f[d] = a_patch[d][x[d]];
                cn[d] = 1;
                continue;
              }
              bnd = bnd || t_bnd[d][x[d]];
              nlay += t_lay[d][x[d]];
              f[d] = t_first[d][x[d]];
              cn[d] = t_cnt[d][x[d]];
            }
            cls[e] = bnd ? CLS_D : (nlay == 2 ? CLS_WB : (nlay == 1 ? CLS_F : CLS_I));
            nown[e] = (uint8_t)(cn[0] * cn[1] * cn[2]);
            uint8_t r = 0;
            for (int z = 0; z < cn[2]; ++z)
              for (int y = 0; y < cn[1]; ++y)
                for (int q = 0; q < cn[0]; ++q) r |= sflag[(f[0] + q) + P[0] * ((f[1] + y) + P[1] * (f[2] + z))];
            region[e] = r;
          }
  }

  PMARK("classes");
  // ---- ranked Kruskal tree (R2) ----
  // rank 0 D; 1..3 conductor-owned WB/F/I; 4..6 insulator-only WB/F/I
  std::vector<uint8_t> rank_of(nedges);
  for (int64_t e = 0; e < nedges; ++e)
    rank_of[e] = cls[e] == CLS_D ? 0 : ((region[e] & 1) ? 1 : 4) + (cls[e] == CLS_WB ? 0 : (cls[e] == CLS_F ? 1 : 2));
  in_tree.assign(nedges, 0);
  DSU dsu(nverts);
  int64_t ntree = 0;
  const int64_t vstride[3] = {1, N[0], N[0] * N[1]};
  for (int rk = 0; rk < 7; ++rk) {
    auto visit = [&](int64_t e, int c, int64_t i, int64_t j, int64_t k) {
      if (rank_of[e] != rk) return;
      const int64_t va = i + N[0] * (j + N[1] * k);
      if (dsu.unite(va, va + vstride[c])) {
        in_tree[e] = 1;
        ++ntree;
      }
    };
    if (tree_order == 1) {  // descending ids within each rank
      int64_t e = nedges - 1;
      for (int c = 2; c >= 0; --c)
        for (int64_t k = edim[c][2] - 1; k >= 0; --k)
          for (int64_t j = edim[c][1] - 1; j >= 0; --j)
            for (int64_t i = edim[c][0] - 1; i >= 0; --i, --e) visit(e, c, i, j, k);
    } else {
      int64_t e = 0;
      for (int c = 0; c < 3; ++c)
        for (int64_t k = 0; k < edim[c][2]; ++k)
          for (int64_t j = 0; j < edim[c][1]; ++j)
            for (int64_t i = 0; i < edim[c][0]; ++i, ++e) visit(e, c, i, j, k);
    }
  }
  if (ntree != nverts - 1) {
    err << "tree has " << ntree << " edges for " << nverts << " vertices";
    return err.str();
  }

  PMARK("tree");
  // ---- partition (R1) ----
  part.assign(nedges, PART_R);
  n_gauge = n_dir = 0;
  for (int64_t e = 0; e < nedges; ++e) {
    bool conductor = region[e] & 1, insulator = region[e] & 2;
    if (cls[e] == CLS_D) {
      part[e] = PART_DIR;
      ++n_dir;
    } else if (in_tree[e] && !conductor) {
      part[e] = PART_GAUGE;
      ++n_gauge;
    } else if (cls[e] == CLS_WB || (in_tree[e] && conductor && insulator)) {
      part[e] = PART_P;
    }
    if (part[e] == PART_R && nown[e] > 2) return "an r-DOF with more than two owners";
  }

  PMARK("partition");
  // ---- numbering: multipliers (b-edges ascending) and primal groups ----
  std::vector<int64_t> lam_of(nedges, -1), grp_of(nedges, -1);
  lam_edge.clear();
  primal_edge.clear();
  for (int64_t e = 0; e < nedges; ++e) {
    if (part[e] == PART_R && nown[e] == 2) {
      lam_of[e] = (int64_t)lam_edge.size();
      lam_edge.push_back(e);
    } else if (part[e] == PART_P) {
      grp_of[e] = (int64_t)primal_edge.size();
      primal_edge.push_back(e);
    }
  }
  m = (int64_t)lam_edge.size();
  nc = (int64_t)primal_edge.size();
  lam_plus.assign(m, -1);
  lam_minus.assign(m, -1);
  lam_plus_pos.assign(m, -1);
  lam_minus_pos.assign(m, -1);

  PMARK("numbering");
  // ---- per patch lists, aug order [i | pad | b | pad | p | pad] ----
  pp.assign(npatch, PatchPlan());
  std::vector<std::vector<std::pair<int, int>>> grp_owners(nc);
  for (int s = 0; s < npatch; ++s) {
    PatchPlan& q = pp[s];
    std::vector<int32_t> li, lb, lp;
    std::vector<int64_t> gb, gpv;  // global ids of the b and p DOFs
    std::vector<int8_t> sb;        // b DOFs: +1 if this patch is the lower-id owner
    {
      const int sx = s % P[0], sy = (s / P[0]) % P[1], sz = s / (P[0] * P[1]);
      const int64_t o3[3] = {(int64_t)sx * (n[0] - 1), (int64_t)sy * (n[1] - 1), (int64_t)sz * (n[2] - 1)};
      int a = 0;
      for (int c = 0; c < 3; ++c)
        for (int k = 0; k < comp_dim(c, 2); ++k)
          for (int j = 0; j < comp_dim(c, 1); ++j)
            for (int i = 0; i < comp_dim(c, 0); ++i, ++a) {
              const int64_t g = edge_id(c, o3[0] + i, o3[1] + j, o3[2] + k);
              if (part[g] == PART_R) {
                if (nown[g] == 1) {
                  li.push_back(a);
                } else {
                  // two owners: they differ along the one transverse direction whose local
                  // coordinate is on the patch's low (other patch has the lower id) or high face
                  const int lc[3] = {i, j, k};
                  int8_t sg = 1;
                  for (int d = 0; d < 3; ++d)
                    if (d != c && t_lay[d][o3[d] + lc[d]]) sg = (lc[d] == 0) ? -1 : 1;
                  lb.push_back(a);
                  gb.push_back(g);
                  sb.push_back(sg);
                }
              } else if (part[g] == PART_P) {
                lp.push_back(a);
                gpv.push_back(g);
              }
            }
    }
    q.ni = (int)li.size();
    q.nb = (int)lb.size();
    q.np = (int)lp.size();
    q.Ti = ceil_tiles(q.ni);
    q.Tb = ceil_tiles(q.nb);
    q.Tp = ceil_tiles(q.np);
    q.aug.assign((size_t)TILE * (q.Ti + q.Tb + q.Tp), -1);
    for (int t = 0; t < q.ni; ++t) q.aug[t] = li[t];
    for (int t = 0; t < q.nb; ++t) q.aug[(size_t)TILE * q.Ti + t] = lb[t];
    for (int t = 0; t < q.np; ++t) q.aug[(size_t)TILE * (q.Ti + q.Tb) + t] = lp[t];
    q.b_lam.resize(q.nb);
    q.b_sign.resize(q.nb);
    for (int t = 0; t < q.nb; ++t) {
      const int64_t g = gb[t];
      int64_t k = lam_of[g];
      q.b_lam[t] = (int32_t)k;
      if (sb[t] > 0) {
        q.b_sign[t] = 1;
        lam_plus[k] = s;
        lam_plus_pos[k] = t;
      } else {
        q.b_sign[t] = -1;
        lam_minus[k] = s;
        lam_minus_pos[k] = t;
      }
    }
    q.p_grp.resize(q.np);
    for (int t = 0; t < q.np; ++t) {
      const int64_t g = gpv[t];
      q.p_grp[t] = (int32_t)grp_of[g];
      grp_owners[grp_of[g]].push_back({s, t});
    }
  }
  for (int64_t k = 0; k < m; ++k)
    if (lam_plus[k] < 0 || lam_minus[k] < 0) return "multiplier without two owners";
  PMARK("patches");
  coarse_ptr.assign(nc + 1, 0);
  coarse_patch.clear();
  coarse_pos.clear();
  for (int64_t g = 0; g < nc; ++g) {
    auto& v = grp_owners[g];
    std::sort(v.begin(), v.end());
    for (auto& pr : v) {
      coarse_patch.push_back(pr.first);
      coarse_pos.push_back(pr.second);
    }
    coarse_ptr[g + 1] = (int32_t)coarse_patch.size();
  }

  PMARK("coarse");
  // ---- sharding: contiguous x-slabs of patches ----
  rank_of_patch.assign(npatch, 0);
  for (int s = 0; s < npatch; ++s) {
    int ix = s % P[0];
    rank_of_patch[s] = (int)((int64_t)ix * world / P[0]);
  }
  PMARK("shard");
  if (tm) fprintf(stderr, "[tcg plan ms]%s\n", tline.c_str());
#undef PMARK
  return "";
}

}  // namespace tcg
