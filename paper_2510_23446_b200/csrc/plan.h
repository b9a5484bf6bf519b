// plan.h — host-side topology, tree-cotree gauge and e/p/r partition (C++17).
//
// Independent reimplementation (no code shared with oracle/) of:
//   P:L78    conforming spaces: a shared DOF is one glued control-grid edge
//   P:L138   splitting into eliminated e, primal p (one value per coupled group), remaining r
//   P:L154   tree built globally "on the wirebasket first, ... faces and at last ... interiors",
//            Gamma tree DOFs primal, Dirichlet and insulator tree DOFs eliminated
// with the readings DESIGN.md R1 (wirebasket edges primal), R2 (ranked Kruskal order),
// R3 (classes), R4 (multiplier sign / ordering).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tcg {

constexpr int TILE = 64;   // tile edge of the dense per-patch factors

enum EdgeClass : uint8_t { CLS_D = 0, CLS_WB = 1, CLS_F = 2, CLS_I = 3 };
enum PartCode : uint8_t { PART_GAUGE = 0, PART_P = 1, PART_R = 2, PART_DIR = 3 };

struct PatchPlan {
  int ni = 0, nb = 0, np = 0;     // interior-r, interface-r (b), primal DOF counts
  int Ti = 0, Tb = 0, Tp = 0;     // tile counts (ceil(n/64))
  std::vector<int32_t> aug;       // aug position -> local DOF id (-1 = padding); size 64*(Ti+Tb+Tp)
  std::vector<int32_t> b_lam;     // per b position: multiplier index
  std::vector<int8_t> b_sign;     // per b position: +1 (lower patch id) / -1
  std::vector<int32_t> p_grp;     // per primal position: global primal group
};

struct Plan {
  // inputs
  int P[3] = {0, 0, 0};
  int p = 0;
  int el[3] = {0, 0, 0};
  double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  std::vector<double> sigma, nu;
  int tree_order = 0;
  int world = 1;
  // topology
  int n[3] = {0, 0, 0};           // B-splines per direction per patch (el + p)
  int64_t N[3] = {0, 0, 0};       // glued vertices per direction
  int npatch = 0;
  int nloc = 0;
  int64_t nverts = 0, nedges = 0;
  int64_t eoff[4] = {0, 0, 0, 0};
  int64_t edim[3][3] = {};
  std::vector<uint8_t> cls, region, in_tree, part;
  // numbering
  int64_t m = 0, nc = 0;
  std::vector<int64_t> lam_edge, lam_plus, lam_minus;       // per multiplier
  std::vector<int32_t> lam_plus_pos, lam_minus_pos;         // b-position in the owning patch
  std::vector<int64_t> primal_edge;                         // per primal group
  std::vector<int32_t> coarse_ptr, coarse_patch, coarse_pos; // CSR group -> (patch, primal position)
  std::vector<PatchPlan> pp;
  std::vector<int32_t> rank_of_patch;
  int64_t n_gauge = 0, n_dir = 0;

  std::string build();            // returns "" on success, else an error message

  // helpers
  int64_t edge_id(int c, int64_t i, int64_t j, int64_t k) const {
    return eoff[c] + i + edim[c][0] * (j + edim[c][1] * k);
  }
  void edge_coords(int64_t e, int& c, int64_t& i, int64_t& j, int64_t& k) const;
  int local_id(int c, int i, int j, int k) const;
  void local_coords(int a, int& c, int& i, int& j, int& k) const;
  int comp_dim(int c, int d) const { return n[d] - (c == d ? 1 : 0); }
  int64_t local_to_global(int s, int a) const;
  void owners(int64_t e, int* out, int& cnt) const;
};

}  // namespace tcg
