// coarse_nd.h — host symbolic analysis of the sparse coarse problem (SURVEY §8(f) row f1,
// "coarse-problem restructuring"): nested dissection of the primal groups by the patch grid,
// elimination tree, supernodal frontal structure, and the index maps the GPU multifrontal
// factorisation and the in-kernel forward/backward solves use. Internal (host C++).
//
// The coarse matrix S_pp = sum_s N_s^T S^s N_s couples two primal groups iff
// some patch owns both. Bisecting the box of patch indices along its longest side, a group
// whose owner patches straddle the cut belongs to that separator node; the two halves are
// dissected recursively. Groups of two different halves share no patch, so separators
// separate, and every coupled pair lies on one root-to-leaf path. Node x eliminates its
// groups V_x; B_x = the ancestor groups coupled to V_x or to B of a child (the update set).
// Frontal index space of x: V_x at [0, n_V), padded to 64 T_V, then B_x, padded to 64 T.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

#include "plan.h"

namespace tcg {

struct NDNode {
  std::vector<int> V, B;        // groups eliminated here / update (ancestor) groups
  int parent = -1;
  std::vector<int> child;
  int height = 0;               // leaves 0; parent = 1 + max(child)
  int first = 0;                // postorder index of the first node of the subtree
  int TV = 0, TB = 0, T = 0;    // tile counts
};

struct CoarseND {
  std::vector<NDNode> nd;       // postorder (children before parents); root last
  std::vector<int> node_of;     // group -> node
  std::vector<int> pos_in_V;    // group -> index within V of its node
  int H = 0;                    // max height

  bool is_anc(int a, int x) const { return nd[a].first <= x && x < a; }  // a proper ancestor of x

  // frontal position of group g in node x (g in V_x or B_x), -1 otherwise
  int fpos(int x, int g) const {
    if (node_of[g] == x) return pos_in_V[g];
    const auto& B = nd[x].B;
    auto it = std::lower_bound(B.begin(), B.end(), g, [&](int a, int b) { return key(a) < key(b); });
    if (it != B.end() && *it == g) return 64 * nd[x].TV + (int)(it - B.begin());
    return -1;
  }
  // B is ordered by (node of the group, group id): ancestors nearest first
  int64_t key(int g) const { return ((int64_t)node_of[g] << 32) | (uint32_t)g; }

  // leaf_max: boxes of at most this many patches are not dissected further (one leaf front
  // eliminates all their groups): fewer levels = a shorter dependent chain per coarse solve
  void build(const Plan& pl, int leaf_max = 1) {
    const int64_t nc = pl.nc;
    node_of.assign(nc, -1);
    pos_in_V.assign(nc, -1);
    std::vector<int> lo(3 * nc), hi(3 * nc);
    for (int64_t g = 0; g < nc; ++g) {
      int l[3] = {1 << 30, 1 << 30, 1 << 30}, u[3] = {-1, -1, -1};
      for (int k = pl.coarse_ptr[g]; k < pl.coarse_ptr[g + 1]; ++k) {
        const int s = pl.coarse_patch[k];
        const int c[3] = {s % pl.P[0], (s / pl.P[0]) % pl.P[1], s / (pl.P[0] * pl.P[1])};
        for (int d = 0; d < 3; ++d) {
          l[d] = std::min(l[d], c[d]);
          u[d] = std::max(u[d], c[d]);
        }
      }
      for (int d = 0; d < 3; ++d) {
        lo[3 * g + d] = l[d];
        hi[3 * g + d] = u[d];
      }
    }
    // recursive bisection (explicit stack, nodes created in preorder, renumbered to postorder)
    struct Tmp {
      std::vector<int> V;
      int parent;
      std::vector<int> child;
    };
    std::vector<Tmp> t;
    struct Job {
      int lo[3], hi[3];
      std::vector<int> groups;
      int parent;
    };
    std::vector<Job> stack;
    Job root;
    for (int d = 0; d < 3; ++d) {
      root.lo[d] = 0;
      root.hi[d] = pl.P[d];
    }
    root.groups.resize(nc);
    for (int64_t g = 0; g < nc; ++g) root.groups[g] = (int)g;
    root.parent = -1;
    stack.push_back(std::move(root));
    while (!stack.empty()) {
      Job j = std::move(stack.back());
      stack.pop_back();
      const int me = (int)t.size();
      t.push_back(Tmp{{}, j.parent, {}});
      if (j.parent >= 0) t[j.parent].child.push_back(me);
      int d = 0;
      for (int e = 1; e < 3; ++e)
        if (j.hi[e] - j.lo[e] > j.hi[d] - j.lo[d]) d = e;
      const int64_t vol = (int64_t)(j.hi[0] - j.lo[0]) * (j.hi[1] - j.lo[1]) * (j.hi[2] - j.lo[2]);
      if (j.hi[d] - j.lo[d] <= 1 || vol <= leaf_max) {
        t[me].V = j.groups;
        continue;
      }
      const int mid = j.lo[d] + (j.hi[d] - j.lo[d]) / 2;
      Job L, R;
      for (int e = 0; e < 3; ++e) {
        L.lo[e] = R.lo[e] = j.lo[e];
        L.hi[e] = R.hi[e] = j.hi[e];
      }
      L.hi[d] = mid;
      R.lo[d] = mid;
      L.parent = R.parent = me;
      for (int g : j.groups) {
        if (lo[3 * g + d] < mid && hi[3 * g + d] >= mid) t[me].V.push_back(g);
        else if (hi[3 * g + d] < mid) L.groups.push_back(g);
        else R.groups.push_back(g);
      }
      // push right first so the left subtree is processed (numbered) first
      stack.push_back(std::move(R));
      stack.push_back(std::move(L));
    }
    // prune empty leaves (repeatedly: a node whose V is empty and has no children)
    std::vector<char> alive(t.size(), 1);
    std::vector<int> nchild(t.size(), 0);
    for (size_t i = 0; i < t.size(); ++i) nchild[i] = (int)t[i].child.size();
    for (int i = (int)t.size() - 1; i >= 0; --i) {  // children have larger preorder ids
      int live = 0;
      for (int c : t[i].child) live += alive[c];
      if (t[i].V.empty() && live == 0 && t[i].parent >= 0) alive[i] = 0;
    }
    // postorder over the live nodes
    std::vector<int> post, newid(t.size(), -1);
    {
      std::vector<std::pair<int, int>> st;  // (node, next child index)
      st.push_back({0, 0});
      while (!st.empty()) {
        auto& top = st.back();
        if (top.second < (int)t[top.first].child.size()) {
          const int c = t[top.first].child[top.second++];
          if (alive[c]) st.push_back({c, 0});
        } else {
          newid[top.first] = (int)post.size();
          post.push_back(top.first);
          st.pop_back();
        }
      }
    }
    nd.assign(post.size(), NDNode{});
    for (size_t k = 0; k < post.size(); ++k) {
      const Tmp& o = t[post[k]];
      NDNode& n = nd[k];
      n.V = o.V;
      std::sort(n.V.begin(), n.V.end());
      n.parent = o.parent >= 0 ? newid[o.parent] : -1;
      for (int c : o.child)
        if (alive[c]) n.child.push_back(newid[c]);
      for (size_t i = 0; i < n.V.size(); ++i) {
        node_of[n.V[i]] = (int)k;
        pos_in_V[n.V[i]] = (int)i;
      }
    }
    for (size_t k = 0; k < nd.size(); ++k) {  // subtree ranges and heights (postorder)
      NDNode& n = nd[k];
      n.first = (int)k;
      n.height = 0;
      for (int c : n.child) {
        n.first = std::min(n.first, nd[c].first);
        n.height = std::max(n.height, nd[c].height + 1);
      }
      H = std::max(H, n.height);
    }
    // symbolic factorisation: B_x = ancestors among adj(V_x) U (U_c B_c)
    std::vector<std::vector<int>> pgrp(pl.npatch);
    for (int s = 0; s < pl.npatch; ++s) pgrp[s].assign(pl.pp[s].p_grp.begin(), pl.pp[s].p_grp.end());
    std::vector<int> mark(nc, -1);
    for (size_t k = 0; k < nd.size(); ++k) {
      NDNode& n = nd[k];
      std::vector<int> cand;
      for (int g : n.V)
        for (int q = pl.coarse_ptr[g]; q < pl.coarse_ptr[g + 1]; ++q)
          for (int h : pgrp[pl.coarse_patch[q]])
            if (mark[h] != (int)k) {
              mark[h] = (int)k;
              cand.push_back(h);
            }
      for (int c : n.child)
        for (int h : nd[c].B)
          if (mark[h] != (int)k) {
            mark[h] = (int)k;
            cand.push_back(h);
          }
      for (int h : cand)
        if (is_anc(node_of[h], (int)k)) n.B.push_back(h);
      std::sort(n.B.begin(), n.B.end(), [&](int a, int b) { return key(a) < key(b); });
      n.TV = (int)((n.V.size() + 63) / 64);
      n.TB = (int)((n.B.size() + 63) / 64);
      n.T = n.TV + n.TB;
    }
  }
};

}  // namespace tcg
