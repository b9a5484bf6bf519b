// device.h — device-side views of the plan and the kernel entry points (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tcg {

// Geometry of one patch type (all patches of a config have the same shape).
struct Geom {
  int P[3];
  int p;
  int el[3];
  int cdim[3][3];  // component c: index range along direction d
  int nloc;
};

// 1D tables (a1): flat buffer with per-direction offsets.
struct Tables1D {
  double* base;
  int64_t off_Mb[3], off_Md[3], off_Kb[3], off_C[3], off_oneD[3], off_sD[3], off_cB[3], off_sB[3];
  int el[3];
  int P[3];
  double h[3];
  double lo[3];
};

// Device copy of the plan and the big device arrays.
constexpr int MAXR = 8;  // ranks (GPUs, or virtual ranks on one GPU) of a sharded solve

// Device view of the plan. Per-patch index arrays are global (all patches, replicated on
// every rank); the big per-patch matrices live on the patch's owning rank: the tile pointer
// of patch s is Ar[owner[s]] + a_off[s] (a_off is relative to the owner's allocation).
// A / Dinv / Sbb are the launching rank's own allocations (setup kernels only touch owned
// patches).
struct DevPlan {
  int npatch;
  int nranks;
  const int* owner;         // per patch: owning rank
  double* Ar[MAXR];         // per rank: augmented factors / inverse factors
  double* Sbbr[MAXR];       // per rank: S_bb stores
  double* SIr[MAXR];        // per rank: explicit S_bb^-1 = X_bb^T X_bb stores (S_bb layout; null if unused)
  int64_t m, nc;
  // per patch
  const int* Ti;
  const int* Tb;
  const int* Tp;
  const int* T;        // Ti+Tb+Tp
  const int* nb;
  const int* np;
  const int64_t* a_off;     // augmented tile-packed factor
  const int64_t* dinv_off;  // diagonal inverse tiles (Ti+Tb tiles)
  const int64_t* sbb_off;   // captured S_bb store
  const int64_t* vec_off;   // aug-ordered per-patch vectors (64*T each)
  const int64_t* aug_off;
  const int* aug;           // aug position -> local id (-1 padding)
  const int* loc2aug;       // per patch (npatch x nloc): local id -> aug position (-1 eliminated)
  const int64_t* b_off;     // per patch offset into b_lam / b_sign
  const int* b_lam;
  const double* b_sign;
  const int64_t* b_part;    // per b position: aug-vector index of the multiplier's other endpoint
  double* b_aown;           // per b position: B_D weight of this side (w+ or w-)
  double* b_apart;          // per b position: -(weight of the other side)
  const int64_t* p_off;     // per patch offset into p_grp
  const int* p_grp;
  const int64_t* tile_start;  // prefix of T(T+1)/2 (npatch+1)
  const double* sigma;
  const double* nu;
  // multipliers
  const int* lam_patch_p;
  const int* lam_patch_m;
  const int* lam_pos_p;
  const int* lam_pos_m;
  const int64_t* lam_idx_p;  // index into aug-ordered vectors (b part) for the + side
  const int64_t* lam_idx_m;
  double* wplus;
  double* wminus;
  // coarse CSR
  const int* coarse_ptr;
  const int64_t* coarse_idx;  // index into aug-ordered vectors (p part)
  const int* coarse_patch;    // patch of each CSR entry (its owner holds the value)
  // big arrays
  double* A;      // augmented factors
  double* Dinv;
  double* Sbb;
  // coarse factor
  double* C;      // tile-packed lower n_c (Tc tiles)
  double* Cinv;   // diagonal inverse tiles of C
  int Tc;
  int maxT, maxTbp;   // largest tile counts (shared-memory layout of the solver kernels)
  int me;             // launching rank (setup kernels)
};

}  // namespace tcg
