// capi.cu — the C ABI (include/tcg_ietidp.h): handle state machine, device memory,
// setup orchestration (assembly -> batched Cholesky -> inverse factors -> coarse) and the
// implicit-Euler stepping (one persistent cooperative launch, pcg.cu). All arithmetic of the
// method runs in the kernels of assembly.cu / chol.cu / pcg.cu, compiled into this TU.
//
// Sharding: patches are owned by ranks (contiguous x-slabs, plan.cpp). A rank
// holds the factors of its patches and the global-layout vectors it owns entries of; values
// owned elsewhere are read through per-rank pointer tables: peer device memory mapped with
// CUDA IPC on a multi-GPU job (one process per GPU, NCCL only to bootstrap), or other
// allocations of the same device for "virtual ranks" (several ranks emulated in one
// cooperative grid on one GPU; tcg_set_virtual_ranks) which exercise the identical sharded
// dataflow where only one GPU is available.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/tcg_ietidp.h"
#include "plan.h"
#include "assembly.cu"
#include "chol.cu"
#include "solve.cu"
#include "pcg.cu"
#include "nd.cu"
#include "mms.cu"
#include "nonlinear.cu"
#include "coarse_nd.h"

using namespace tcg;

// ---- NCCL, loaded at run time (only for world > 1) ---------------------------------------
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclChar = 0, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (lib) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!lib) lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) {
      err = "libnccl.so.2 not found";
      return false;
    }
    commInitRank = (decltype(commInitRank))dlsym(lib, "ncclCommInitRank");
    getUniqueId = (decltype(getUniqueId))dlsym(lib, "ncclGetUniqueId");
    allGather = (decltype(allGather))dlsym(lib, "ncclAllGather");
    allReduce = (decltype(allReduce))dlsym(lib, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(lib, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(lib, "ncclGetErrorString");
    if (!commInitRank || !allGather || !allReduce || !commDestroy) {
      err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;
}  // namespace

// One rank's device data (this process's rank on a multi-GPU job, or one virtual rank).
struct RankDev {
  int r = 0;
  std::vector<int> plist;  // owned patches
  int* d_plist = nullptr;
  int64_t* d_tstart = nullptr;
  int64_t ntiles = 0;
  double *A = nullptr, *Dinv = nullptr, *Sbb = nullptr, *xscr = nullptr;
  double* SI = nullptr;  // explicit S_bb^-1 (S_bb layout) when the iteration applies it (sbbinv)
  double *Wr = nullptr, *FWr = nullptr, *dsave = nullptr, *wpart = nullptr;  // warm start (lazy)
  CholDesc* d_desc = nullptr;
  int ndesc = 0, maxT = 0, maxTr = 0, maxTb = 0;
  // global-layout vectors (entries of owned patches / lambda chunks valid)
  double *F = nullptr, *Z = nullptr, *XJ = nullptr, *JS = nullptr, *XW = nullptr, *Y = nullptr, *Y2 = nullptr, *PW = nullptr;
  double *a_loc = nullptr, *lam = nullptr, *r0 = nullptr, *r1 = nullptr, *pk0 = nullptr, *pk1 = nullptr, *q = nullptr;
  double *Ppart = nullptr, *Pc = nullptr, *partials = nullptr, *hist = nullptr;
  int* iters = nullptr;
  BarMem* bar = nullptr;
  PcgState* st = nullptr;
  DevError* derr = nullptr;
  // nonlinear patches (nonlinear.cu): owned list, tile prefix, Gauss-point
  // coefficients Q, Newton right-hand-side vector g (aug layout), a^l and the iterate a_k
  std::vector<int> nlist;
  int* d_nlist = nullptr;
  CholDesc* d_nldesc = nullptr;
  int nl_maxT = 0, nl_maxTr = 0, nl_maxTb = 0;
  int64_t* d_ntstart = nullptr;
  int64_t nl_ntiles = 0;
  double *Q = nullptr, *gnl = nullptr, *a_old = nullptr, *a_k = nullptr, *nl_part = nullptr, *Kel = nullptr;
  // replicated coarse problem (computed by the first local rank, aliased by other local ranks)
  double *C = nullptr, *Cinv = nullptr, *CX = nullptr, *Sinv = nullptr;
  DevPlan D{};  // DevPlan with me / A / Dinv / Sbb of this rank
};

struct tcg_ctx {
  int device = 0, rank = 0, world = 1;
  int vranks = 1;  // virtual ranks emulated in this process (world must be 1)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Plan plan;
  bool have_patches = false, have_materials = false, have_time = false;
  bool planned = false, setup_done = false, broken = false;
  int source = TCG_SOURCE_CURL_PSI;
  // the paper's experiment (TCG_SOURCE_PAPER, mms.cu): 1D projections, Dirichlet DOF list and
  // template values; error tracking state
  double* proj = nullptr;
  ProjTables ptab{};
  int64_t *d_dlist = nullptr, *d_doff = nullptr;
  int64_t* d_poff = nullptr;
  double* aD0 = nullptr;
  int64_t ndir = 0;  // Dirichlet DOFs (patch-local copies) of the paper's experiment
  bool track = false;
  std::vector<double*> a_prev;     // per local rank: a_loc before the step
  double *err_part = nullptr, *err_acc = nullptr, *err_step = nullptr;
  int err_blocks = 0;
  double src_amp = 1.0, src_freq = 1.0;  // tcg_set_source params
  // nonlinear reluctivity (tcg_set_nonlinear): Brauer (k1,k2,k3) per patch
  std::vector<double> nlk;
  int n_nl = 0;
  double newton_tol = 1e-8;
  int newton_max = 20;
  double* d_nlk = nullptr;
  unsigned char* d_nlflag = nullptr;  // per patch: 1 = nonlinear
  double* rho_diag = nullptr;         // per multiplier: W^ diagonal at its + and - copies
  bool err_nl = false;                // the last factorisation ran over the nonlinear lists
  double* nltab = nullptr;
  NlTab ntab{};
  size_t nl_smem = 0;
  std::vector<int> newton_its, solve_its;
  std::vector<double> solve_inc;
  double ms_newton_numeric = 0.0;  // device time of the Newton re-assemblies + factorisations
  bool is_nl(int s) const { return n_nl > 0 && (nlk[3 * s] != 0.0 || nlk[3 * s + 1] != 0.0 || nlk[3 * s + 2] != 0.0); }
  // patches whose right-hand side is recomputed every step (mass term or Newton vector)
  bool dyn(int s) const { return plan.sigma[s] > 0 || is_nl(s); }
  double T = 1.0;
  int n_steps = 0;
  double rtol = 1e-10;
  int max_iter = 5000;
  int scaling = TCG_SCALING_RHO;
  int tree_order = 0;
  int stable_mask = 0;  // bit2: TRSM by substitution (env TCG_STABLE)
  unsigned char nccl_id[128];
  ncclComm_t comm = nullptr;
  std::string err;

  // device state
  std::vector<void*> allocs;       // cudaMalloc (multi-GPU: IPC-exportable)
  std::vector<void*> pool_allocs;  // cudaMallocFromPoolAsync from the library's own pool
  bool pool_user = false;          // counted in the device's live-handle count of that pool
  double* agree_buf = nullptr;     // world > 1: per-launch agreement of the warm-start state
  std::vector<void*> ipc_opened;
  int64_t device_bytes = 0;
  int nranks = 1;  // ranks of the job: world (real) or vranks (virtual)
  std::vector<RankDev> rd;  // local ranks
  DevPlan D{};              // global arrays + per-rank tables (me/A/Dinv/Sbb unset)
  Geom G{};
  Tables1D tb{};
  CholDesc* d_cdesc = nullptr;
  InvDesc* d_cinv = nullptr;
  int* d_colour = nullptr;
  std::vector<int64_t> colour_off;
  int* d_crow_owner = nullptr;
  int64_t* d_glued_src = nullptr;
  double* glued = nullptr;
  double* a_all = nullptr;  // gathered local coefficients (readout)
  int64_t* d_aloc_src = nullptr;
  PcgState* h_st = nullptr;  // pinned
  int maxT = 0, maxTr = 0, maxTb = 0, maxTp = 0, Tc = 0;
  int64_t nb_total = 0, vec_total = 0;
  // sparse coarse problem (nested dissection + multifrontal); sparse = 0: dense S_pp^-1
  int sparse = 0;
  CoarseND nd;
  struct NDDev {
    double *FR = nullptr, *FDinv = nullptr, *Fscr = nullptr;
    // solve state per local rank (each rank runs the replicated coarse solve on its blocks)
    std::vector<double*> CW, Pcs, pb;
    std::vector<unsigned int*> cnt, dflow;
    int64_t fr_size = 0;
    std::vector<std::vector<int>> lvl;            // node ids per height
    std::vector<CholDesc*> ldesc;                 // per level
    std::vector<int*> lplist;                     // per level node list (device)
    std::vector<int> lmaxT, lmaxTV;
    std::vector<std::vector<int*>> lkids;         // [level][slot] children (device)
    std::vector<std::vector<int>> nkids;
    DevPlan Dn{};                                 // patch-like view of the nodes (k_xinv_row)
    int *tv = nullptr, *tt = nullptr, *nv = nullptr, *nbv = nullptr, *parent = nullptr;
    int64_t *aoff = nullptr, *moff = nullptr, *map = nullptr, *xo = nullptr;
    int* ext = nullptr;
    int64_t* prog = nullptr;
    int *vl = nullptr, *bl = nullptr;
    ItemDesc *fw = nullptr, *bw = nullptr;
    int *fw_off = nullptr, *bw_off = nullptr;     // [(level) * (nblocks + 1) + block]
    int kw = 1;                                    // forward gather sources per position
    int4* node = nullptr;                          // per node: parent, #fw items, #bw items, #children's fw items
    int2* bwdep = nullptr;                         // per node: backward dependency (ancestor or -1), its item count
    int nn = 0;
  } ndd;
  // stepper work items per phase: ItemDesc lists ordered by (rank, block), per-block offsets
  ItemDesc* d_items[NPH] = {};
  int* d_boff[NPH] = {};
  std::vector<int> h_boff[NPH];
  std::vector<ItemDesc> h_items[NPH];
  int* d_bpl = nullptr;
  int* d_bploff = nullptr;
  int cache_bpos = 0;
  int cache_items = 0, cache_lam = 0, cache_pcprog = 0;
  int npf = 0;  // prefetched tiles per phase (stepper)
  // the PCG iteration applies W_rr^-1 restricted to b as the explicit S_bb^-1 = X_bb^T X_bb
  // (one symmetric read) instead of X_bb^T (X_bb v) (two reads); TCG_SBBINV=0 restores the latter
  bool sbbinv = true;
  bool ovl = false;     // S_bb^-1 items as side work of the sparse coarse solve (TCG_OVERLAP)
  int ovl_chain = 0;    // blocks that run the coarse levels above the leaves and take no side items
  // local factorisation order: left-looking (deep-K column updates, default) or right-looking
  // (TCG_CHOL=right)
  bool chol_left = true;
  int warm = 0;  // warm-start subspace dimension k (tcg_set_warm_start), 0 = off
  int64_t warm_base = 0;  // first step of the current warm-start history (k changed / refactor)
  int64_t* d_pcprog = nullptr;
  size_t smem_steps = 0;  // dynamic shared memory of k_steps: item scratch + caches
  int coarse_ch = 1, coarse_maxch = 1;
  size_t smem_pcg = 0, smem_tables = 0;
  int nbr = 0;  // persistent blocks per rank
  int64_t lam_chunk = 1;
  unsigned int bar_round = 0;  // barrier rounds completed (monotone counters, never reset)
  std::vector<std::vector<void*>> peer_bufs;  // [rank][buffer] device pointers (own or peer)
  double* sync_tok = nullptr;
  unsigned long long* tstamp = nullptr;
  double* itime = nullptr;
  int itime_stride = 0;
  double* dbgA = nullptr;
  double* dbgC = nullptr;
  std::vector<int64_t> h_a_off, h_vec_off, h_sbb_off;
  std::vector<int> h_T, h_owner;

  // results
  int64_t steps_done = 0, total_iters = 0, hist_len = 0;
  std::vector<int> iters;
  std::vector<double> final_rel, hist_all;
  std::vector<int64_t> hist_per_step;  // relres-history entries of each step (Newton: all its solves)
  int64_t nlaunch = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  int prof_id = 0;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<int> prof_tag;
  size_t prof_used = 0;
  double prof_ms = 0;
  int64_t prof_count = 0;
  double ms_plan = 0, ms_assembly = 0, ms_factor = 0, ms_coarse = 0, ms_steps = 0;

  ~tcg_ctx() { release(); }
  // The library's own stream-ordered memory pool per device (never the device's default
  // pool): freed memory is kept while handles live on the device (re-creating a handle costs
  // no driver allocations) and trimmed to zero when the last handle of the device is released.
  struct PoolReg {
    std::mutex mu;
    cudaMemPool_t pool[64] = {};
    int live[64] = {};
  };
  static PoolReg& pools() {
    static PoolReg r;
    return r;
  }
  static cudaMemPool_t lib_pool(int device) {
    PoolReg& R = pools();
    std::lock_guard<std::mutex> lk(R.mu);
    if (device < 0 || device >= 64) return nullptr;
    if (!R.pool[device]) {
      cudaMemPoolProps pp{};
      pp.allocType = cudaMemAllocationTypePinned;
      pp.location.type = cudaMemLocationTypeDevice;
      pp.location.id = device;
      cudaMemPool_t mp = nullptr;
      if (cudaMemPoolCreate(&mp, &pp) != cudaSuccess) return nullptr;
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
      R.pool[device] = mp;
    }
    return R.pool[device];
  }
  // pinned PcgState buffers are recycled across handles (cudaMallocHost costs ~ms)
  static std::vector<PcgState*>& pinned_free() {
    static std::vector<PcgState*> v;
    return v;
  }
  static std::mutex& pinned_mu() {
    static std::mutex m;
    return m;
  }
  void release() {
    if (!allocs.empty() || !pool_allocs.empty() || stream) cudaSetDevice(device);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    ipc_opened.clear();
    for (void* p : pool_allocs) cudaFreeAsync(p, stream);
    pool_allocs.clear();
    if (stream) cudaStreamSynchronize(stream);
    if (pool_user) {  // last handle on this device: hand the pool's memory back to the driver
      PoolReg& R = pools();
      std::lock_guard<std::mutex> lk(R.mu);
      const char* keep = getenv("TCG_POOL_RETAIN");  // experiment: keep the freed memory cached
      if (--R.live[device] == 0 && R.pool[device] && !(keep && atoi(keep))) cudaMemPoolTrimTo(R.pool[device], 0);
      pool_user = false;
    }
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
    if (h_st) {
      std::lock_guard<std::mutex> lk(pinned_mu());
      pinned_free().push_back(h_st);
    }
    h_st = nullptr;
    for (auto e : prof_ev) cudaEventDestroy(e);
    prof_ev.clear();
    if (comm && g_nccl.commDestroy) g_nccl.commDestroy(comm);
    comm = nullptr;
    if (own_stream && stream) cudaStreamDestroy(stream);
    stream = nullptr;
  }
};

namespace {

tcg_status fail(tcg_ctx* h, tcg_status s, const std::string& msg) {
  if (h) h->err = msg;
  return s;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) {                                                                      \
      h->broken = (e_ != cudaErrorMemoryAllocation);                                              \
      return fail(h, e_ == cudaErrorMemoryAllocation ? TCG_ENOMEM : TCG_ECUDA,                    \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                            \
    }                                                                                             \
  } while (0)

#define CKL()                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = cudaGetLastError();                                                          \
    if (e_ != cudaSuccess) {                                                                      \
      h->broken = true;                                                                           \
      return fail(h, TCG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_) + " at " + \
                                    std::to_string(__LINE__));                                    \
    }                                                                                             \
  } while (0)

#define TRY(x)                   \
  do {                           \
    tcg_status s_ = (x);         \
    if (s_ != TCG_OK) return s_; \
  } while (0)

// Device allocations: single-process handles use the library's own stream-ordered pool
// (tcg_ctx::lib_pool; trimmed when the device's last handle is released); multi-GPU handles
// use cudaMalloc (their buffers are exported with CUDA IPC).

template <class T>
tcg_status dalloc(tcg_ctx* h, T** out, size_t n) {
  size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  void* p = nullptr;
  cudaError_t e;
  if (h->world == 1) {
    cudaMemPool_t mp = tcg_ctx::lib_pool(h->device);
    if (!mp) return fail(h, TCG_ECUDA, "cudaMemPoolCreate failed");
    if (!h->pool_user) {
      std::lock_guard<std::mutex> lk(tcg_ctx::pools().mu);
      ++tcg_ctx::pools().live[h->device];
      h->pool_user = true;
    }
    e = cudaMallocFromPoolAsync(&p, bytes, mp, h->stream);
    if (e == cudaSuccess) h->pool_allocs.push_back(p);
  } else {
    e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) h->allocs.push_back(p);
  }
  if (e != cudaSuccess) return fail(h, TCG_ENOMEM, std::string("cudaMalloc ") + std::to_string(bytes) + ": " + cudaGetErrorString(e));
  static const bool poison = getenv("TCG_POISON") && atoi(getenv("TCG_POISON")) != 0;  // debug: NaN-fill
  if (poison) cudaMemsetAsync(p, 0xff, bytes, h->stream);
  h->device_bytes += (int64_t)bytes;
  *out = static_cast<T*>(p);
  return TCG_OK;
}

template <class T>
tcg_status dzero(tcg_ctx* h, T** out, size_t n) {
  TRY(dalloc(h, out, n));
  cudaError_t e = cudaMemsetAsync(*out, 0, std::max<size_t>(n, 1) * sizeof(T), h->stream);
  if (e != cudaSuccess) return fail(h, TCG_ECUDA, std::string("memset: ") + cudaGetErrorString(e));
  return TCG_OK;
}

template <class T>
tcg_status dupload(tcg_ctx* h, T** out, const std::vector<T>& v) {
  tcg_status s = dalloc(h, out, v.size());
  if (s != TCG_OK) return s;
  if (!v.empty()) {
    cudaError_t e = cudaMemcpyAsync(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, h->stream);
    h->h2d_bytes += (int64_t)(v.size() * sizeof(T));
    if (e != cudaSuccess) return fail(h, TCG_ECUDA, std::string("upload: ") + cudaGetErrorString(e));
  }
  return TCG_OK;
}

double elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

tcg_status set_smem(tcg_ctx* h, const void* fn, size_t bytes) {
  if (bytes > 227 * 1024) return fail(h, TCG_EINVAL, "kernel needs " + std::to_string(bytes) + " B shared memory (> 227 KB)");
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(bytes, 48 * 1024)));
  return TCG_OK;
}

// Cross-process barrier on the stream (multi-GPU only): a 1-element NCCL allreduce.
tcg_status sync_ranks(tcg_ctx* h) {
  if (h->world <= 1) return TCG_OK;
  if (!h->sync_tok) TRY(dzero(h, &h->sync_tok, 1));
  ncclResult_t r = g_nccl.allReduce(h->sync_tok, h->sync_tok, 1, ncclFloat64, ncclSum, h->comm, h->stream);
  if (r != 0) return fail(h, TCG_ENCCL, std::string("ncclAllReduce: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?"));
  CK(cudaStreamSynchronize(h->stream));
  return TCG_OK;
}

}  // namespace

// =========================================================================================
// plan
// =========================================================================================
static tcg_status do_plan(tcg_ctx* h) {
  if (h->planned) return TCG_OK;
  if (!h->have_patches || !h->have_materials || !h->have_time)
    return fail(h, TCG_ESTATE, "set_patches, set_materials and set_time are required");
  auto t0 = std::chrono::steady_clock::now();
  h->nranks = std::max(h->world, h->vranks);
  h->plan.tree_order = h->tree_order;
  h->plan.world = h->nranks;
  std::string e = h->plan.build();
  if (!e.empty()) return fail(h, TCG_EINVAL, "plan: " + e);
  h->planned = true;
  h->ms_plan = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return TCG_OK;
}

// =========================================================================================
// numeric setup (assembly, batched Cholesky, inverse factors, coarse)
// =========================================================================================
// maxTtail > 0: left-looking (k_colupd per column, k_tailupd for the trailing block of at
// most maxTtail tiles); 0: right-looking (k_capture_sbb / k_update per column)
static tcg_status run_cholesky(tcg_ctx* h, const CholDesc* d_desc, int nmat, int maxT, int maxTf, int maxTb,
                               double* base, double* dinv, double* sbb, DevError* derr, int coarse, int maxTtail = 0) {
  const int subst = (h->stable_mask & 4) ? 1 : 0;
  if (maxTtail > 0) {
    for (int J = 0; J < maxTf; ++J) {
      k_colupd<<<dim3((unsigned)(maxT - J), (unsigned)nmat), 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(
          d_desc, J, base, sbb);
      k_potrf<<<nmat, 256, 2 * TS * PS * sizeof(double), h->stream>>>(d_desc, J, base, dinv, derr, coarse);
      h->nlaunch += 2;
      CKL();
      const int rows = maxT - J - 1;
      if (rows > 0) {
        k_trsm<<<dim3(rows, nmat), 128, 2 * TS * SPAD * sizeof(double), h->stream>>>(d_desc, J, base, dinv, subst);
        ++h->nlaunch;
        CKL();
      }
    }
    k_tailupd<<<dim3((unsigned)tri_tiles(maxTtail), (unsigned)nmat), 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(
        d_desc, base);
    ++h->nlaunch;
    CKL();
    return TCG_OK;
  }
  for (int k = 0; k < maxTf; ++k) {
    if (sbb && maxTb > 0) {
      dim3 gc((unsigned)tri_tiles(maxTb), nmat);
      k_capture_sbb<<<gc, 256, 0, h->stream>>>(d_desc, k, base, sbb);
      ++h->nlaunch;
      CKL();
    }
    k_potrf<<<nmat, 256, 2 * TS * PS * sizeof(double), h->stream>>>(d_desc, k, base, dinv, derr, coarse);
    ++h->nlaunch;
    CKL();
    int rows = maxT - k - 1;
    if (rows > 0) {
      dim3 gt(rows, nmat);
      k_trsm<<<gt, 128, 2 * TS * SPAD * sizeof(double), h->stream>>>(d_desc, k, base, dinv, subst);
      ++h->nlaunch;
      CKL();
      dim3 gu((unsigned)tri_tiles(rows), nmat);
      k_update<<<gu, 128, 2 * TS * SPAD * sizeof(double), h->stream>>>(d_desc, k, base);
      ++h->nlaunch;
      CKL();
    }
  }
  return TCG_OK;
}

// Sparse coarse numeric setup: zero + pad the frontal matrices, scatter every patch's S^s,
// then bottom-up per level: extend-add the children's update matrices, partial Cholesky of
// the V columns, in-place inverse [L_VV^-1 ; L_BV L_VV^-1].
static tcg_status numeric_sparse_coarse(tcg_ctx* h) {
  auto& g = h->ndd;
  const auto& N = h->nd.nd;
  const int nn = (int)N.size();
  RankDev& R = h->rd[0];
  if (nn == 0) return TCG_OK;
  CK(cudaMemsetAsync(g.FR, 0, sizeof(double) * (size_t)g.fr_size, h->stream));
  k_nd_pad<<<nn, 256, 0, h->stream>>>(g.tv, g.tt, g.nv, g.nbv, g.aoff, g.FR);
  ++h->nlaunch;
  CKL();
  for (int c = 0; c < 8; ++c) {
    const int cnt = (int)(h->colour_off[c + 1] - h->colour_off[c]);
    if (cnt == 0) continue;
    const int chunks = std::max(1, std::min(32, 2 * 148 / std::max(cnt, 1)));
    k_nd_scatter<<<dim3(cnt, chunks), 256, 0, h->stream>>>(R.D, h->d_colour + h->colour_off[c], cnt, g.moff, g.map, g.FR);
    ++h->nlaunch;
    CKL();
  }
  for (int lv = 0; lv <= h->nd.H; ++lv) {
    const int nlv = (int)g.lvl[lv].size();
    if (nlv == 0) continue;
    for (int slot = 0; slot < 2; ++slot) {
      const int nk = g.nkids[lv][slot];
      if (nk == 0) continue;
      k_nd_extend<<<dim3(64, nk), 256, 0, h->stream>>>(g.lkids[lv][slot], nk, g.parent, g.tv, g.nbv, g.aoff, g.xo, g.ext,
                                                       g.FR);
      ++h->nlaunch;
      CKL();
    }
    TRY(run_cholesky(h, g.ldesc[lv], nlv, g.lmaxT[lv], g.lmaxTV[lv], 0, g.FR, g.FDinv, nullptr, R.derr, 1));
    for (int I = 0; I < g.lmaxT[lv]; ++I) {
      dim3 gr(std::max(1, std::min(I + 1, g.lmaxTV[lv])), (unsigned)nlv);
      k_xinv_row<<<gr, 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(g.Dn, I, g.Fscr, g.Dn.dinv_off, g.lplist[lv]);
      ++h->nlaunch;
      k_xrow_copy<<<gr, 256, 0, h->stream>>>(g.Dn, I, g.Fscr, g.Dn.dinv_off, g.lplist[lv]);
      ++h->nlaunch;
      CKL();
    }
  }
  return TCG_OK;
}

static tcg_status check_err(tcg_ctx* h) {
  CK(cudaStreamSynchronize(h->stream));
  for (auto& R : h->rd) {
    DevError herr;
    CK(cudaMemcpy(&herr, R.derr, sizeof(DevError), cudaMemcpyDeviceToHost));
    if (herr.flag) {
      h->broken = true;
      std::ostringstream o;
      if (herr.matrix >= 0) o << "local Cholesky: patch " << (h->err_nl ? R.nlist : R.plist)[herr.matrix];
      else o << "coarse Cholesky";
      o << " pivot " << herr.index << " value " << herr.value;
      return fail(h, TCG_ENOTSPD, o.str());
    }
  }
  return TCG_OK;
}

// newton = true: one Newton iterate's re-assembly and factorisation (nonlinear.cu, tcg_step):
// the nonlinear patches' tangent matrices at the current coefficients a_loc, the Newton
// right-hand-side vector g; the time-stepping state (a, steps, histories) is kept.
static tcg_status do_numeric(tcg_ctx* h, const std::function<tcg_status()>& mid = nullptr, bool newton = false) {
  Plan& pl = h->plan;
  const int Tc = h->Tc;
  const double dt = h->T / h->n_steps;
  struct Events {  // destroyed on every return path
    cudaEvent_t e[4];
    Events() {
      for (auto& x : e) cudaEventCreate(&x);
    }
    ~Events() {
      for (auto& x : e) cudaEventDestroy(x);
    }
  } ev;
  cudaEvent_t e0 = ev.e[0], e1 = ev.e[1], e2 = ev.e[2], e3 = ev.e[3];
  CK(cudaEventRecord(e0, h->stream));
  // Newton iterates re-assemble and re-factorise the nonlinear patches only: the linear
  // patches' factors, S_bb, inverse factors, S^s and load vectors are unchanged
  if (!newton) {
    k_tables1d<<<3, 256, h->smem_tables, h->stream>>>(h->tb, pl.p, h->source == TCG_SOURCE_PAPER ? 1.0 : M_PI);
    ++h->nlaunch;
    CKL();
  }
  if (h->source == TCG_SOURCE_PAPER) {
    const int maxP = std::max(pl.P[0], std::max(pl.P[1], pl.P[2]));
    int maxn = 0;
    for (int d = 0; d < 3; ++d) maxn = std::max(maxn, pl.el[d] + pl.p);
    k_proj1d<<<dim3(maxP, 3), 32, sizeof(double) * ((size_t)maxn * maxn + maxn), h->stream>>>(h->tb, pl.p, h->d_poff,
                                                                                               h->d_poff + 3, h->proj);
    ++h->nlaunch;
    CKL();
    if (h->track) {
      CK(cudaMemsetAsync(h->err_acc, 0, 8 * sizeof(double), h->stream));
    }
  }
  h->err_nl = newton;
  for (auto& R : h->rd) {
    CK(cudaMemsetAsync(R.derr, 0, sizeof(DevError), h->stream));
    if (newton) continue;
    if (R.ntiles > 0) {
      k_assemble<<<(unsigned)R.ntiles, 256, 0, h->stream>>>(R.D, h->tb, h->G, 1.0 / dt, R.d_plist, R.d_tstart,
                                                           (int)R.plist.size());
      ++h->nlaunch;
      CKL();
    }
    if (!R.plist.empty() && h->source == TCG_SOURCE_PAPER) {
      // a(0) = amp Pi_h S, Dirichlet template, load template with the lifting folded in (mms.cu)
      k_mms_init<<<(unsigned)R.plist.size(), 256, 0, h->stream>>>(R.D, h->G, h->ptab, h->src_amp, R.d_plist, R.a_loc,
                                                                   h->d_dlist, h->d_doff, h->aD0);
      ++h->nlaunch;
      k_mms_load<<<(unsigned)R.plist.size(), 256, 0, h->stream>>>(R.D, h->tb, h->G, 1.0 / dt, R.d_plist, h->d_dlist,
                                                                   h->d_doff, h->aD0, R.JS);
      ++h->nlaunch;
      CKL();
    } else if (!R.plist.empty()) {
      k_load_vector<<<(unsigned)R.plist.size(), 256, 0, h->stream>>>(R.D, h->tb, h->G, h->source, R.JS, R.d_plist);
      ++h->nlaunch;
      CKL();
    }
  }
  if (h->n_nl > 0) {
    // nonlinear patches (nonlinear.cu): Gauss-point B, nu, nu' from the current coefficients
    // (zero at setup / refactor: the time stepping restarts from A = 0), the tangent matrix
    // J = Kt + (sigma/dt) M over k_assemble's tiles, and g = (Kt - K) a
    if (!newton) {
      k_nl_tab1d<<<3, 128, 0, h->stream>>>(h->nltab, h->ntab, h->tb, pl.p);
      ++h->nlaunch;
      CKL();
    }
    const int64_t nqp = (int64_t)h->ntab.nq[0] * h->ntab.nq[1] * h->ntab.nq[2];
    for (auto& R : h->rd) {
      if (!newton) CK(cudaMemsetAsync(R.a_loc, 0, sizeof(double) * (size_t)pl.npatch * pl.nloc, h->stream));
      const unsigned nn = (unsigned)R.nlist.size();
      if (nn == 0) continue;
      k_nl_quad<<<dim3(nn, (unsigned)std::min<int64_t>(64, (nqp + 255) / 256)), 256, 0, h->stream>>>(
          h->G, h->ntab, R.d_nlist, R.a_loc, h->d_nlk, R.Q);
      launch_nl_assemble(pl.p, (unsigned)R.nl_ntiles, h->nl_smem, h->stream, R.D, h->tb, h->G, h->ntab, 1.0 / dt,
                         R.d_nlist, R.d_ntstart, (int)nn, R.Q, R.Kel);
      k_nl_g<<<dim3(nn, (unsigned)((pl.nloc + 255) / 256)), 256, h->nl_smem, h->stream>>>(R.D, h->G, h->ntab, R.d_nlist,
                                                                                        R.Q, R.gnl);
      h->nlaunch += 3;
      CKL();
    }
  }
  if (const char* ns = newton ? nullptr : getenv("TCG_DEBUG_NOTSPD")) {  // test hook: first pivot of patch s := -1
    const int sbad = atoi(ns);
    for (auto& R : h->rd)
      if (sbad >= 0 && sbad < pl.npatch && pl.rank_of_patch[sbad] == R.r) {
        const double neg = -1.0;
        CK(cudaMemcpyAsync(R.A + h->h_a_off[sbad], &neg, sizeof(double), cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
      }
  }
  TRY(sync_ranks(h));  // every rank's W^ assembled (rho weights read both interface sides)
  for (auto& R : h->rd) {
    if (pl.m > 0) {
      // diagonal of W^ at both sides of every multiplier, captured from the freshly assembled
      // tiles (Newton: the nonlinear patches' sides only; the rest keep the linear values)
      k_rho_capture<<<(unsigned)((pl.m + 255) / 256), 256, 0, h->stream>>>(R.D, h->rho_diag, newton ? h->d_nlflag : nullptr);
      ++h->nlaunch;
      k_rho_weights<<<(unsigned)((pl.m + 255) / 256), 256, 0, h->stream>>>(R.D, h->scaling, h->rho_diag);
      ++h->nlaunch;
      CKL();
    }
    if (h->nb_total > 0) {
      k_btables<<<(unsigned)((h->nb_total + 255) / 256), 256, 0, h->stream>>>(R.D, h->nb_total);
      ++h->nlaunch;
      CKL();
    }
    break;  // wplus/wminus/b tables are global arrays shared by the local ranks of this process
  }
  CK(cudaEventRecord(e1, h->stream));
  TRY(sync_ranks(h));  // rho weights read before any rank overwrites its W^ with the factor
  if (h->dbgA && h->rd.size() == 1)
    CK(cudaMemcpyAsync(h->dbgA, h->rd[0].A, sizeof(double) * h->h_a_off.back(), cudaMemcpyDeviceToDevice, h->stream));
  for (auto& R : h->rd) {
    const int nmat = newton ? (int)R.nlist.size() : R.ndesc;
    if (nmat == 0) continue;
    const int mT = newton ? R.nl_maxT : R.maxT, mTr = newton ? R.nl_maxTr : R.maxTr, mTb = newton ? R.nl_maxTb : R.maxTb;
    const int* lst = newton ? R.d_nlist : R.d_plist;
    TRY(run_cholesky(h, newton ? R.d_nldesc : R.d_desc, nmat, mT, mTr, mTb, R.A, R.Dinv, R.Sbb, R.derr, 0,
                     h->chol_left ? std::max(1, h->maxTp) : 0));
    // in-place inverse of the augmented factor: Xaug = [L_rr^-1 ; W_pr W_rr^-1]
    const int64_t* scr_off = h->D.dinv_off;  // scratch rows share the Dinv layout (Tr tiles)
    for (int I = 0; I < mT; ++I) {
      dim3 g(std::min(I + 1, mTr), (unsigned)nmat);
      k_xinv_row<<<g, 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(R.D, I, R.xscr, scr_off, lst);
      ++h->nlaunch;
      k_xrow_copy<<<g, 256, 0, h->stream>>>(R.D, I, R.xscr, scr_off, lst);
      ++h->nlaunch;
      CKL();
    }
    if (h->sbbinv && mTb > 0) {  // S_bb^-1 = X_bb^T X_bb for the PCG iteration
      k_sbbinv<<<dim3((unsigned)tri_tiles(mTb), (unsigned)nmat), 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(
          R.D, lst, R.SI);
      ++h->nlaunch;
      CKL();
    }
  }
  CK(cudaEventRecord(e2, h->stream));
  TRY(sync_ranks(h));  // S^s of every patch final before the (replicated) coarse assembly
  if (h->sparse) {
    TRY(numeric_sparse_coarse(h));
  } else {
    RankDev& R = h->rd[0];  // the coarse problem is computed once per process
    CK(cudaMemsetAsync(R.C, 0, sizeof(double) * (size_t)tri_tiles(Tc) * TSZ, h->stream));
    if (pl.nc > 0) {
      DevPlan Dc = R.D;
      Dc.C = R.C;
      for (int c = 0; c < 8; ++c) {
        int cnt = (int)(h->colour_off[c + 1] - h->colour_off[c]);
        if (cnt == 0) continue;
        const int chunks = std::max(1, std::min(32, 2 * 148 / std::max(cnt, 1)));  // fill the GPU
        k_coarse_scatter<<<dim3(cnt, chunks), 256, 0, h->stream>>>(Dc, h->d_colour + h->colour_off[c], cnt);
        ++h->nlaunch;
        CKL();
      }
      int npad = Tc * TS - (int)pl.nc;
      if (npad > 0) {
        k_coarse_pad<<<(npad + 255) / 256, 256, 0, h->stream>>>(Dc);
        ++h->nlaunch;
        CKL();
      }
      if (h->dbgC) CK(cudaMemcpyAsync(h->dbgC, R.C, sizeof(double) * tri_tiles(Tc) * TSZ, cudaMemcpyDeviceToDevice, h->stream));
      TRY(run_cholesky(h, h->d_cdesc, 1, Tc, Tc, 0, R.C, R.Cinv, nullptr, R.derr, 1));
      for (int I = 0; I < Tc; ++I) {
        dim3 g(I + 1, 1);
        k_trinv_row<<<g, 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(h->d_cinv, I, R.C, R.CX, R.Cinv);
        ++h->nlaunch;
        CKL();
      }
      k_sinv<<<dim3(Tc, Tc), 128, MMA_SMEM_DOUBLES * sizeof(double), h->stream>>>(R.CX, R.Sinv, Tc);
      ++h->nlaunch;
      CKL();
    }
  }
  if (mid) TRY(mid());  // host work overlapped with the kernels above (first setup only)
  // insulator precompute: XJ = [X_rr j_S,r ; j_S,p - Phi^T j_S,r] for owned patches (the
  // nonlinear patches never use it: their rhs is recomputed every step)
  for (auto& R : h->rd) {
    if (newton) break;
    const int b0 = h->h_boff[PH_FWA][R.r * h->nbr], n = h->h_boff[PH_FWA][(R.r + 1) * h->nbr] - b0;
    if (n > 0) {
      k_fw<<<n, NTHR, h->smem_pcg, h->stream>>>(R.D, h->d_items[PH_FWA] + b0, n, R.JS, R.XJ);
      ++h->nlaunch;
      CKL();
    }
    if (h->source != TCG_SOURCE_PAPER && !newton)  // (the paper's experiment starts from a(0) = amp Pi_h S, set above)
      CK(cudaMemsetAsync(R.a_loc, 0, sizeof(double) * (size_t)pl.npatch * pl.nloc, h->stream));
  }
  CK(cudaEventRecord(e3, h->stream));
  TRY(check_err(h));
  TRY(sync_ranks(h));
  h->ms_assembly = elapsed_ms(e0, e1);
  h->ms_factor = elapsed_ms(e1, e2);
  h->ms_coarse = elapsed_ms(e2, e3);
  if (newton) {
    h->ms_newton_numeric += elapsed_ms(e0, e3);
    return TCG_OK;
  }
  h->newton_its.clear();
  h->solve_its.clear();
  h->solve_inc.clear();
  h->ms_newton_numeric = 0.0;
  h->steps_done = 0;
  h->warm_base = 0;  // refactor / setup: the time integration restarts, so does the warm history
  h->hist_len = 0;
  h->total_iters = 0;
  h->iters.clear();
  h->hist_per_step.clear();
  h->final_rel.clear();
  h->hist_all.clear();
  return TCG_OK;
}

// =========================================================================================
// setup: layouts, uploads, per-rank allocations, peer tables
// =========================================================================================
// Work items of one stepper phase, per rank: (cost, item). Dealt to the rank's nbr persistent
// blocks by LPT (largest first onto the least-loaded block; ties to the lower block), each
// block's items kept in that order. A fixed per-item overhead models the gather latency.
struct ItemLists {
  std::vector<std::vector<std::pair<int, ItemDesc>>> per_rank;
  explicit ItemLists(int nr) : per_rank(nr) {}
};

static tcg_status deal_items(tcg_ctx* h, ItemLists& L, int ph, int overhead, bool group = false, int skip_first = 0) {
  const int nbr = h->nbr;
  auto bycost = [](const std::pair<int, ItemDesc>& x, const std::pair<int, ItemDesc>& y) {
    return x.first != y.first ? x.first > y.first
                              : (x.second.s != y.second.s ? x.second.s < y.second.s : x.second.I < y.second.I);
  };
  std::vector<ItemDesc> all;
  std::vector<int> boff(1, 0);
  for (auto& v : L.per_rank) {
    std::stable_sort(v.begin(), v.end(), bycost);
    std::vector<std::vector<ItemDesc>> blk(nbr);
    std::vector<std::pair<int64_t, int>> heap;  // (load, block) min-heap
    for (int b = 0; b < nbr; ++b) heap.push_back({b < skip_first ? ((int64_t)1 << 50) : 0, b});  // the first skip_first blocks get nothing
    auto cmp = [](const std::pair<int64_t, int>& x, const std::pair<int64_t, int>& y) { return x > y; };
    std::make_heap(heap.begin(), heap.end(), cmp);
    if (group) {
      // many patches per block: deal whole (patch, part) groups, so each block gathers a
      // patch's input vector once for all its rows / columns
      std::vector<std::pair<int64_t, std::vector<ItemDesc>>> grp;
      std::map<std::pair<int, int>, size_t> keys;
      for (auto& e : v) {
        const std::pair<int, int> key{e.second.s, e.second.part};
        auto kit = keys.find(key);
        size_t gi;
        if (kit == keys.end()) {
          gi = grp.size();
          keys[key] = gi;
          grp.push_back({0, {}});
        } else {
          gi = kit->second;
        }
        grp[gi].first += e.first + 1;
        grp[gi].second.push_back(e.second);
      }
      std::stable_sort(grp.begin(), grp.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
      for (auto& gr : grp) {
        std::pop_heap(heap.begin(), heap.end(), cmp);
        auto& top = heap.back();
        blk[top.second].insert(blk[top.second].end(), gr.second.begin(), gr.second.end());
        top.first += gr.first + overhead;
        std::push_heap(heap.begin(), heap.end(), cmp);
      }
    } else {
      for (auto& e : v) {
        std::pop_heap(heap.begin(), heap.end(), cmp);
        auto& top = heap.back();
        blk[top.second].push_back(e.second);
        top.first += e.first + overhead;
        std::push_heap(heap.begin(), heap.end(), cmp);
      }
    }
    for (int b = 0; b < nbr; ++b) {
      // same-patch items adjacent: the kernel gathers a patch's input once per run
      std::stable_sort(blk[b].begin(), blk[b].end(), [](const ItemDesc& x, const ItemDesc& y) {
        return x.s != y.s ? x.s < y.s : (x.part != y.part ? x.part < y.part : x.I < y.I);
      });
      // gather codes (bits 4-5 of part): reuse the previous item's input / gather all of it
      std::vector<int> code(blk[b].size());
      auto same = [&](size_t a, size_t c) { return blk[b][a].s == blk[b][c].s && blk[b][a].part == blk[b][c].part; };
      for (size_t j = 0; j < blk[b].size(); ++j)
        code[j] = (j > 0 && same(j - 1, j)) ? 0 : ((j + 1 < blk[b].size() && same(j + 1, j)) ? 2 : 1);
      for (size_t j = 0; j < blk[b].size(); ++j) blk[b][j].part |= code[j] << 4;
      all.insert(all.end(), blk[b].begin(), blk[b].end());
      boff.push_back((int)all.size());
    }
  }
  for (auto& d : all) d.bc = -1;
  h->h_items[ph] = all;
  h->h_boff[ph] = boff;
  return TCG_OK;
}

// Sparse coarse problem: nested-dissection symbolic analysis (coarse_nd.h), node
// storage, assembly maps, per-level factorisation descriptors, the forward gather programs and
// the stepper's per-level work items (single-rank handles; requires h->nbr).
// host-side timeline of do_setup (TCG_HOST_TIMING=1: one line on stderr per setup)
struct HostMarks {
  bool on = getenv("TCG_HOST_TIMING") && atoi(getenv("TCG_HOST_TIMING")) != 0;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  std::string line;
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    char b[96];
    snprintf(b, sizeof b, " %s %.3f", what, std::chrono::duration<double, std::milli>(t - last).count());
    line += b;
    last = t;
  }
  ~HostMarks() {
    if (on) fprintf(stderr, "[tcg host ms]%s total %.3f\n", line.c_str(),
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

static tcg_status setup_sparse_coarse(tcg_ctx* h, const std::vector<int>& owner, const std::vector<int64_t>& cidx,
                                      const std::vector<int>& cpat) {
  Plan& pl = h->plan;
  CoarseND& nd = h->nd;
  HostMarks hm;
  hm.line = " [sparse coarse]";
  nd = CoarseND();
  {
    // leaf boxes of up to 32 patches (TCG_ND_LEAF): measured on cfg4 / cfg5, profiles/round2_notes.md
    const char* e = getenv("TCG_ND_LEAF");
    nd.build(pl, e ? std::max(1, atoi(e)) : 32);
  }
  hm.mark("nd-build");
  const auto& N = nd.nd;
  const int nn = (int)N.size();
  auto& g = h->ndd;
  std::vector<int64_t> aoff(nn), doff(nn), voff(nn);
  int64_t fa = 0, fd = 0, fv = 0;
  for (int x = 0; x < nn; ++x) {
    aoff[x] = fa;
    fa += tri_tiles(N[x].T) * TSZ;
    doff[x] = fd;
    fd += (int64_t)N[x].TV * TSZ;
    voff[x] = fv;
    fv += (int64_t)N[x].T * TS;
  }
  g.fr_size = fa;
  TRY(dalloc(h, &g.FR, std::max<int64_t>(fa, 1)));
  TRY(dalloc(h, &g.FDinv, std::max<int64_t>(fd, 1)));
  TRY(dalloc(h, &g.Fscr, std::max<int64_t>(fd, 1)));
  const int nlocal = (h->world > 1) ? 1 : h->vranks;  // local ranks (same order as h->rd)
  g.CW.assign(nlocal, nullptr);
  g.Pcs.assign(nlocal, nullptr);
  g.pb.assign(nlocal, nullptr);
  g.cnt.assign(nlocal, nullptr);
  g.dflow.assign(nlocal, nullptr);
  for (int li = 0; li < nlocal; ++li) {
    TRY(dzero(h, &g.CW[li], std::max<int64_t>(fv, 1)));
    TRY(dzero(h, &g.Pcs[li], std::max<int64_t>(pl.nc, 1)));
  }
  std::vector<int> tv(nn), tt(nn), nvv(nn), nbv(nn), par(nn), zero(nn, 0);
  for (int x = 0; x < nn; ++x) {
    tv[x] = N[x].TV;
    tt[x] = N[x].T;
    nvv[x] = (int)N[x].V.size();
    nbv[x] = (int)N[x].B.size();
    par[x] = N[x].parent;
  }
  int *dzero_i, *dtv, *dtt;
  int64_t *daoff, *ddoff;
  TRY(dupload(h, &dzero_i, zero));
  TRY(dupload(h, &dtv, tv));
  TRY(dupload(h, &dtt, tt));
  TRY(dupload(h, &g.nv, nvv));
  TRY(dupload(h, &g.nbv, nbv));
  TRY(dupload(h, &g.parent, par));
  TRY(dupload(h, &daoff, aoff));
  TRY(dupload(h, &ddoff, doff));
  g.tv = dtv;
  g.tt = dtt;
  g.aoff = daoff;
  g.Dn = DevPlan{};
  g.Dn.Ti = dzero_i;
  g.Dn.Tb = dtv;
  g.Dn.T = dtt;
  g.Dn.a_off = daoff;
  g.Dn.dinv_off = ddoff;
  g.Dn.A = g.FR;
  g.Dn.Dinv = g.FDinv;
  // levels: factorisation descriptors, node lists, child slots
  g.lvl.assign(nd.H + 1, {});
  for (int x = 0; x < nn; ++x) g.lvl[N[x].height].push_back(x);
  g.ldesc.assign(nd.H + 1, nullptr);
  g.lplist.assign(nd.H + 1, nullptr);
  g.lmaxT.assign(nd.H + 1, 0);
  g.lmaxTV.assign(nd.H + 1, 0);
  g.lkids.assign(nd.H + 1, {});
  g.nkids.assign(nd.H + 1, {});
  for (int lv = 0; lv <= nd.H; ++lv) {
    std::vector<CholDesc> dsc;
    for (int x : g.lvl[lv]) {
      dsc.push_back(CholDesc{aoff[x], doff[x], -1, N[x].T, N[x].TV, -1, 0});
      g.lmaxT[lv] = std::max(g.lmaxT[lv], N[x].T);
      g.lmaxTV[lv] = std::max(g.lmaxTV[lv], N[x].TV);
    }
    TRY(dupload(h, &g.ldesc[lv], dsc));
    TRY(dupload(h, &g.lplist[lv], g.lvl[lv]));
    for (int slot = 0; slot < 2; ++slot) {
      std::vector<int> kids;
      for (int x : g.lvl[lv])
        if ((int)N[x].child.size() > slot) kids.push_back(N[x].child[slot]);
      int* dk = nullptr;
      if (!kids.empty()) TRY(dupload(h, &dk, kids));
      g.lkids[lv].push_back(dk);
      g.nkids[lv].push_back((int)kids.size());
    }
    for (int x : g.lvl[lv])
      if (N[x].child.size() > 2) return fail(h, TCG_EINVAL, "nested dissection: more than 2 children");
  }
  hm.mark("levels");
  // S^s -> frontal scatter maps (one entry per (a, b) of each patch, -1 = counted elsewhere)
  {
    std::vector<int64_t> moff(pl.npatch + 1, 0);
    for (int s2 = 0; s2 < pl.npatch; ++s2) {
      const int np2 = (int)pl.pp[s2].p_grp.size();
      moff[s2 + 1] = moff[s2] + (int64_t)np2 * np2;
    }
    std::vector<int64_t> map(std::max<int64_t>(moff[pl.npatch], 1), -1);
    // each entry (ga >= gb) goes to the front of the node eliminating the first of the two
    // groups, at the groups' frontal positions (CoarseND::fpos); patches are independent, so
    // host threads split them (the map is a pure function of the plan)
    std::atomic<int> bad{0};
    auto work = [&](int t0, int nt) {
      for (int s2 = t0; s2 < pl.npatch; s2 += nt) {
        const auto& grp = pl.pp[s2].p_grp;
        const int np2 = (int)grp.size();
        for (int a = 0; a < np2; ++a)
          for (int b = 0; b < np2; ++b) {
            const int ga = grp[a], gb = grp[b];
            if (ga < gb) continue;
            const int x = std::min(nd.node_of[ga], nd.node_of[gb]);  // postorder: descendant first
            const int fa2 = nd.fpos(x, ga), fb2 = nd.fpos(x, gb);
            if (fa2 < 0 || fb2 < 0) {
              bad = 1;
              continue;
            }
            const int r = std::max(fa2, fb2), cc = std::min(fa2, fb2);
            map[moff[s2] + (int64_t)a * np2 + b] = aoff[x] + tri_off(r >> 6, cc >> 6) + (int64_t)(r & 63) * TS + (cc & 63);
          }
      }
    };
    {
      const int nt = std::max(1, std::min(16, (int)std::thread::hardware_concurrency()));
      std::vector<std::thread> th;
      for (int t0 = 1; t0 < nt; ++t0) th.emplace_back(work, t0, nt);
      work(0, nt);
      for (auto& x : th) x.join();
    }
    if (bad) return fail(h, TCG_EINVAL, "nested dissection: coupled pair outside a front");
    TRY(dupload(h, &g.moff, moff));
    TRY(dupload(h, &g.map, map));
  }
  hm.mark("scatter-maps");
  // extend-add maps and forward gather programs
  std::vector<int64_t> xo(nn + 1, 0);
  std::vector<int> ext;
  std::vector<std::vector<std::vector<int64_t>>> src(nn);  // [node][frontal pos] sources
  for (int x = 0; x < nn; ++x) {
    src[x].assign((size_t)N[x].T * TS, {});
    for (size_t e = 0; e < N[x].V.size(); ++e) {
      const int gg = N[x].V[e];
      for (int k = pl.coarse_ptr[gg]; k < pl.coarse_ptr[gg + 1]; ++k)
        src[x][e].push_back(cidx[k] | ((int64_t)owner[cpat[k]] << 56));
    }
  }
  for (int c = 0; c < nn; ++c) {
    xo[c] = (int64_t)ext.size();
    const int p = N[c].parent;
    for (size_t i = 0; i < N[c].B.size(); ++i) {
      const int pp2 = nd.fpos(p, N[c].B[i]);
      if (pp2 < 0) return fail(h, TCG_EINVAL, "nested dissection: update row outside the parent front");
      ext.push_back(pp2);
      src[p][pp2].push_back((voff[c] + (int64_t)N[c].TV * TS + (int64_t)i) | (1ll << 55));
    }
  }
  xo[nn] = (int64_t)ext.size();
  if (ext.empty()) ext.push_back(0);
  TRY(dupload(h, &g.xo, xo));
  TRY(dupload(h, &g.ext, ext));
  std::vector<int64_t> prog, poff(nn);
  std::vector<int> vl, bl;
  std::vector<int64_t> vlo(nn), blo(nn);
  int kw = 1;
  for (int x = 0; x < nn; ++x)
    for (const auto& v : src[x]) kw = std::max(kw, (int)v.size());
  if (kw > kKwMax) return fail(h, TCG_EINVAL, "sparse coarse: more than kKwMax sources per frontal position");
  g.kw = kw;
  for (int x = 0; x < nn; ++x) {
    poff[x] = (int64_t)prog.size();  // fixed width: kw slots per position, -1 = none
    for (const auto& v : src[x])
      for (int q = 0; q < kw; ++q) prog.push_back(q < (int)v.size() ? v[q] : -1);
    vlo[x] = (int64_t)vl.size();
    vl.insert(vl.end(), N[x].V.begin(), N[x].V.end());
    blo[x] = (int64_t)bl.size();
    bl.insert(bl.end(), N[x].B.begin(), N[x].B.end());
  }
  if (prog.empty()) prog.push_back(0);
  if (vl.empty()) vl.push_back(0);
  if (bl.empty()) bl.push_back(0);
  TRY(dupload(h, &g.prog, prog));
  TRY(dupload(h, &g.vl, vl));
  TRY(dupload(h, &g.bl, bl));
  hm.mark("extend+programs");
  // stepper items: forward rows (x, I < T) and backward V columns (x, J < TV), per level, LPT
  const int nb2 = h->nbr;
  int64_t npb = 0;
  int ncnt = 0;
  std::vector<ItemDesc> fwi, bwi;
  std::vector<int> fwo(1, 0), bwo(1, 0);
  for (int lv = 0; lv <= nd.H; ++lv) {
    for (int dir = 0; dir < 2; ++dir) {
      // chunk width of this level: about one chunk per block in total (at least 4 tiles)
      int64_t lvl_tiles = 0;
      for (int x : g.lvl[lv]) {
        if (dir == 0) {
          const int rows = (N[x].parent >= 0) ? N[x].T : N[x].TV;
          for (int I = 0; I < rows; ++I) lvl_tiles += I < N[x].TV ? I + 1 : N[x].TV;
        } else {
          for (int J = 0; J < N[x].TV; ++J) lvl_tiles += N[x].T - J;
        }
      }
      // (overlap with chain blocks: the levels above the leaves go to the first ovl_chain blocks)
      const int nbl = (lv > 0 && h->ovl_chain > 0) ? h->ovl_chain : nb2;
      const int cw = (int)std::max<int64_t>(4, std::min<int64_t>(64, (lvl_tiles + nbl - 1) / nbl));
      std::vector<std::pair<int, ItemDesc>> items;
      for (int x : g.lvl[lv]) {
        ItemDesc d{};
        d.s = x;
        d.Ti = 0;
        d.Tb = N[x].TV;
        d.Tp = N[x].TB;
        d.T = N[x].T;
        d.nb = (int)N[x].B.size();
        d.np = (int)N[x].V.size();
        d.a_off = aoff[x];
        d.vec_off = voff[x];
        d.p_off = poff[x];
        d.b_off = blo[x];
        d.sbb_off = vlo[x];
        d.bc = -1;
        if (dir == 0) {
          const int rows = (N[x].parent >= 0) ? N[x].T : N[x].TV;  // the root passes nothing up
          for (int I = 0; I < rows; ++I) {
            d.I = I;
            const int Jn = I < N[x].TV ? I + 1 : N[x].TV;
            const int nch = std::max(1, (Jn + cw - 1) / cw);  // column chunks of this row
            d.bc = nch;
            d.Tp = cw;
            d.sbb_off = npb;  // first partial slot (fw items do not use the V list)
            d.Ti = ncnt++;
            npb += nch;
            for (int c = 0; c < nch; ++c) {
              d.part = c;
              items.push_back({std::min(cw, std::max(1, Jn - c * cw)) + 1, d});
            }
          }
        } else {
          for (int J = 0; J < N[x].TV; ++J) {
            d.I = J;
            const int nch = (N[x].T - J + cw - 1) / cw;  // row chunks of this column
            d.bc = nch;
            d.Tp = cw;
            d.p_off = npb;   // first partial slot
            d.Ti = ncnt++;   // arrival counter
            npb += nch;
            for (int c = 0; c < nch; ++c) {
              d.part = c;
              items.push_back({std::min(cw, N[x].T - J - c * cw), d});
            }
          }
        }
      }
      std::stable_sort(items.begin(), items.end(), [](const auto& a, const auto& b) {
        return a.first != b.first ? a.first > b.first : (a.second.s != b.second.s ? a.second.s < b.second.s : a.second.I < b.second.I);
      });
      std::vector<std::vector<ItemDesc>> blk(nb2);
      std::vector<std::pair<int64_t, int>> heap;
      for (int b = 0; b < nbl; ++b) heap.push_back({0, b});
      auto cmp = [](const std::pair<int64_t, int>& a, const std::pair<int64_t, int>& b) { return a > b; };
      std::make_heap(heap.begin(), heap.end(), cmp);
      for (auto& e : items) {
        std::pop_heap(heap.begin(), heap.end(), cmp);
        blk[heap.back().second].push_back(e.second);
        heap.back().first += e.first + 2;
        std::push_heap(heap.begin(), heap.end(), cmp);
      }
      auto& all = dir == 0 ? fwi : bwi;
      auto& off = dir == 0 ? fwo : bwo;
      for (int b = 0; b < nb2; ++b) {
        all.insert(all.end(), blk[b].begin(), blk[b].end());
        off.push_back((int)all.size());
      }
    }
  }
  if (fwi.empty()) fwi.push_back(ItemDesc{});
  if (bwi.empty()) bwi.push_back(ItemDesc{});
  {  // forward rows gather up to T_V tiles of the node rhs into the item scratch
    int maxTV = 0;
    for (const auto& n : N) maxTV = std::max(maxTV, n.TV);
    size_t need = (size_t)maxTV * TS + 16 * TS;
    need = (need + 1) & ~(size_t)1;
    h->smem_pcg = std::max(h->smem_pcg, need * sizeof(double));
  }
  {  // dataflow between levels (no grid barriers inside a coarse solve): item counts per node
    std::vector<int4> nodev(nn);
    for (int x = 0; x < nn; ++x) nodev[x] = make_int4(N[x].parent, 0, 0, 0);
    for (const auto& d : fwi)
      if (d.bc > 0) nodev[d.s].y++;
    for (const auto& d : bwi)
      if (d.bc > 0) nodev[d.s].z++;
    for (int x = 0; x < nn; ++x)
      if (N[x].parent >= 0) nodev[N[x].parent].w += nodev[x].y;
    // backward dependency: the nearest ancestor with backward items (its x_V are x's x_B
    // values, and it finishes after all of its own ancestors), -1 if none; the kernel also
    // waits for x's own forward rows (y_V)
    std::vector<int2> dep(nn);
    for (int x = 0; x < nn; ++x) {
      int a = N[x].parent;
      while (a >= 0 && nodev[a].z == 0) a = N[a].parent;
      dep[x] = a >= 0 ? make_int2(a, nodev[a].z) : make_int2(-1, 0);
    }
    TRY(dupload(h, &g.node, nodev));
    TRY(dupload(h, &g.bwdep, dep));
    for (auto& df : g.dflow) TRY(dzero(h, &df, (size_t)3 * std::max(nn, 1)));
    g.nn = nn;
  }
  TRY(dupload(h, &g.fw, fwi));
  TRY(dupload(h, &g.bw, bwi));
  TRY(dupload(h, &g.fw_off, fwo));
  TRY(dupload(h, &g.bw_off, bwo));
  for (auto& q : g.pb) TRY(dzero(h, &q, std::max<int64_t>(npb, 1) * TS));
  for (auto& q : g.cnt) TRY(dzero(h, &q, std::max(ncnt, 1)));
  return TCG_OK;
}

static tcg_status open_peer_tables(tcg_ctx* h, std::vector<std::vector<void*>>& bufs_by_rank);

static tcg_status do_setup(tcg_ctx* h) {
  HostMarks hm;
  TRY(do_plan(h));
  hm.mark("plan");
  Plan& pl = h->plan;
  CK(cudaSetDevice(h->device));
  if (const char* pe = getenv("TCG_ALLOC_PAD_KB")) {  // experiment: shift the device-memory layout
    char* pad;
    TRY(dalloc(h, &pad, (size_t)atoll(pe) * 1024));
  }
  {
    int major = 0;  // (cudaGetDeviceProperties costs milliseconds per call)
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device));
    if (major < 10) return fail(h, TCG_ECUDA, "device " + std::to_string(h->device) + " is not sm_100 class");
  }
  if (!h->stream) {
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  if (h->world > 1) {
    std::string e;
    if (!g_nccl.load(e)) return fail(h, TCG_ENCCL, e);
    ncclUniqueId id;
    std::memcpy(id.internal, h->nccl_id, 128);
    ncclResult_t r = g_nccl.commInitRank(&h->comm, h->world, id, h->rank);
    if (r != 0) return fail(h, TCG_ENCCL, std::string("ncclCommInitRank: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?"));
  }
  {
    const char* ev = getenv("TCG_STABLE");
    if (ev) h->stable_mask = atoi(ev);
    // explicit S_bb^-1 in the iteration when the local factors stream from HBM (packed X_bb
    // beyond 16 MB: cfg3-cfg5); on L2-resident working sets (cfg1, cfg2) the two row/column
    // GEMVs of X_bb are 3-5 % faster than the symmetric product (profiles/round2_notes.md)
    const char* cl = getenv("TCG_CHOL");
    h->chol_left = !(cl && std::string(cl) == "right");
    const char* si = getenv("TCG_SBBINV");
    double xbb = 0.0;
    for (const auto& q : h->plan.pp) xbb += 4.0 * q.nb * (q.nb + 1.0);
    h->sbbinv = si ? atoi(si) != 0 : xbb > 16e6;
  }
  const int P = pl.npatch;
  const int NR = h->nranks;
  if (NR > MAXR) return fail(h, TCG_EINVAL, "more than " + std::to_string(MAXR) + " ranks");

  hm.mark("pre-geometry");
  // ---- geometry ----
  Geom& G = h->G;
  for (int d = 0; d < 3; ++d) {
    G.P[d] = pl.P[d];
    G.el[d] = pl.el[d];
  }
  G.p = pl.p;
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d) G.cdim[c][d] = pl.comp_dim(c, d);
  G.nloc = pl.nloc;

  hm.mark("geometry");
  // ---- per-patch layout (offsets relative to the owning rank's allocations) ----
  std::vector<int> Ti(P), Tb(P), Tp(P), T(P), nb(P), np(P), owner(P);
  std::vector<int64_t> a_off(P), dinv_off(P), sbb_off(P), vec_off(P), aug_off(P), b_off(P + 1), p_off(P + 1);
  std::vector<int64_t> oa(NR, 0), od(NR, 0), os(NR, 0);
  std::vector<int> aug_all, b_lam_all, p_grp_all;
  std::vector<double> b_sign_all;
  int64_t ov = 0, og = 0;
  b_off[0] = p_off[0] = 0;
  h->maxT = h->maxTr = h->maxTb = h->maxTp = 0;
  for (int s = 0; s < P; ++s) {
    const PatchPlan& q = pl.pp[s];
    const int r = pl.rank_of_patch[s];
    owner[s] = r;
    Ti[s] = q.Ti;
    Tb[s] = q.Tb;
    Tp[s] = q.Tp;
    T[s] = q.Ti + q.Tb + q.Tp;
    nb[s] = q.nb;
    np[s] = q.np;
    a_off[s] = oa[r];
    oa[r] += tri_tiles(T[s]) * TSZ;
    dinv_off[s] = od[r];
    od[r] += (int64_t)(q.Ti + q.Tb) * TSZ;
    sbb_off[s] = os[r];
    os[r] += tri_tiles(q.Tb) * TSZ;
    vec_off[s] = ov;
    ov += (int64_t)T[s] * TS;
    aug_off[s] = og;
    og += (int64_t)T[s] * TS;
    aug_all.insert(aug_all.end(), q.aug.begin(), q.aug.end());
    b_off[s + 1] = b_off[s] + q.nb;
    p_off[s + 1] = p_off[s] + q.np;
    for (int t = 0; t < q.nb; ++t) {
      b_lam_all.push_back(q.b_lam[t]);
      b_sign_all.push_back((double)q.b_sign[t]);
    }
    for (int t = 0; t < q.np; ++t) p_grp_all.push_back(q.p_grp[t]);
    h->maxT = std::max(h->maxT, T[s]);
    h->maxTr = std::max(h->maxTr, q.Ti + q.Tb);
    h->maxTb = std::max(h->maxTb, q.Tb);
    h->maxTp = std::max(h->maxTp, q.Tp);
  }
  h->vec_total = ov;
  h->h_a_off = a_off;
  h->h_vec_off = vec_off;
  h->h_sbb_off = sbb_off;
  h->h_T = T;
  h->h_owner = owner;
  std::vector<int> lpp(pl.m), lpm(pl.m), lsp(pl.m), lsm(pl.m);
  std::vector<int64_t> lip(pl.m), lim(pl.m);
  for (int64_t k = 0; k < pl.m; ++k) {
    lpp[k] = (int)pl.lam_plus[k];
    lpm[k] = (int)pl.lam_minus[k];
    lsp[k] = pl.lam_plus_pos[k];
    lsm[k] = pl.lam_minus_pos[k];
    lip[k] = vec_off[lpp[k]] + (int64_t)Ti[lpp[k]] * TS + lsp[k];
    lim[k] = vec_off[lpm[k]] + (int64_t)Ti[lpm[k]] * TS + lsm[k];
  }
  std::vector<int64_t> cidx(pl.coarse_patch.size());
  std::vector<int> cpat(pl.coarse_patch.size());
  for (size_t e = 0; e < cidx.size(); ++e) {
    int s = pl.coarse_patch[e];
    cpat[e] = s;
    cidx[e] = vec_off[s] + (int64_t)(Ti[s] + Tb[s]) * TS + pl.coarse_pos[e];
  }
  const int Tc = (int)((pl.nc + TS - 1) / TS);
  h->Tc = Tc;

  hm.mark("layout");
  // ---- global uploads (shared by the local ranks) ----
  DevPlan& D = h->D;
  D.npatch = P;
  D.nranks = NR;
  D.m = pl.m;
  D.nc = pl.nc;
  D.Tc = Tc;
  D.maxT = h->maxT;
  {
    int *dTi, *dTb, *dTp, *dT, *dnb, *dnp, *daug, *dbl, *dpg, *dlpp, *dlpm, *dlsp, *dlsm, *dcp, *dcpat, *down;
    int64_t *dao, *ddo, *dso, *dvo, *dgo, *dbo, *dpo, *dlip, *dlim, *dci;
    double *dbs, *dsig, *dnu;
    TRY(dupload(h, &dTi, Ti));
    TRY(dupload(h, &dTb, Tb));
    TRY(dupload(h, &dTp, Tp));
    TRY(dupload(h, &dT, T));
    TRY(dupload(h, &dnb, nb));
    TRY(dupload(h, &dnp, np));
    TRY(dupload(h, &down, owner));
    TRY(dupload(h, &dao, a_off));
    TRY(dupload(h, &ddo, dinv_off));
    TRY(dupload(h, &dso, sbb_off));
    TRY(dupload(h, &dvo, vec_off));
    TRY(dupload(h, &dgo, aug_off));
    TRY(dupload(h, &daug, aug_all));
    TRY(dupload(h, &dbo, b_off));
    TRY(dupload(h, &dbl, b_lam_all));
    TRY(dupload(h, &dbs, b_sign_all));
    TRY(dupload(h, &dpo, p_off));
    TRY(dupload(h, &dpg, p_grp_all));
    TRY(dupload(h, &dsig, pl.sigma));
    TRY(dupload(h, &dnu, pl.nu));
    TRY(dupload(h, &dlpp, lpp));
    TRY(dupload(h, &dlpm, lpm));
    TRY(dupload(h, &dlsp, lsp));
    TRY(dupload(h, &dlsm, lsm));
    TRY(dupload(h, &dlip, lip));
    TRY(dupload(h, &dlim, lim));
    TRY(dupload(h, &dcp, pl.coarse_ptr));
    TRY(dupload(h, &dci, cidx));
    TRY(dupload(h, &dcpat, cpat));
    D.Ti = dTi; D.Tb = dTb; D.Tp = dTp; D.T = dT; D.nb = dnb; D.np = dnp; D.owner = down;
    D.a_off = dao; D.dinv_off = ddo; D.sbb_off = dso; D.vec_off = dvo; D.aug_off = dgo;
    D.aug = daug; D.b_off = dbo; D.b_lam = dbl; D.b_sign = dbs; D.p_off = dpo; D.p_grp = dpg;
    D.sigma = dsig; D.nu = dnu;
    D.lam_patch_p = dlpp; D.lam_patch_m = dlpm; D.lam_pos_p = dlsp; D.lam_pos_m = dlsm;
    D.lam_idx_p = dlip; D.lam_idx_m = dlim; D.coarse_ptr = dcp; D.coarse_idx = dci; D.coarse_patch = dcpat;
    std::vector<int64_t> bpart(b_lam_all.size());
    for (int s = 0; s < P; ++s) {
      const PatchPlan& q = pl.pp[s];
      for (int t = 0; t < q.nb; ++t) {
        const int64_t k = q.b_lam[t];
        bpart[b_off[s] + t] = (q.b_sign[t] > 0) ? lim[k] : lip[k];
      }
    }
    int64_t* dbp;
    TRY(dupload(h, &dbp, bpart));
    D.b_part = dbp;
    TRY(dalloc(h, &D.b_aown, bpart.size()));
    TRY(dalloc(h, &D.b_apart, bpart.size()));
    h->nb_total = (int64_t)bpart.size();
    TRY(dalloc(h, &D.wplus, pl.m));
    TRY(dalloc(h, &D.wminus, pl.m));
    std::vector<int> l2a((size_t)P * pl.nloc, -1);
    for (int s = 0; s < P; ++s) {
      const auto& aug = pl.pp[s].aug;
      for (size_t pos = 0; pos < aug.size(); ++pos)
        if (aug[pos] >= 0) l2a[(size_t)s * pl.nloc + aug[pos]] = (int)pos;
    }
    int* dl2a;
    TRY(dupload(h, &dl2a, l2a));
    D.loc2aug = dl2a;
  }

  hm.mark("uploads");
  // ---- 1D tables ----
  Tables1D& tb = h->tb;
  int64_t toff = 0;
  for (int d = 0; d < 3; ++d) {
    int n = pl.el[d] + pl.p;
    tb.el[d] = pl.el[d];
    tb.P[d] = pl.P[d];
    tb.h[d] = (pl.hi[d] - pl.lo[d]) / pl.P[d];
    tb.lo[d] = pl.lo[d];
    tb.off_Mb[d] = toff; toff += (int64_t)n * n;
    tb.off_Md[d] = toff; toff += (int64_t)(n - 1) * (n - 1);
    tb.off_Kb[d] = toff; toff += (int64_t)n * n;
    tb.off_C[d] = toff; toff += (int64_t)(n - 1) * n;
    tb.off_oneD[d] = toff; toff += n - 1;
    tb.off_sD[d] = toff; toff += (int64_t)pl.P[d] * (n - 1);
    tb.off_cB[d] = toff; toff += (int64_t)pl.P[d] * n;
    tb.off_sB[d] = toff; toff += (int64_t)pl.P[d] * n;
    if (pl.el[d] + 2 * pl.p > 160) return fail(h, TCG_EINVAL, "elements + 2p must be <= 160");
  }
  TRY(dalloc(h, &tb.base, toff));
  if (h->n_nl > 0) {  // nonlinear patches (nonlinear.cu): Gauss-point tables, Brauer parameters
    NlTab& NT = h->ntab;
    NT.stride = 1 + 3 * (pl.p + 1);
    int64_t o = 0;
    for (int d = 0; d < 3; ++d) {
      NT.nq[d] = pl.el[d] * (pl.p + 1);
      NT.off[d] = o;
      o += (int64_t)NT.nq[d] * NT.stride;
    }
    TRY(dalloc(h, &h->nltab, (size_t)o));
    NT.base = h->nltab;
    h->nl_smem = sizeof(double) * (size_t)o;
    if (h->nl_smem > 200 * 1024) return fail(h, TCG_EINVAL, "nonlinear patches: Gauss-point tables exceed shared memory");
    TRY(set_smem(h, (const void*)k_nl_g, h->nl_smem));
    CK(nl_assemble_smem(h->nl_smem));
    TRY(dupload(h, &h->d_nlk, h->nlk));
    std::vector<unsigned char> fl(pl.npatch);
    for (int s = 0; s < pl.npatch; ++s) fl[s] = h->is_nl(s) ? 1 : 0;
    TRY(dupload(h, &h->d_nlflag, fl));
  }
  TRY(dzero(h, &h->rho_diag, 2 * (size_t)std::max<int64_t>(pl.m, 1)));
  {
    int maxn = 0, maxel = 0;
    for (int d = 0; d < 3; ++d) {
      maxn = std::max(maxn, pl.el[d] + pl.p);
      maxel = std::max(maxel, pl.el[d]);
    }
    h->smem_tables = sizeof(double) * (2 * (pl.p + 1) + (size_t)maxel * (pl.p + 1) * (3 * maxn + 2));
  }

  if (h->source == TCG_SOURCE_PAPER) {
    // 1D projection tables (cos: n per patch index, sin: n-1), Dirichlet DOF list per patch
    std::vector<int64_t> poff(6);
    int64_t o = 0;
    for (int d = 0; d < 3; ++d) {
      const int n = pl.el[d] + pl.p;
      if (n > kProjMaxN) return fail(h, TCG_EINVAL, "source 3: elements + p per patch and direction must be <= 72");
      poff[d] = o;
      o += (int64_t)pl.P[d] * n;
      poff[3 + d] = o;
      o += (int64_t)pl.P[d] * (n - 1);
      h->ptab.off_cos[d] = poff[d];
      h->ptab.off_sin[d] = poff[3 + d];
      h->ptab.n[d] = n;
    }
    TRY(dalloc(h, &h->proj, o));
    TRY(dupload(h, &h->d_poff, poff));
    h->ptab.base = h->proj;
    std::vector<int64_t> dl, doff(1, 0);
    for (int s2 = 0; s2 < P; ++s2) {
      for (int a = 0; a < pl.nloc; ++a)
        if (pl.part[pl.local_to_global(s2, a)] == PART_DIR) dl.push_back((int64_t)s2 * pl.nloc + a);
      doff.push_back((int64_t)dl.size());
    }
    h->ndir = (int64_t)dl.size();
    if (dl.empty()) dl.push_back(0);
    TRY(dupload(h, &h->d_dlist, dl));
    TRY(dupload(h, &h->d_doff, doff));
    TRY(dzero(h, &h->aD0, dl.size()));
  }
  hm.mark("tables");
  // ---- shared memory and persistent grid ----
  int dev_sms = 148;
  CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->device));
  h->coarse_ch = (int)std::max<int64_t>(1, std::min<int64_t>(64, (int64_t)Tc * Tc / (4 * (int64_t)dev_sms)));
  h->coarse_maxch = std::max(1, (Tc + h->coarse_ch - 1) / h->coarse_ch);
  int per = 2;  // persistent blocks per SM
  {
    size_t p1 = (size_t)h->maxTb * TS;
    size_t p5 = (size_t)(h->maxTb + h->maxTp) * TS + 8 * TS;
    size_t pcs = (size_t)h->coarse_ch * TS;
    p5 = std::max(p5, (size_t)h->maxTp * TS + 16 * TS);  // whole-patch Phi_b item (p5_phi_patch)
    size_t syv = (size_t)h->maxTb * TS + 9 * TS;
    syv = std::max(syv, (size_t)2 * h->maxTb * TS + 16 * TS);  // whole-patch S_bb apply (symv_patch)
    size_t fwb = (size_t)h->maxT * TS + 8 * TS;
    size_t maxcomp = 0;
    for (int c = 0; c < 3; ++c) maxcomp = std::max(maxcomp, (size_t)pl.comp_dim(c, 0) * pl.comp_dim(c, 1) * pl.comp_dim(c, 2));
    fwb = std::max(fwb, 2 * maxcomp);
    size_t scratch = std::max(std::max(p1, p5), std::max(std::max(pcs, fwb), syv));
    scratch = (scratch + 1) & ~(size_t)1;  // keep the item cache 16-byte aligned
    h->smem_pcg = sizeof(double) * scratch;
    TRY(set_smem(h, (const void*)k_fw, h->smem_pcg));
    TRY(set_smem(h, (const void*)k_xinv_row, MMA_SMEM_DOUBLES * sizeof(double)));
    TRY(set_smem(h, (const void*)k_sinv, MMA_SMEM_DOUBLES * sizeof(double)));
    TRY(set_smem(h, (const void*)k_sbbinv, MMA_SMEM_DOUBLES * sizeof(double)));
    TRY(set_smem(h, (const void*)k_colupd, MMA_SMEM_DOUBLES * sizeof(double)));
    TRY(set_smem(h, (const void*)k_tailupd, MMA_SMEM_DOUBLES * sizeof(double)));
    TRY(set_smem(h, (const void*)k_trinv_row, MMA_SMEM_DOUBLES * sizeof(double)));
    TRY(set_smem(h, (const void*)k_tables1d, h->smem_tables));
    TRY(set_smem(h, (const void*)k_potrf, 2 * TS * PS * sizeof(double)));
    TRY(set_smem(h, (const void*)k_trsm, 2 * TS * SPAD * sizeof(double)));
    TRY(set_smem(h, (const void*)k_update, 2 * TS * SPAD * sizeof(double)));
    for (const void* f : {(const void*)k_steps<false, false>, (const void*)k_steps<true, false>,
                          (const void*)k_steps<false, true>, (const void*)k_steps<true, true>})
      TRY(set_smem(h, f, h->smem_pcg));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_steps<true, true>, NTHR, h->smem_pcg));
    if (occ < 1) return fail(h, TCG_ECUDA, "persistent stepper kernel does not fit on an SM");
    const char* ev = getenv("TCG_PCG_BLOCKS_PER_SM");
    per = std::min(occ, ev ? std::max(1, atoi(ev)) : 2);
    int total = dev_sms * per;  // co-resident blocks on this device
    h->nbr = std::max(1, total / (int)(h->world > 1 ? 1 : h->vranks));
    h->lam_chunk = std::max<int64_t>(1, (pl.m + (int64_t)NR * h->nbr - 1) / ((int64_t)NR * h->nbr));
  }

  {
    // per-iteration working set of the stepper ([X_bb; Phi_b^T], S_bb, S_pp^-1): when it is
    // L2-resident the L1 prefetch of the first tiles only adds instructions (bit 0 = off)
    double ws = 8.0 * (double)pl.nc * pl.nc;
    for (int s2 = 0; s2 < P; ++s2) {
      const double b = pl.pp[s2].nb, q = pl.pp[s2].np;
      ws += 8.0 * (b * (b + 1) / 2 + b * q) + 4.0 * b * (b + 1);
    }
    const char* fe = getenv("TCG_STEP_FLAGS");
    const int flags = fe ? atoi(fe) : (ws < 48e6 ? 1 : 0);
    CK(cudaMemcpyToSymbol(c_step_flags, &flags, sizeof(int)));
  }
  hm.mark("smem");
  // ---- coarse problem: dense S_pp^-1 (small n_c) or sparse multifrontal ----
  {
    const char* ce = getenv("TCG_COARSE");  // "dense", "sparse", default auto
    const bool want = ce ? (std::strcmp(ce, "sparse") == 0) : (pl.nc > 8192);
    h->sparse = (want && pl.nc > 0) ? 1 : 0;  // several ranks: every rank runs the whole solve
    // TCG_OVERLAP: the S_bb^-1 items leave P1 for their own list (PH_P1B) and run while their
    // block waits for dependencies of the sparse coarse solve, which needs only P1's Phi_b^T
    // rows (default: on where the coarse chain is latency-bound, i.e. without whole-patch dealing).
    // TCG_OVL_CHAIN=k: the levels above the leaves are dealt to the first k blocks of a rank,
    // which take no side items, so the dependent chain is not delayed by them.
    {
      const bool grp0 = ((int64_t)P >= 2 * (int64_t)NR * h->nbr || (getenv("TCG_GROUP") && atoi(getenv("TCG_GROUP")))) &&
                        !(getenv("TCG_NO_GROUP") && atoi(getenv("TCG_NO_GROUP")));
      h->ovl = h->sbbinv && h->sparse && (getenv("TCG_OVERLAP") ? atoi(getenv("TCG_OVERLAP")) != 0 : !grp0);
      const char* ce2 = getenv("TCG_OVL_CHAIN");
      // default with row items: 0.54 of the blocks (cfg4 sweep over k = 0 .. 280 of 296 blocks:
      // 89.8, 64.6 (24), 79.1 (48), 91.4 (96), 95.1 (160), 89.6 (192), 80.0 (224) steps/s;
      // profiles/round2_ab_overlap.txt); whole-patch side items (forced overlap): none
      const int kdef = grp0 ? 0 : (int)(0.54 * h->nbr + 0.5);
      h->ovl_chain = h->ovl ? std::max(0, std::min(h->nbr - 1, ce2 ? atoi(ce2) : kdef)) : 0;
    }
  }
  // ---- work items per rank, dealt to the rank's persistent blocks (LPT) ----
  std::vector<int> crow_owner(std::max(Tc, 1));
  for (int I = 0; I < Tc; ++I) crow_owner[I] = (int)((int64_t)I * NR / Tc);
  TRY(dupload(h, &h->d_crow_owner, crow_owner));
  // The stepper's work items and shared-memory caches are built on the host while the
  // assembly / factorisation / coarse kernels run (do_numeric calls this after launching
  // them, before the insulator precompute that needs the items).
  auto deal_phase = [&]() -> tcg_status {
    {
      auto desc = [&](int s, int I) {
        ItemDesc d{};
        d.s = s;
        d.I = I;
        d.Ti = Ti[s]; d.Tb = Tb[s]; d.Tp = Tp[s]; d.T = T[s];
        d.nb = nb[s]; d.np = np[s];
        d.a_off = a_off[s]; d.vec_off = vec_off[s]; d.b_off = b_off[s]; d.p_off = p_off[s]; d.sbb_off = sbb_off[s];
        return d;
      };
      ItemLists p1(NR), p1b(NR), p5(NR), sy(NR), pcv(NR), fw(NR), fwa(NR), bw(NR), bwc(NR), rhs(NR), e1(NR), e5(NR);
      const bool si = h->sbbinv;
      // whole-patch dealing when there are many patches per block (cfg5: 2048 patches)
      // (TCG_GROUP=1 forces it: the parity tests exercise the whole-patch items on small configs)
      const bool grp = ((int64_t)P >= 2 * (int64_t)NR * h->nbr || (getenv("TCG_GROUP") && atoi(getenv("TCG_GROUP")))) &&
                       !(getenv("TCG_NO_GROUP") && atoi(getenv("TCG_NO_GROUP")));
      const bool grp5 = grp && !(getenv("TCG_P5_SPLIT") && atoi(getenv("TCG_P5_SPLIT")));
      const bool grp_syp = grp && !(getenv("TCG_SY_SPLIT") && atoi(getenv("TCG_SY_SPLIT")));
      // with sbbinv: the Phi_b^T rows join the whole-patch S_bb^-1 item, one whole-patch Phi_b item
      // per patch in P5 (TCG_SI_MERGE=0: separate row / column items)
      const bool simerge = grp_syp && !(getenv("TCG_SI_MERGE") && atoi(getenv("TCG_SI_MERGE")) == 0);
      // (h->ovl: the S_bb^-1 items go to PH_P1B, side work of the sparse coarse solve)
      const bool ovl = h->ovl;
      const bool p1merge = simerge && !ovl;
      for (int s = 0; s < P; ++s) {
        const int r = owner[s];
        const int Trs = Ti[s] + Tb[s];
        for (int I = 0; I < T[s]; ++I) {
          const int cost = I < Trs ? I + 1 : Trs;
          if (h->dyn(s)) fw.per_rank[r].push_back({cost, desc(s, I)});
          fwa.per_rank[r].push_back({cost, desc(s, I)});
        }
        for (int J = 0; J < std::max(Trs, 1); ++J) {
          bw.per_rank[r].push_back({T[s] - J, desc(s, J)});
          if (h->dyn(s)) bwc.per_rank[r].push_back({T[s] - J, desc(s, J)});
        }
        if (h->dyn(s))
          for (int c = 0; c < 3; ++c) rhs.per_rank[r].push_back({pl.nloc / 3, desc(s, c)});
        else
          rhs.per_rank[r].push_back({T[s] * TS / 8, desc(s, -1)});
        // E1 / E5 (per-step uses of the F-apply halves, X_bb form); with sbbinv, E5 keeps the
        // split items (X_bb^T -> Y, Phi_b -> Y2) because the iteration writes Y2 every time
        for (int I = 0; I < Tb[s] + Tp[s]; ++I) {
          e1.per_rank[r].push_back({I < Tb[s] ? I + 1 : Tb[s], desc(s, I)});
          if (!si || (I >= Tb[s] && !(p1merge && Tb[s] > 0))) p1.per_rank[r].push_back({I < Tb[s] ? I + 1 : Tb[s], desc(s, I)});
        }
        for (int J = 0; J < Tb[s]; ++J) {
          if (grp5 && np[s] > 0 && !si) {  // whole-patch dealing: one item per column (fewer item starts)
            ItemDesc d = desc(s, J);
            d.part = 2;
            e5.per_rank[r].push_back({Tb[s] - J + Tp[s], d});
            p5.per_rank[r].push_back({Tb[s] - J + Tp[s], d});
            continue;
          }
          e5.per_rank[r].push_back({Tb[s] - J, desc(s, J)});
          if (!si) p5.per_rank[r].push_back({Tb[s] - J, desc(s, J)});
          if (np[s] > 0) {
            ItemDesc d = desc(s, J);
            d.part = 1;
            e5.per_rank[r].push_back({Tp[s], d});
            if (!(si && simerge)) p5.per_rank[r].push_back({Tp[s], d});
          }
        }
        if (si && simerge && np[s] > 0 && Tb[s] > 0) {  // whole-patch Phi_b item (pcg.cu p5_phi_patch)
          ItemDesc d = desc(s, 0);
          d.part = 3;
          p5.per_rank[r].push_back({Tp[s] * Tb[s], d});
        }
        if (si && Tb[s] > 0) {  // the iteration's local half: y1 = S_bb^-1 v (ItemDesc part bit 3)
          if (grp_syp) {  // + the Phi_b^T rows on the same gathered input (part bit 2)
            ItemDesc d = desc(s, 0);
            d.part = p1merge ? (8 | 4 | 2) : (8 | 2);
            (ovl ? p1b : p1).per_rank[r].push_back({Tb[s] * (Tb[s] + 1) / 2 + (p1merge ? Tp[s] * Tb[s] : 0), d});
          } else {
            for (int I = 0; I < Tb[s]; ++I) {
              ItemDesc d = desc(s, I);
              d.part = 8;
              (ovl ? p1b : p1).per_rank[r].push_back({Tb[s], d});
            }
          }
        }
        if (grp_syp) {  // whole-patch S_bb apply: every stored tile read once (pcg.cu symv_patch)
          ItemDesc d = desc(s, 0);
          d.part = 2;
          if (Tb[s] > 0) sy.per_rank[r].push_back({Tb[s] * (Tb[s] + 1) / 2, d});
        } else {
          for (int I = 0; I < Tb[s]; ++I) sy.per_rank[r].push_back({Tb[s], desc(s, I)});
        }
      }
      const int ch = h->coarse_ch;
      // PC gather programs (one per column chunk; shared by the chunk's row-block items)
      std::vector<int64_t> prog;
      std::vector<int64_t> prog_off(h->coarse_maxch), prog_len(h->coarse_maxch);
      for (int c = 0; c < h->coarse_maxch; ++c) {
        const int J0 = c * ch, J1 = std::min(Tc, J0 + ch);
        const int nE = (J1 - J0) * TS;
        prog_off[c] = (int64_t)prog.size();
        std::vector<int64_t> offs(nE + 1, 0), ent;
        for (int e = 0; e < nE; ++e) {
          const int64_t g = (int64_t)J0 * TS + e;
          if (g < pl.nc)
            for (int k = pl.coarse_ptr[g]; k < pl.coarse_ptr[g + 1]; ++k)
              ent.push_back(cidx[k] | ((int64_t)owner[cpat[k]] << 56));
          offs[e + 1] = (int64_t)ent.size();
        }
        prog.insert(prog.end(), offs.begin(), offs.end());
        prog.insert(prog.end(), ent.begin(), ent.end());
        prog_len[c] = (int64_t)prog.size() - prog_off[c];
      }
      if (prog.empty()) prog.push_back(0);
      TRY(dupload(h, &h->d_pcprog, prog));
      for (int I = 0; I < (h->sparse ? 0 : Tc); ++I)
        for (int c = 0; c < h->coarse_maxch; ++c) {
          ItemDesc d{};
          d.s = I;
          d.I = c;
          d.vec_off = prog_off[c];
          d.b_off = prog_len[c];
          pcv.per_rank[crow_owner[I]].push_back({std::min(Tc, (c + 1) * ch) - c * ch, d});
        }
      // fixed per-item overhead (tile units) of the latency-bound item phases
      TRY(deal_items(h, p1, PH_P1, 2, grp));
      TRY(deal_items(h, p1b, PH_P1B, 2, grp, h->ovl_chain));
      TRY(deal_items(h, e1, PH_E1, 2, grp));
      TRY(deal_items(h, e5, PH_E5, 2, grp));
      TRY(deal_items(h, pcv, PH_PC, 2));
      TRY(deal_items(h, p5, PH_P5, 2, grp));
      // S_bb rows are dealt one by one: whole-patch groups (one u gather per patch,
      // TCG_SY_GROUP=1) measured slower on cfg5 (patch-granular imbalance; round2_notes.md)
      const bool grp_sy = grp && getenv("TCG_SY_GROUP") && atoi(getenv("TCG_SY_GROUP")) != 0;
      TRY(deal_items(h, sy, PH_SY, 2, grp_sy));
      TRY(deal_items(h, fw, PH_FW, 2));
      TRY(deal_items(h, fwa, PH_FWA, 2));
      TRY(deal_items(h, bw, PH_BW, 2));
      TRY(deal_items(h, bwc, PH_BWC, 2));
      TRY(deal_items(h, rhs, PH_RHS, 0));
      hm.mark("deal");
    }
    // shared-memory caches of the per-iteration item lists and the lambda chunk, if they fit
    // next to the scratch at `per` blocks per SM
    {
      int max_items = 0;
      for (int gb = 0; gb < NR * h->nbr; ++gb) {
        int n = 0;
        for (int ph = 0; ph < NCACHE; ++ph) n += h->h_boff[ph][gb + 1] - h->h_boff[ph][gb];
        max_items = std::max(max_items, n);
      }
      const size_t items_b = (size_t)max_items * sizeof(ItemDesc);
      int64_t max_prog = 0;
      {
        const std::vector<ItemDesc>& hp = h->h_items[PH_PC];
        for (int gb = 0; gb < NR * h->nbr; ++gb) {
          int64_t n = 0;
          for (int j = h->h_boff[PH_PC][gb]; j < h->h_boff[PH_PC][gb + 1]; ++j) n += hp[j].b_off;
          max_prog = std::max<int64_t>(max_prog, (n + 1) & ~(int64_t)1);
        }
      }
      const size_t prog_b = (size_t)max_prog * sizeof(int64_t);
      const size_t lam_b = (size_t)h->lam_chunk * sizeof(LamC);
      int smem_sm = 0, reserved = 0;
      CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device));
      CK(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, h->device));
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, k_steps<true, true>));
      int64_t budget = (int64_t)smem_sm / per - reserved - (int64_t)fa.sharedSizeBytes - 256;
      // tile prefetch buffer first (bulk copies of the next phase's first tiles during barriers)
      {
        const char* ne = getenv("TCG_NPF");
        int npf = ne ? std::max(0, std::min(2, atoi(ne))) : 1;  // 2 tiles shrink L1 too much on the HBM-bound configs
        while (npf > 0 && (int64_t)(h->smem_pcg + (size_t)npf * TSZ * sizeof(double)) > budget) --npf;
        h->npf = npf;
        budget -= (int64_t)npf * TSZ * sizeof(double);
      }
      const char* ev = getenv("TCG_NO_SMEM_CACHE");
      const bool allow = !(ev && atoi(ev) != 0);
      h->cache_items = allow && (int64_t)(h->smem_pcg + items_b) <= budget && items_b <= 48 * 1024;
      h->cache_pcprog = allow && h->cache_items && (int64_t)(h->smem_pcg + items_b + prog_b) <= budget && prog_b <= 32 * 1024;
      const size_t used = h->smem_pcg + (h->cache_items ? items_b : 0) + (h->cache_pcprog ? prog_b : 0);
      h->cache_lam = allow && (int64_t)(used + lam_b) <= budget && lam_b <= 32 * 1024;
      size_t used2 = used + (h->cache_lam ? lam_b : 0);
      // b-position records of the patches of each block's P1 / P5 / SY items
      std::vector<int> bpl, bploff(1, 0);
      size_t max_bp = 0;
      for (int gb = 0; gb < NR * h->nbr; ++gb) {
        std::vector<int> pats;
        for (int ph : {PH_P1, PH_P1B, PH_P5, PH_SY})
          for (int j = h->h_boff[ph][gb]; j < h->h_boff[ph][gb + 1]; ++j) pats.push_back(h->h_items[ph][j].s);
        std::sort(pats.begin(), pats.end());
        pats.erase(std::unique(pats.begin(), pats.end()), pats.end());
        int off = 0;
        for (int sp : pats) {
          bpl.push_back(sp);
          bpl.push_back(off);
          off += nb[sp];
        }
        bploff.push_back((int)(bpl.size() / 2));
        max_bp = std::max(max_bp, (size_t)off * sizeof(BPos));
      }
      h->cache_bpos = allow && h->cache_items && (int64_t)(used2 + max_bp) <= budget && max_bp <= 48 * 1024;
      if (h->cache_bpos) {
        used2 += max_bp;
        for (int ph : {PH_P1, PH_P1B, PH_P5, PH_SY})
          for (int gb = 0; gb < NR * h->nbr; ++gb)
            for (int j = h->h_boff[ph][gb]; j < h->h_boff[ph][gb + 1]; ++j) {
              ItemDesc& d = h->h_items[ph][j];
              for (int q = bploff[gb]; q < bploff[gb + 1]; ++q)
                if (bpl[2 * q] == d.s) d.bc = bpl[2 * q + 1];
            }
      }
      if (bpl.empty()) bpl.assign(2, 0);
      TRY(dupload(h, &h->d_bpl, bpl));
      TRY(dupload(h, &h->d_bploff, bploff));
      for (int ph = 0; ph < NPH; ++ph) {
        std::vector<ItemDesc> all = h->h_items[ph];
        if (all.empty()) all.push_back(ItemDesc{});
        TRY(dupload(h, &h->d_items[ph], all));
        TRY(dupload(h, &h->d_boff[ph], h->h_boff[ph]));
      }
      h->smem_steps = used2 + (size_t)h->npf * TSZ * sizeof(double);
      for (const void* f : {(const void*)k_steps<false, false>, (const void*)k_steps<true, false>,
                            (const void*)k_steps<false, true>, (const void*)k_steps<true, true>})
        TRY(set_smem(h, f, h->smem_steps));
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_steps<true, true>, NTHR, h->smem_steps));
      if (occ < per) return fail(h, TCG_ECUDA, "persistent stepper: shared-memory caches broke occupancy");
    }
    if (getenv("TCG_PHASE_TIMING") && atoi(getenv("TCG_PHASE_TIMING")) != 0) {
      TRY(dzero(h, &h->tstamp, 8 * 64 + 16 + 8 * 4096 + 8 * 64));
      int mx = 1;
      for (int ph = 0; ph < NCACHE; ++ph) mx = std::max(mx, (int)h->h_items[ph].size());
      h->itime_stride = mx;
      TRY(dzero(h, &h->itime, (size_t)NCACHE * mx));
    }
    hm.mark("items+caches (overlapped)");
    return TCG_OK;
  };
  if (h->sparse) TRY(setup_sparse_coarse(h, owner, cidx, cpat));
  hm.mark("sparse-coarse");
  // ---- per-rank allocations ----
  std::vector<int> local_ranks;
  if (h->world > 1) local_ranks.push_back(h->rank);
  else
    for (int r = 0; r < h->vranks; ++r) local_ranks.push_back(r);
  h->rd.assign(local_ranks.size(), RankDev());
  for (size_t li = 0; li < local_ranks.size(); ++li) {
    RankDev& R = h->rd[li];
    R.r = local_ranks[li];
    for (int s = 0; s < P; ++s)
      if (owner[s] == R.r) R.plist.push_back(s);
    std::vector<int64_t> tstart(1, 0);
    std::vector<CholDesc> desc;
    for (int s : R.plist) {
      tstart.push_back(tstart.back() + tri_tiles(T[s]));
      desc.push_back(CholDesc{a_off[s], dinv_off[s], sbb_off[s], T[s], Ti[s] + Tb[s], Ti[s], Tb[s]});
      R.maxT = std::max(R.maxT, T[s]);
      R.maxTr = std::max(R.maxTr, Ti[s] + Tb[s]);
      R.maxTb = std::max(R.maxTb, Tb[s]);
    }
    R.ntiles = tstart.back();
    R.ndesc = (int)desc.size();
    TRY(dupload(h, &R.d_plist, R.plist));
    TRY(dupload(h, &R.d_tstart, tstart));
    TRY(dupload(h, &R.d_desc, desc));
    TRY(dalloc(h, &R.A, oa[R.r]));
    TRY(dalloc(h, &R.Dinv, od[R.r]));
    TRY(dalloc(h, &R.xscr, od[R.r]));
    TRY(dalloc(h, &R.Sbb, os[R.r]));
    if (h->sbbinv) TRY(dalloc(h, &R.SI, os[R.r]));
    TRY(dzero(h, &R.F, ov));
    TRY(dzero(h, &R.Z, ov));
    TRY(dzero(h, &R.XJ, ov));
    TRY(dzero(h, &R.JS, ov));
    TRY(dzero(h, &R.XW, ov));
    TRY(dzero(h, &R.Y, ov));
    TRY(dzero(h, &R.Y2, ov));
    TRY(dzero(h, &R.PW, ov));
    TRY(dzero(h, &R.a_loc, (size_t)P * pl.nloc));
    TRY(dzero(h, &R.lam, pl.m));
    TRY(dzero(h, &R.r0, pl.m));
    TRY(dzero(h, &R.r1, pl.m));
    TRY(dzero(h, &R.pk0, pl.m));
    TRY(dzero(h, &R.pk1, pl.m));
    TRY(dzero(h, &R.q, pl.m));
    TRY(dzero(h, &R.Ppart, (size_t)Tc * h->coarse_maxch * TS));
    TRY(dzero(h, &R.Pc, pl.nc));
    TRY(dzero(h, &R.partials, 2 * (size_t)h->nbr + 1));
    TRY(dzero(h, &R.hist, (size_t)(h->n_steps + 1) * (h->max_iter + 1)));
    TRY(dzero(h, &R.iters, (size_t)h->n_steps + 1));
    TRY(dzero(h, &R.bar, 1));
    TRY(dzero(h, &R.st, 1));
    TRY(dzero(h, &R.derr, 1));
    for (int s : R.plist)
      if (h->is_nl(s)) R.nlist.push_back(s);
    if (!R.nlist.empty()) {
      std::vector<int64_t> nts(1, 0);
      std::vector<CholDesc> nd;
      for (int s : R.nlist) {
        nts.push_back(nts.back() + tri_tiles(T[s]));
        nd.push_back(CholDesc{a_off[s], dinv_off[s], sbb_off[s], T[s], Ti[s] + Tb[s], Ti[s], Tb[s]});
        R.nl_maxT = std::max(R.nl_maxT, T[s]);
        R.nl_maxTr = std::max(R.nl_maxTr, Ti[s] + Tb[s]);
        R.nl_maxTb = std::max(R.nl_maxTb, Tb[s]);
      }
      TRY(dupload(h, &R.d_nldesc, nd));
      R.nl_ntiles = nts.back();
      TRY(dupload(h, &R.d_nlist, R.nlist));
      TRY(dupload(h, &R.d_ntstart, nts));
      const int64_t nqp = (int64_t)h->ntab.nq[0] * h->ntab.nq[1] * h->ntab.nq[2];
      TRY(dalloc(h, &R.Q, (size_t)R.nlist.size() * 9 * nqp));
      // element tangent matrices (p <= 3; TCG_NL_ELEM=0: the per-entry Gauss-point kernel)
      const size_t ke = nl_elem_doubles(pl.p, pl.el[0] * pl.el[1] * pl.el[2]);
      const char* ne = getenv("TCG_NL_ELEM");
      if (ke > 0 && !(ne && atoi(ne) == 0)) TRY(dalloc(h, &R.Kel, R.nlist.size() * ke));
    }
    if (h->n_nl > 0) {  // every rank joins the Newton loop (right-hand side vector, iterates, norms)
      TRY(dzero(h, &R.gnl, ov));
      TRY(dzero(h, &R.a_old, (size_t)P * pl.nloc));
      TRY(dzero(h, &R.a_k, (size_t)P * pl.nloc));
      TRY(dzero(h, &R.nl_part, 2 * (size_t)NL_NORM_BLOCKS));
    }
    if (li == 0) {
      const int Tcd = h->sparse ? 1 : Tc;  // the sparse coarse keeps no dense factor / inverse
      TRY(dalloc(h, &R.C, (size_t)tri_tiles(Tcd) * TSZ));
      TRY(dalloc(h, &R.Cinv, (size_t)Tcd * TSZ));
      TRY(dalloc(h, &R.CX, (size_t)tri_tiles(Tcd) * TSZ));
      TRY(dalloc(h, &R.Sinv, (size_t)Tcd * Tcd * TSZ));
    } else {
      R.C = h->rd[0].C;
      R.Cinv = h->rd[0].Cinv;
      R.CX = h->rd[0].CX;
      R.Sinv = h->rd[0].Sinv;
    }
  }
  hm.mark("rank-alloc");
  // ---- per-rank pointer tables (peer memory for real ranks) ----
  {
    std::vector<std::vector<void*>> bufs(NR);  // [rank][buffer] in a fixed order
    for (auto& R : h->rd)
      bufs[R.r] = {R.A, R.Sbb, R.Z, R.XW, R.Y, R.PW, R.lam, R.r0, R.r1, R.pk0, R.pk1, R.Ppart, R.bar, R.a_loc, R.Y2};
    if (h->world > 1) TRY(open_peer_tables(h, bufs));
    for (int r = 0; r < NR; ++r) {
      D.Ar[r] = (double*)bufs[r][0];
      D.Sbbr[r] = (double*)bufs[r][1];
    }
    h->D.me = 0;
    for (auto& R : h->rd) D.SIr[R.r] = R.SI;  // own patches only (items run on the owner)
    for (auto& R : h->rd) {
      R.D = D;
      R.D.me = R.r;
      R.D.A = R.A;
      R.D.Dinv = R.Dinv;
      R.D.Sbb = R.Sbb;
      R.D.C = R.C;
      R.D.Cinv = R.Cinv;
    }
    // keep the table for step_args
    h->peer_bufs = bufs;
  }
  std::vector<CholDesc> cdesc(1, CholDesc{0, 0, -1, Tc, Tc, -1, 0});
  TRY(dupload(h, &h->d_cdesc, cdesc));
  std::vector<InvDesc> cinv(1, InvDesc{0, 0, 0, 0, Tc});
  TRY(dupload(h, &h->d_cinv, cinv));
  // colour lists (parity classes) for the conflict-free coarse scatter
  {
    std::vector<int> colour_all;
    h->colour_off.assign(9, 0);
    for (int c = 0; c < 8; ++c) {
      for (int s = 0; s < P; ++s) {
        int ix = s % pl.P[0], iy = (s / pl.P[0]) % pl.P[1], iz = s / (pl.P[0] * pl.P[1]);
        if (((ix & 1) | ((iy & 1) << 1) | ((iz & 1) << 2)) == c) colour_all.push_back(s);
      }
      h->colour_off[c + 1] = (int64_t)colour_all.size();
    }
    TRY(dupload(h, &h->d_colour, colour_all));
  }
  // readout maps: glued edge -> (patch*nloc + local) of its lowest-id owner; gathered a
  {
    std::vector<int64_t> src(pl.nedges, -1);
    for (int s = 0; s < P; ++s) {  // local DOF a -> glued edge, in local order (no divisions)
      const int sx = s % pl.P[0], sy = (s / pl.P[0]) % pl.P[1], sz = s / (pl.P[0] * pl.P[1]);
      const int64_t o0 = (int64_t)sx * (pl.n[0] - 1), o1 = (int64_t)sy * (pl.n[1] - 1), o2 = (int64_t)sz * (pl.n[2] - 1);
      int a = 0;
      for (int c = 0; c < 3; ++c)
        for (int k = 0; k < pl.comp_dim(c, 2); ++k)
          for (int j = 0; j < pl.comp_dim(c, 1); ++j)
            for (int i = 0; i < pl.comp_dim(c, 0); ++i, ++a) {
              const int64_t g = pl.edge_id(c, o0 + i, o1 + j, o2 + k);
              if (src[g] < 0) src[g] = (int64_t)s * pl.nloc + a;
            }
    }
    TRY(dupload(h, &h->d_glued_src, src));
    TRY(dalloc(h, &h->glued, pl.nedges));
    TRY(dalloc(h, &h->a_all, (size_t)P * pl.nloc));
  }
  if (!h->h_st) {
    {
      std::lock_guard<std::mutex> lk(tcg_ctx::pinned_mu());
      if (!tcg_ctx::pinned_free().empty()) {
        h->h_st = tcg_ctx::pinned_free().back();
        tcg_ctx::pinned_free().pop_back();
      }
    }
    if (!h->h_st) CK(cudaMallocHost(&h->h_st, sizeof(PcgState)));
  }
  if (getenv("TCG_DEBUG_KEEP") && atoi(getenv("TCG_DEBUG_KEEP")) != 0) {
    TRY(dalloc(h, &h->dbgA, h->rd[0].A ? (size_t)oa[h->rd[0].r] : 1));
    TRY(dalloc(h, &h->dbgC, (size_t)tri_tiles(Tc) * TSZ));
  }
  h->bar_round = 0;
  TRY(sync_ranks(h));
  hm.mark("tables+state");
  TRY(do_numeric(h, deal_phase));
  hm.mark("numeric");
  h->setup_done = true;
  return TCG_OK;
}

// Exchange CUDA IPC handles of every rank's buffers through NCCL and open the peers' ones.
static tcg_status open_peer_tables(tcg_ctx* h, std::vector<std::vector<void*>>& bufs) {
  const int NR = h->nranks;
  const size_t nb = bufs[h->rank].size();
  std::vector<cudaIpcMemHandle_t> mine(nb);
  for (size_t i = 0; i < nb; ++i) CK(cudaIpcGetMemHandle(&mine[i], bufs[h->rank][i]));
  const size_t bytes = nb * sizeof(cudaIpcMemHandle_t);
  char *dsend, *drecv;
  TRY(dalloc(h, &dsend, bytes));
  TRY(dalloc(h, &drecv, bytes * NR));
  CK(cudaMemcpyAsync(dsend, mine.data(), bytes, cudaMemcpyHostToDevice, h->stream));
  ncclResult_t r = g_nccl.allGather(dsend, drecv, bytes, ncclInt8, h->comm, h->stream);
  if (r != 0) return fail(h, TCG_ENCCL, "ncclAllGather (IPC handles) failed");
  std::vector<cudaIpcMemHandle_t> all(nb * NR);
  CK(cudaMemcpyAsync(all.data(), drecv, bytes * NR, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  for (int q = 0; q < NR; ++q) {
    if (q == h->rank) continue;
    bufs[q].assign(nb, nullptr);
    for (size_t i = 0; i < nb; ++i) {
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, all[q * nb + i], cudaIpcMemLazyEnablePeerAccess));
      h->ipc_opened.push_back(p);
      bufs[q][i] = p;
    }
  }
  return TCG_OK;
}

// =========================================================================================
// steps
// =========================================================================================
static void prof_begin(tcg_ctx* h, int id) {
  if (h->prof_id != id) return;
  if (2 * h->prof_used + 2 > h->prof_ev.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    h->prof_ev.push_back(a);
    h->prof_ev.push_back(b);
  }
  cudaEventRecord(h->prof_ev[2 * h->prof_used], h->stream);
}
static void prof_end(tcg_ctx* h, int id) {
  if (h->prof_id != id) return;
  cudaEventRecord(h->prof_ev[2 * h->prof_used + 1], h->stream);
  h->prof_used++;
}
static void prof_collect(tcg_ctx* h) {
  for (size_t i = 0; i < h->prof_used; ++i) {
    h->prof_ms += elapsed_ms(h->prof_ev[2 * i], h->prof_ev[2 * i + 1]);
    h->prof_count += 1;
  }
  h->prof_used = 0;
}

static StepArgs step_args(tcg_ctx* h) {
  StepArgs A{};
  const auto& B = h->peer_bufs;
  for (int r = 0; r < h->nranks; ++r) {
    A.Z[r] = (double*)B[r][2];
    A.XW[r] = (double*)B[r][3];
    A.Y[r] = (double*)B[r][4];
    A.PW[r] = (double*)B[r][5];
    A.lam[r] = (double*)B[r][6];
    A.r[0][r] = (double*)B[r][7];
    A.r[1][r] = (double*)B[r][8];
    A.pk[0][r] = (double*)B[r][9];
    A.pk[1][r] = (double*)B[r][10];
    A.Ppart[r] = (double*)B[r][11];
    A.bar[r] = (BarMem*)B[r][12];
    A.a_loc[r] = (double*)B[r][13];
    A.Y2[r] = (double*)B[r][14];
  }
  for (auto& R : h->rd) {  // own-only buffers of the local ranks
    A.F[R.r] = R.F;
    A.XJ[R.r] = R.XJ;
    A.JS[R.r] = R.JS;
    A.Sinv[R.r] = R.Sinv;
    A.Pc[R.r] = R.Pc;
    A.partials[R.r] = R.partials;
    A.hist[R.r] = R.hist;
    A.iters[R.r] = R.iters;
    A.st[R.r] = R.st;
  }
  A.crow_owner = h->d_crow_owner;
  A.ch = h->coarse_ch;
  A.maxch = h->coarse_maxch;
  for (int ph = 0; ph < NPH; ++ph) {
    A.items[ph] = h->d_items[ph];
    A.boff[ph] = h->d_boff[ph];
  }
  A.cache_items = h->cache_items;
  A.cache_pcprog = h->cache_pcprog;
  A.cache_bpos = h->cache_bpos;
  A.bpl = h->d_bpl;
  A.bploff = h->d_bploff;
  A.pcprog = h->d_pcprog;
  A.cache_lam = h->cache_lam;
  A.scratch = (int)(h->smem_pcg / sizeof(double));
  A.npf = h->npf;
  A.warm = h->warm;
  A.warm_base = (int)h->warm_base;
  for (auto& R : h->rd) {
    A.Wr[R.r] = R.Wr;
    A.FWr[R.r] = R.FWr;
    A.dsave[R.r] = R.dsave;
    A.wpart[R.r] = R.wpart;
  }
  A.mode = 0;
  A.dbg_stop = getenv("TCG_DEBUG_STOP") ? atoi(getenv("TCG_DEBUG_STOP")) : 0;
  A.sparse = h->sparse;
  if (h->sparse) {
    const auto& g = h->ndd;
    A.cf_levels = h->nd.H + 1;
    A.cf_fw = g.fw;
    A.cf_fw_off = g.fw_off;
    A.cf_bw = g.bw;
    A.cf_bw_off = g.bw_off;
    A.FR = g.FR;
    A.cf_prog = g.prog;
    A.cf_kw = g.kw;
    A.cf_vl = g.vl;
    A.cf_bl = g.bl;
    for (size_t li = 0; li < h->rd.size(); ++li) {
      const int r = h->rd[li].r;
      A.CW[r] = g.CW[li];
      A.Pcs[r] = g.Pcs[li];
      A.cf_pb[r] = g.pb[li];
      A.cf_cnt[r] = g.cnt[li];
      A.cf_dflow[r] = g.dflow[li];
    }
    A.cf_node = g.node;
    A.cf_bwdep = g.bwdep;
    A.cf_nn = g.nn;
    A.cf_sync = getenv("TCG_CF_LEVELSYNC") && atoi(getenv("TCG_CF_LEVELSYNC")) != 0;
  }
  A.tstamp = h->tstamp;
  A.itime = h->itime;
  A.itime_stride = h->itime_stride;
  A.rtol = h->rtol;
  A.max_iter = h->max_iter;
  A.nranks = h->nranks;
  A.nbr = h->nbr;
  A.rank_base = (h->world > 1) ? h->rank : 0;
  A.sys_scope = (h->world > 1) ? 1 : 0;
  A.lam_chunk = h->lam_chunk;
  A.source = h->source;
  A.dlist = h->d_dlist;
  A.aD0 = h->aD0;
  A.nd = (h->source == TCG_SOURCE_PAPER) ? h->ndir : 0;
  A.src_amp = h->src_amp;
  A.src_freq = h->src_freq;
  A.dt = h->T / h->n_steps;
  A.step0 = (int)h->steps_done;
  A.nsteps = 0;
  A.hist_off = h->hist_len;
  A.round0 = h->bar_round;
  A.tb = h->tb;
  A.G = h->G;
  return A;
}

// The warm-start state (k, first step of the history) decides which barriers a launch runs;
// every rank must agree or the monotone barrier counters would pair different rounds. One
// NCCL max-allreduce of (k, base, -k, -base) per tcg_step on world > 1 handles.
static tcg_status agree_warm(tcg_ctx* h) {
  if (!h->agree_buf) TRY(dzero(h, &h->agree_buf, 4));
  const double v[4] = {(double)h->warm, (double)h->warm_base, -(double)h->warm, -(double)h->warm_base};
  CK(cudaMemcpyAsync(h->agree_buf, v, sizeof v, cudaMemcpyHostToDevice, h->stream));
  ncclResult_t r = g_nccl.allReduce(h->agree_buf, h->agree_buf, 4, ncclFloat64, ncclMax, h->comm, h->stream);
  if (r != 0) return fail(h, TCG_ENCCL, "ncclAllReduce (warm-start agreement) failed");
  double w[4];
  CK(cudaMemcpyAsync(w, h->agree_buf, sizeof w, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (w[0] != -w[2] || w[1] != -w[3])
    return fail(h, TCG_EINVAL, "tcg_set_warm_start is collective: ranks disagree on k or on the step it was set at");
  return TCG_OK;
}

// n implicit-Euler steps in ONE persistent cooperative launch (k_steps) over all local ranks.
// newton_it != nullptr: one linear solve of a Newton iterate of step steps_done (n = 1; the
// mass term reads a_old, the right-hand side adds gnl); its PCG iterations and final relres go
// to *newton_it / *newton_rel and its history is appended, but the step is not counted.
static tcg_status do_steps(tcg_ctx* h, int n, int* newton_it = nullptr, double* newton_rel = nullptr) {
  if (n <= 0) return TCG_OK;
  if (h->steps_done + n > h->n_steps) return fail(h, TCG_EINVAL, "more steps than set_time allows (n_steps)");
  for (auto& R : h->rd) CK(cudaMemsetAsync(R.st, 0, sizeof(PcgState), h->stream));
  if (h->sparse)
    for (auto* df : h->ndd.dflow) CK(cudaMemsetAsync(df, 0, 3 * sizeof(unsigned int) * std::max(h->ndd.nn, 1), h->stream));
  if (h->warm)
    for (auto& R : h->rd)
      if (!R.Wr) {  // warm-start rings: k solutions and k F-products at the lambda level
        const size_t m = (size_t)std::max<int64_t>(1, h->plan.m);
        TRY(dzero(h, &R.Wr, (size_t)KW * m));
        TRY(dzero(h, &R.FWr, (size_t)KW * m));
        TRY(dzero(h, &R.dsave, m));
        TRY(dzero(h, &R.wpart, (size_t)2 * h->nbr * KW_NV));
      }
  if (h->world > 1) TRY(agree_warm(h));
  StepArgs A = step_args(h);
  A.nsteps = n;
  if (newton_it) {
    for (auto& R : h->rd) {
      A.a_old[R.r] = R.a_old;
      A.gnl[R.r] = R.gnl;
    }
    A.hist_off = 0;  // each solve's history starts at the buffer's head (copied out below)
  }
  DevPlan D = h->D;
  void* args[] = {(void*)&D, (void*)&A};
  const int grid = h->nbr * (int)h->rd.size();
  prof_begin(h, 7);
  const void* fn = (h->nranks > 1) ? (h->cache_bpos ? (const void*)k_steps<true, true> : (const void*)k_steps<true, false>)
                                     : (h->cache_bpos ? (const void*)k_steps<false, true> : (const void*)k_steps<false, false>);
  CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(NTHR), args, h->smem_steps, h->stream));
  ++h->nlaunch;
  prof_end(h, 7);

  RankDev& R0 = h->rd[0];
  CK(cudaMemcpyAsync(h->h_st, R0.st, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  h->d2h_bytes += (int64_t)sizeof(PcgState);
  CK(cudaStreamSynchronize(h->stream));
  prof_collect(h);
  const PcgState hs = *h->h_st;
  const int64_t hl = hs.counter[2];
  h->bar_round = hs.counter[3];  // barrier rounds of every rank after this launch
  std::vector<int> it(n);
  CK(cudaMemcpy(it.data(), R0.iters + h->steps_done, sizeof(int) * n, cudaMemcpyDeviceToHost));
  std::vector<double> hh(std::max<int64_t>(hl, 1));
  // histories are written by rank 0 (block 0); on other ranks use the local iteration counts
  const bool have_hist = (h->world == 1 || h->rank == 0);
  if (have_hist && hl > 0)
    CK(cudaMemcpy(hh.data(), R0.hist + (newton_it ? 0 : h->hist_len), sizeof(double) * hl, cudaMemcpyDeviceToHost));
  h->d2h_bytes += (int64_t)(sizeof(int) * n + sizeof(double) * hl);
  if (hs.failed) {
    std::ostringstream o;
    o << "PCG did not converge: step " << hs.rp + 1 << ", iterations " << hs.iter << ", relres "
      << (hs.rho0 > 0 ? std::sqrt(std::max(hs.rz, 0.0) / hs.rho0) : 0.0) << (hs.nan ? " (curvature/NaN guard)" : "");
    h->broken = true;
    return fail(h, TCG_ENOCONV, o.str());
  }
  if (newton_it) {
    *newton_it = it[0];
    *newton_rel = have_hist ? hh[it[0]] : 0.0;
    if (have_hist) h->hist_all.insert(h->hist_all.end(), hh.begin(), hh.begin() + hl);
    else h->hist_all.insert(h->hist_all.end(), (size_t)hl, 0.0);
    h->hist_len += hl;
    return TCG_OK;
  }
  int64_t off = 0;
  for (int i = 0; i < n; ++i) {
    h->iters.push_back(it[i]);
    h->hist_per_step.push_back(it[i] + 1);
    h->final_rel.push_back(have_hist ? hh[off + it[i]] : 0.0);
    off += it[i] + 1;
    h->total_iters += it[i];
  }
  if (have_hist) h->hist_all.insert(h->hist_all.end(), hh.begin(), hh.begin() + hl);
  else h->hist_all.insert(h->hist_all.end(), (size_t)hl, 0.0);
  h->hist_len += hl;
  h->steps_done += n;
  return TCG_OK;
}

// One implicit-Euler step with nonlinear patches (R25): Newton from
// a_0 = a^l; iterate k re-assembles and factorises at a_k (do_numeric newton mode: the
// nonlinear patches' tangent matrices and g = (Kt - K) a_k), then one linear IETI-DP solve of
// J(a_k) a_{k+1} = g + (sigma/dt) M a^l + j^(l+1) in the persistent stepper. Stops when
// ||a_{k+1} - a_k|| <= newton_tol ||a_{k+1}|| (all patches' local vectors; fixed-order sums
// of per-block partials in rank order, NCCL sum across processes).
static tcg_status do_newton_step(tcg_ctx* h) {
  const Plan& pl = h->plan;
  const int64_t nall = (int64_t)pl.npatch * pl.nloc;
  const size_t nb = sizeof(double) * (size_t)nall;
  for (auto& R : h->rd) CK(cudaMemcpyAsync(R.a_old, R.a_loc, nb, cudaMemcpyDeviceToDevice, h->stream));
  int total = 0, it = 0;
  double rel = 0.0, inc = 0.0;
  std::vector<double> part(2 * NL_NORM_BLOCKS);
  for (it = 1;; ++it) {
    for (auto& R : h->rd) CK(cudaMemcpyAsync(R.a_k, R.a_loc, nb, cudaMemcpyDeviceToDevice, h->stream));
    TRY(do_numeric(h, nullptr, true));
    int its = 0;
    TRY(do_steps(h, 1, &its, &rel));
    total += its;
    double sums[2] = {0.0, 0.0};
    for (auto& R : h->rd) {
      k_nl_norms<<<NL_NORM_BLOCKS, 256, 0, h->stream>>>(R.a_loc, R.a_k, h->D.owner, R.r, pl.nloc, nall, R.nl_part);
      ++h->nlaunch;
      CKL();
      CK(cudaMemcpyAsync(part.data(), R.nl_part, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      for (int b = 0; b < NL_NORM_BLOCKS; ++b) {
        sums[0] += part[2 * b];
        sums[1] += part[2 * b + 1];
      }
    }
    if (h->world > 1) {
      if (!h->agree_buf) TRY(dzero(h, &h->agree_buf, 4));
      CK(cudaMemcpyAsync(h->agree_buf, sums, sizeof sums, cudaMemcpyHostToDevice, h->stream));
      ncclResult_t r = g_nccl.allReduce(h->agree_buf, h->agree_buf, 2, ncclFloat64, ncclSum, h->comm, h->stream);
      if (r != 0) return fail(h, TCG_ENCCL, "ncclAllReduce (Newton increment) failed");
      CK(cudaMemcpyAsync(sums, h->agree_buf, sizeof sums, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    inc = sums[1] > 0.0 ? std::sqrt(sums[0] / sums[1]) : 0.0;
    h->solve_its.push_back(its);
    h->solve_inc.push_back(inc);
    if (inc <= h->newton_tol) break;
    if (it >= h->newton_max) {
      h->broken = true;
      std::ostringstream o;
      o << "Newton did not converge: step " << h->steps_done + 1 << ", " << it << " iterations, increment " << inc;
      return fail(h, TCG_ENOCONV, o.str());
    }
  }
  h->newton_its.push_back(it);
  h->hist_per_step.push_back(total + it);
  h->iters.push_back(total);
  h->final_rel.push_back(rel);
  h->total_iters += total;
  h->steps_done += 1;
  return TCG_OK;
}

// gather the local coefficient vectors of every patch (from its owner) into a_all
__global__ void k_gather_aloc(double* out, StepArgs A, const int* owner, int nloc, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = A.a_loc[owner[i / nloc]][i];
}

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

tcg_status tcg_create(tcg_handle* out, int device, int rank, int world, const unsigned char* nccl_id, void* cuda_stream) {
  if (!out) return TCG_EINVAL;
  *out = nullptr;
  if (world < 1 || world > MAXR || rank < 0 || rank >= world || device < 0) return TCG_EINVAL;
  if (world > 1 && !nccl_id) return TCG_EINVAL;
  tcg_ctx* h = new tcg_ctx();
  h->device = device;
  h->rank = rank;
  h->world = world;
  if (nccl_id) std::memcpy(h->nccl_id, nccl_id, 128);
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  *out = h;
  return TCG_OK;
}

tcg_status tcg_nccl_unique_id(unsigned char* out) {
  if (!out) return TCG_EINVAL;
  std::string e;
  if (!g_nccl.load(e) || !g_nccl.getUniqueId) return TCG_ENCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != 0) return TCG_ENCCL;
  std::memcpy(out, id.internal, 128);
  return TCG_OK;
}

tcg_status tcg_set_virtual_ranks(tcg_handle h, int vranks) {
  if (!h) return TCG_EINVAL;
  if (h->planned || h->setup_done) return fail(h, TCG_ESTATE, "set_virtual_ranks after plan/setup");
  if (vranks < 1 || vranks > MAXR) return fail(h, TCG_EINVAL, "virtual ranks 1.." + std::to_string(MAXR));
  if (vranks > 1 && h->world > 1) return fail(h, TCG_EINVAL, "virtual ranks need world == 1");
  h->vranks = vranks;
  return TCG_OK;
}

tcg_status tcg_set_patches(tcg_handle h, const int npatch[3], const double lo[3], const double hi[3], int degree_p,
                           const int elems[3]) {
  if (!h) return TCG_EINVAL;
  if (h->planned || h->setup_done) return fail(h, TCG_ESTATE, "set_patches after plan/setup");
  if (!npatch || !lo || !hi || !elems) return fail(h, TCG_EINVAL, "null argument");
  if (degree_p < 1) return fail(h, TCG_EINVAL, "degree p must be >= 1");
  for (int d = 0; d < 3; ++d) {
    if (npatch[d] < 1 || elems[d] < 1) return fail(h, TCG_EINVAL, "patch/element counts must be >= 1");
    if (!(lo[d] < hi[d])) return fail(h, TCG_EINVAL, "degenerate box");
    h->plan.P[d] = npatch[d];
    h->plan.el[d] = elems[d];
    h->plan.lo[d] = lo[d];
    h->plan.hi[d] = hi[d];
  }
  h->plan.p = degree_p;
  h->have_patches = true;
  return TCG_OK;
}

tcg_status tcg_set_materials(tcg_handle h, const double* sigma, const double* nu, size_t n) {
  if (!h) return TCG_EINVAL;
  if (h->planned || h->setup_done) return fail(h, TCG_ESTATE, "set_materials after plan/setup");
  if (!h->have_patches) return fail(h, TCG_ESTATE, "set_patches first");
  size_t P = (size_t)h->plan.P[0] * h->plan.P[1] * h->plan.P[2];
  if (!sigma || !nu || n != P) return fail(h, TCG_EINVAL, "materials need one sigma and one nu per patch (" + std::to_string(P) + ")");
  for (size_t s = 0; s < n; ++s) {
    if (!(sigma[s] >= 0) || !std::isfinite(sigma[s])) return fail(h, TCG_EINVAL, "sigma must be finite and >= 0");
    if (!(nu[s] > 0) || !std::isfinite(nu[s])) return fail(h, TCG_EINVAL, "nu must be finite and > 0");
  }
  h->plan.sigma.assign(sigma, sigma + n);
  h->plan.nu.assign(nu, nu + n);
  h->have_materials = true;
  return TCG_OK;
}

tcg_status tcg_set_source(tcg_handle h, int kind, const double* params, size_t nparams) {
  if (!h) return TCG_EINVAL;
  if (h->setup_done) return fail(h, TCG_ESTATE, "set_source after setup");
  if (kind < 0 || kind > 3) return fail(h, TCG_EINVAL, "unknown source kind");
  const size_t maxp = kind == 1 ? 2 : (kind >= 2 ? 1 : 0);
  if (nparams > maxp || (nparams > 0 && !params))
    return fail(h, TCG_EINVAL, "source kind " + std::to_string(kind) + " takes at most " + std::to_string(maxp) + " parameters");
  double amp = 1.0, freq = 1.0;
  if (nparams >= 1) amp = params[0];
  if (nparams >= 2) freq = params[1];
  if (!std::isfinite(amp) || !std::isfinite(freq)) return fail(h, TCG_EINVAL, "source parameters must be finite");
  h->source = kind;
  h->src_amp = amp;
  h->src_freq = freq;
  return TCG_OK;
}

tcg_status tcg_set_nonlinear(tcg_handle h, const double* k, size_t n, double newton_tol, int newton_max) {
  if (!h) return TCG_EINVAL;
  if (h->planned || h->setup_done) return fail(h, TCG_ESTATE, "set_nonlinear after plan/setup");
  if (!h->have_patches) return fail(h, TCG_ESTATE, "set_patches first");
  const size_t P = (size_t)h->plan.P[0] * h->plan.P[1] * h->plan.P[2];
  if (n != 0 && (!k || n != P)) return fail(h, TCG_EINVAL, "one (k1, k2, k3) triple per patch (" + std::to_string(P) + ")");
  if (!(newton_tol > 0) || !std::isfinite(newton_tol) || newton_max < 1)
    return fail(h, TCG_EINVAL, "newton_tol > 0 and newton_max >= 1 required");
  int cnt = 0;
  for (size_t s = 0; s < n; ++s) {
    const double k1 = k[3 * s], k2 = k[3 * s + 1], k3 = k[3 * s + 2];
    if (!std::isfinite(k1) || !std::isfinite(k2) || !std::isfinite(k3))
      return fail(h, TCG_EINVAL, "Brauer parameters must be finite");
    if (k1 == 0.0 && k2 == 0.0 && k3 == 0.0) continue;
    if (!(k1 >= 0.0) || !(k2 >= 0.0) || !(k3 > 0.0))
      return fail(h, TCG_EINVAL, "Brauer parameters need k1 >= 0, k2 >= 0, k3 > 0 (patch " + std::to_string(s) + ")");
    ++cnt;
  }
  if (cnt > 0 && h->plan.p > NL_MAXP) return fail(h, TCG_EINVAL, "nonlinear patches need p <= " + std::to_string(NL_MAXP));
  if (cnt > 0 && h->warm) return fail(h, TCG_EINVAL, "warm start is not available with nonlinear patches");
  h->nlk.assign(k ? k : nullptr, k ? k + 3 * n : nullptr);
  h->n_nl = cnt;
  h->newton_tol = newton_tol;
  h->newton_max = newton_max;
  return TCG_OK;
}

tcg_status tcg_get_newton(tcg_handle h, int* newton_iters, size_t nsteps, int* solve_iters, double* increments,
                          size_t nsolves) {
  if (!h) return TCG_EINVAL;
  if (nsteps > h->newton_its.size())
    return fail(h, TCG_EINVAL, "only " + std::to_string(h->newton_its.size()) + " Newton steps recorded");
  if (nsolves > h->solve_its.size())
    return fail(h, TCG_EINVAL, "only " + std::to_string(h->solve_its.size()) + " linear solves recorded");
  for (size_t i = 0; i < nsteps; ++i)
    if (newton_iters) newton_iters[i] = h->newton_its[i];
  for (size_t i = 0; i < nsolves; ++i) {
    if (solve_iters) solve_iters[i] = h->solve_its[i];
    if (increments) increments[i] = h->solve_inc[i];
  }
  return TCG_OK;
}

tcg_status tcg_set_time(tcg_handle h, double T, int n_steps) {
  if (!h) return TCG_EINVAL;
  if (h->setup_done) return fail(h, TCG_ESTATE, "set_time after setup");
  if (!(T > 0) || n_steps < 1) return fail(h, TCG_EINVAL, "T > 0 and n_steps >= 1 required");
  h->T = T;
  h->n_steps = n_steps;
  h->have_time = true;
  return TCG_OK;
}

tcg_status tcg_set_solver(tcg_handle h, double rtol, int max_iter, int scaling, int tree_order) {
  if (!h) return TCG_EINVAL;
  if (h->planned || h->setup_done) return fail(h, TCG_ESTATE, "set_solver after plan/setup");
  if (!(rtol > 0) || max_iter < 1 || (scaling != 0 && scaling != 1) || (tree_order != 0 && tree_order != 1))
    return fail(h, TCG_EINVAL, "invalid solver parameters");
  h->rtol = rtol;
  h->max_iter = max_iter;
  h->scaling = scaling;
  h->tree_order = tree_order;
  return TCG_OK;
}

tcg_status tcg_set_warm_start(tcg_handle h, int on) {
  if (!h) return TCG_EINVAL;
  if (on && h->n_nl > 0) return fail(h, TCG_EINVAL, "warm start is not available with nonlinear patches");
  if (on < 0 || on > KW) return fail(h, TCG_EINVAL, "warm start subspace dimension must be in [0, " + std::to_string(KW) + "]");
  if (on != h->warm) h->warm_base = h->steps_done;  // a new subspace size restarts the history
  h->warm = on;
  return TCG_OK;
}

tcg_status tcg_set_error_tracking(tcg_handle h, int on) {
  if (!h) return TCG_EINVAL;
  if (on && h->n_nl > 0) return fail(h, TCG_EINVAL, "error tracking is not available with nonlinear patches");
  if (on && h->source != TCG_SOURCE_PAPER) return fail(h, TCG_EINVAL, "error tracking needs TCG_SOURCE_PAPER (the exact solution)");
  if (on && h->world > 1) return fail(h, TCG_EINVAL, "error tracking needs a single-process handle");
  if (h->setup_done && h->steps_done > 0) return fail(h, TCG_ESTATE, "enable error tracking before the first step");
  if (on && !h->err_acc) {
    cudaSetDevice(h->device);
    if (!h->stream) {
      CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->own_stream = true;
    }
    TRY(dzero(h, &h->err_acc, 8));
  }
  h->track = on != 0;
  return TCG_OK;
}

tcg_status tcg_get_errors(tcg_handle h, double* eps_B, double* eps_E, double* per_step, size_t nsteps) {
  if (!h) return TCG_EINVAL;
  if (!h->track || !h->err_acc) return fail(h, TCG_ESTATE, "error tracking is off");
  if (nsteps > (size_t)h->steps_done) return fail(h, TCG_EINVAL, "only " + std::to_string(h->steps_done) + " steps done");
  cudaSetDevice(h->device);
  double acc[8];
  CK(cudaMemcpyAsync(acc, h->err_acc, sizeof acc, cudaMemcpyDeviceToHost, h->stream));
  if (per_step && nsteps > 0)
    CK(cudaMemcpyAsync(per_step, h->err_step, 2 * nsteps * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->d2h_bytes += (int64_t)(sizeof acc + (per_step ? 2 * nsteps * sizeof(double) : 0));
  if (eps_B) *eps_B = h->steps_done ? acc[3] : 0.0;
  if (eps_E) *eps_E = h->steps_done ? acc[4] : 0.0;
  return TCG_OK;
}

tcg_status tcg_plan(tcg_handle h) {
  if (!h) return TCG_EINVAL;
  return do_plan(h);
}

tcg_status tcg_get_plan(tcg_handle h, int what, int64_t* out, size_t len) {
  if (!h) return TCG_EINVAL;
  if (!h->planned) return fail(h, TCG_ESTATE, "plan first");
  const Plan& p = h->plan;
  size_t need = 0;
  switch (what) {
    case TCG_PLAN_EDGE_CLASS: case TCG_PLAN_EDGE_REGION: case TCG_PLAN_TREE: case TCG_PLAN_PART: need = p.nedges; break;
    case TCG_PLAN_PATCH_COUNTS: need = 3 * (size_t)p.npatch; break;
    case TCG_PLAN_LAMBDA: need = 3 * (size_t)p.m; break;
    case TCG_PLAN_PRIMAL: need = p.nc; break;
    case TCG_PLAN_RANK_OF_PATCH: need = p.npatch; break;
    default: return fail(h, TCG_EINVAL, "unknown plan array");
  }
  if (!out || len < need) return fail(h, TCG_EINVAL, "buffer too short: need " + std::to_string(need));
  for (size_t i = 0; i < need; ++i) {
    int64_t v = 0;
    switch (what) {
      case TCG_PLAN_EDGE_CLASS: v = p.cls[i]; break;
      case TCG_PLAN_EDGE_REGION: v = p.region[i]; break;
      case TCG_PLAN_TREE: v = p.in_tree[i]; break;
      case TCG_PLAN_PART: v = p.part[i]; break;
      case TCG_PLAN_PATCH_COUNTS: {
        const PatchPlan& q = p.pp[i / 3];
        v = (i % 3 == 0) ? q.ni : (i % 3 == 1 ? q.nb : q.np);
        break;
      }
      case TCG_PLAN_LAMBDA: {
        size_t k = i / 3;
        v = (i % 3 == 0) ? p.lam_edge[k] : (i % 3 == 1 ? p.lam_plus[k] : p.lam_minus[k]);
        break;
      }
      case TCG_PLAN_PRIMAL: v = p.primal_edge[i]; break;
      case TCG_PLAN_RANK_OF_PATCH: v = p.rank_of_patch[i]; break;
    }
    out[i] = v;
  }
  return TCG_OK;
}

tcg_status tcg_setup(tcg_handle h) {
  if (!h) return TCG_EINVAL;
  if (h->setup_done) return fail(h, TCG_ESTATE, "setup already done");
  if (h->broken) return fail(h, TCG_ESTATE, "handle is in a failed state");
  if (h->n_nl > 0 && h->source == TCG_SOURCE_PAPER)
    return fail(h, TCG_EINVAL, "nonlinear patches need a source without Dirichlet lifting (kinds 0-2)");
  if (h->n_nl > 0 && h->track) return fail(h, TCG_EINVAL, "error tracking is not available with nonlinear patches");
  tcg_status s = do_setup(h);
  if (s != TCG_OK) h->broken = true;  // ENOTSPD included: only get_* / destroy afterwards
  return s;
}

tcg_status tcg_refactor(tcg_handle h) {
  if (!h) return TCG_EINVAL;
  if (!h->setup_done || h->broken) return fail(h, TCG_ESTATE, "setup first (or handle failed)");
  cudaSetDevice(h->device);
  tcg_status s = do_numeric(h);
  if (s != TCG_OK) h->broken = true;
  return s;
}

tcg_status tcg_step(tcg_handle h, int n) {
  if (!h) return TCG_EINVAL;
  if (!h->setup_done || h->broken) return fail(h, TCG_ESTATE, "setup first (or handle failed)");
  if (n < 0) return fail(h, TCG_EINVAL, "n >= 0");
  cudaSetDevice(h->device);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, h->stream);
  tcg_status s = TCG_OK;
  if (h->track) {
    // the paper's error norms (mms.cu): one step per launch (so every patch's
    // coefficients, insulators included, are recovered), then the error kernels
    const Plan& pl = h->plan;
    const size_t nall = (size_t)pl.npatch * pl.nloc;
    if (h->a_prev.empty()) {
      h->a_prev.assign(h->rd.size(), nullptr);
      for (auto& q : h->a_prev) {
        s = dalloc(h, &q, nall);
        if (s != TCG_OK) return s;
      }
      int nbk = 0;
      for (auto& R : h->rd) nbk += (int)R.plist.size() * pl.el[2];
      h->err_blocks = nbk;
      if ((s = dalloc(h, &h->err_part, 2 * (size_t)std::max(nbk, 1))) != TCG_OK) return s;
      if ((s = dalloc(h, &h->err_step, 2 * (size_t)h->n_steps)) != TCG_OK) return s;
    }
    const double dt = h->T / h->n_steps;
    for (int i = 0; i < n && s == TCG_OK; ++i) {
      for (size_t li = 0; li < h->rd.size(); ++li)
        CK(cudaMemcpyAsync(h->a_prev[li], h->rd[li].a_loc, nall * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
      s = do_steps(h, 1);
      if (s != TCG_OK) break;
      int64_t boff = 0;
      for (size_t li = 0; li < h->rd.size(); ++li) {
        RankDev& R = h->rd[li];
        if (R.plist.empty()) continue;
        k_mms_errors<<<dim3((unsigned)R.plist.size(), pl.el[2]), 256, 0, h->stream>>>(
            R.D, h->G, h->tb, h->steps_done * dt, dt, h->src_amp, R.d_plist, R.a_loc, h->a_prev[li], h->err_part + 2 * boff);
        ++h->nlaunch;
        boff += (int64_t)R.plist.size() * pl.el[2];
      }
      k_mms_accumulate<<<1, 32, 0, h->stream>>>(h->err_part, h->err_blocks, dt, h->err_acc, h->err_step,
                                                 (int)h->steps_done - 1);
      ++h->nlaunch;
      CKL();
    }
  } else if (h->n_nl > 0) {
    if (h->steps_done + n > h->n_steps) s = fail(h, TCG_EINVAL, "more steps than set_time allows (n_steps)");
    for (int i = 0; i < n && s == TCG_OK; ++i) s = do_newton_step(h);
  } else {
    s = do_steps(h, n);
  }
  if (s == TCG_OK) {
    cudaEventRecord(e1, h->stream);
    cudaEventSynchronize(e1);
    h->ms_steps += elapsed_ms(e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return s;
}

tcg_status tcg_get_coefficients(tcg_handle h, int layout, double* out, size_t len) {
  if (!h) return TCG_EINVAL;
  if (!h->setup_done) return fail(h, TCG_ESTATE, "setup first");
  const Plan& p = h->plan;
  cudaSetDevice(h->device);
  const int64_t nall = (int64_t)p.npatch * p.nloc;
  {
    StepArgs A = step_args(h);
    int* down = const_cast<int*>(h->D.owner);
    k_gather_aloc<<<592, 256, 0, h->stream>>>(h->a_all, A, down, p.nloc, nall);
    ++h->nlaunch;
    CKL();
  }
  if (layout == 0) {
    size_t need = (size_t)nall;
    if (!out || len < need) return fail(h, TCG_EINVAL, "buffer too short: need " + std::to_string(need));
    CK(cudaMemcpyAsync(out, h->a_all, need * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    h->d2h_bytes += (int64_t)(need * sizeof(double));
  } else if (layout == 1) {
    size_t need = (size_t)p.nedges;
    if (!out || len < need) return fail(h, TCG_EINVAL, "buffer too short: need " + std::to_string(need));
    k_gather_glued<<<592, 256, 0, h->stream>>>(h->glued, h->a_all, h->d_glued_src, p.nedges);
    ++h->nlaunch;
    CKL();
    CK(cudaMemcpyAsync(out, h->glued, need * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    h->d2h_bytes += (int64_t)(need * sizeof(double));
  } else {
    return fail(h, TCG_EINVAL, "layout must be 0 or 1");
  }
  CK(cudaStreamSynchronize(h->stream));
  return TCG_OK;
}

tcg_status tcg_get_history(tcg_handle h, int* iters, double* final_relres, size_t nsteps, double* relres_hist,
                           size_t hist_len) {
  if (!h) return TCG_EINVAL;
  if (nsteps > h->iters.size()) return fail(h, TCG_EINVAL, "only " + std::to_string(h->iters.size()) + " steps recorded");
  for (size_t i = 0; i < nsteps; ++i) {
    if (iters) iters[i] = h->iters[i];
    if (final_relres) final_relres[i] = h->final_rel[i];
  }
  if (relres_hist) {
    size_t need = 0;
    for (size_t i = 0; i < nsteps; ++i) need += h->hist_per_step[i];
    if (hist_len < need) return fail(h, TCG_EINVAL, "history buffer too short: need " + std::to_string(need));
    std::copy(h->hist_all.begin(), h->hist_all.begin() + need, relres_hist);
  }
  return TCG_OK;
}

tcg_status tcg_get_info(tcg_handle h, tcg_info* out) {
  if (!h || !out) return TCG_EINVAL;
  std::memset(out, 0, sizeof(tcg_info));
  out->rank = h->rank;
  out->world = std::max(h->world, h->vranks);
  if (!h->planned) return TCG_OK;
  const Plan& p = h->plan;
  out->n_patches = p.npatch;
  out->n_local = p.nloc;
  out->n_edges = p.nedges;
  out->n_verts = p.nverts;
  out->m = p.m;
  out->n_c = p.nc;
  out->n_gauge = p.n_gauge;
  out->n_dirichlet = p.n_dir;
  out->nr_min = out->nb_min = out->np_min = INT64_MAX;
  double bf = 0, bm = 0, bs = 0, fl = 0, bsi = 0;
  for (int s = 0; s < p.npatch; ++s) {
    const PatchPlan& q = p.pp[s];
    int64_t nr = q.ni + q.nb;
    out->nr_min = std::min(out->nr_min, nr);
    out->nr_max = std::max(out->nr_max, nr);
    out->nb_min = std::min<int64_t>(out->nb_min, q.nb);
    out->nb_max = std::max<int64_t>(out->nb_max, q.nb);
    out->np_min = std::min<int64_t>(out->np_min, q.np);
    out->np_max = std::max<int64_t>(out->np_max, q.np);
    out->n_primal_local_total += q.np;
    // algorithmic bytes: per F-apply [X_bb; Phi_b^T] read twice (P1, P5);
    // per preconditioner apply packed S_bb read once
    bf += 8.0 * q.nb * (q.nb + 1) + 16.0 * q.nb * q.np;
    bm += 4.0 * q.nb * (q.nb + 1);
    // sbbinv: the iteration's F-apply reads the packed S_bb^-1 once instead of X_bb twice
    bsi += 4.0 * q.nb * (q.nb + 1) + 16.0 * q.nb * q.np;
    if (h->sbbinv) fl += (double)q.nb * q.nb * q.nb / 3.0;
    const double nrp = (double)nr;
    // per step outside PCG: conductors read [X_rr; Phi^T] twice (R2 forward, E3 backward)
    if (h->dyn(s)) bs += 2.0 * 8.0 * (nrp * (nrp + 1) / 2 + nrp * q.np);
    // Cholesky + p-row TRSM + S^s update, then the inverse factors X_rr = L_rr^-1 (nr^3/3) and
    // X_pr = L_pr X_rr (np nr^2)
    fl += nrp * nrp * nrp / 3.0 + 2.0 * nrp * nrp * q.np + 2.0 * nrp * q.np * q.np;
    fl += nrp * nrp * nrp / 3.0 + nrp * nrp * q.np;
  }
  const double nc = (double)p.nc;
  if (h->sparse) {
    // sparse coarse: forward and backward each read every node's [L_VV^-1 (lower) ; L_BV L_VV^-1]
    for (const auto& n : h->nd.nd) {
      const double v = (double)n.V.size(), b = (double)n.B.size();
      bf += 2.0 * 8.0 * (v * (v + 1) / 2 + v * b);
    }
    bf += 40.0 * p.m;
    for (const auto& n : h->nd.nd) {
      const double v = (double)n.V.size(), b = (double)n.B.size();
      bsi += 2.0 * 8.0 * (v * (v + 1) / 2 + v * b);
    }
    bsi += 40.0 * p.m;
  } else {
    bf += 8.0 * nc * (nc + 1) + 40.0 * p.m;  // dense S_pp^-1 read once = two triangular passes
    bsi += 8.0 * nc * (nc + 1) + 40.0 * p.m;
  }
  bm += 40.0 * p.m;
  bs += bf + bm;  // R3/R4/E1/E2 (one F-apply worth) and the z0 preconditioner apply (R5)
  if (h->sparse) {
    for (const auto& n : h->nd.nd) {  // partial Cholesky of the V columns + in-place inverse
      const double v = (double)n.V.size(), b = (double)n.B.size();
      fl += v * v * v / 3.0 + v * v * b + v * b * b + v * v * v / 3.0 + v * v * b;
    }
  } else {
    fl += nc * nc * nc / 3.0;
  }
  out->coarse_sparse = h->sparse;
  out->coarse_nodes = h->sparse ? (int64_t)h->nd.nd.size() : 0;
  out->coarse_levels = h->sparse ? h->nd.H + 1 : 1;
  {
    double cb = 0.0;
    if (h->sparse)
      for (const auto& n : h->nd.nd) {
        const double v = (double)n.V.size(), b = (double)n.B.size();
        cb += 2.0 * 8.0 * (v * (v + 1) / 2 + v * b);
      }
    else
      cb = 8.0 * nc * nc;
    out->coarse_factor_bytes = cb;
  }
  out->bytes_fapply = h->sbbinv ? bsi : bf;  // (bytes_step_fixed keeps the X_bb form of R4 / E1)
  out->bytes_precond = bm;
  out->bytes_step_fixed = bs;
  out->flops_factor = fl;
  out->steps_done = h->steps_done;
  out->total_iters = h->total_iters;
  out->device_bytes = h->device_bytes;
  out->kernel_launches = h->nlaunch;
  out->ms_plan = h->ms_plan;
  out->ms_assembly = h->ms_assembly;
  out->ms_factor = h->ms_factor;
  out->ms_coarse = h->ms_coarse;
  out->ms_steps = h->ms_steps;
  out->prof_ms = h->prof_ms;
  out->prof_launches = h->prof_count;
  out->prof_bytes_per_launch = 0.0;  // per-launch bytes of the stepper depend on iterations (bench.py)
  out->h2d_bytes = h->h2d_bytes;
  out->d2h_bytes = h->d2h_bytes;
  out->n_nonlinear = h->n_nl;
  out->newton_iters = 0;
  for (int v : h->newton_its) out->newton_iters += v;
  out->linear_solves = (int64_t)h->solve_its.size();
  out->hist_len = 0;
  for (int64_t v : h->hist_per_step) out->hist_len += v;
  out->ms_newton_numeric = h->ms_newton_numeric;
  return TCG_OK;
}

// n applications q = F p inside the persistent stepper (mode 1), p = pk[0], q -> r[1]; *ms =
// device time (CUDA events on the library stream). Single-process handles.
static tcg_status run_fapply(tcg_ctx* h, int n, double* ms) {
  if (!h->setup_done || h->broken) return fail(h, TCG_ESTATE, "setup first");
  if (h->world > 1) return fail(h, TCG_EINVAL, "F-apply hooks need a single-process handle");
  CK(cudaSetDevice(h->device));
  for (auto& R : h->rd) CK(cudaMemsetAsync(R.st, 0, sizeof(PcgState), h->stream));
  if (h->sparse)
    for (auto* df : h->ndd.dflow) CK(cudaMemsetAsync(df, 0, 3 * sizeof(unsigned int) * std::max(h->ndd.nn, 1), h->stream));
  if (h->warm)
    for (auto& R : h->rd)
      if (!R.Wr) {  // warm-start rings: k solutions and k F-products at the lambda level
        const size_t m = (size_t)std::max<int64_t>(1, h->plan.m);
        TRY(dzero(h, &R.Wr, (size_t)KW * m));
        TRY(dzero(h, &R.FWr, (size_t)KW * m));
        TRY(dzero(h, &R.dsave, m));
        TRY(dzero(h, &R.wpart, (size_t)2 * h->nbr * KW_NV));
      }
  StepArgs A = step_args(h);
  A.nsteps = n;
  A.mode = 1;
  DevPlan D = h->D;
  void* args[] = {(void*)&D, (void*)&A};
  const int grid = h->nbr * (int)h->rd.size();
  const void* fn = (h->nranks > 1) ? (h->cache_bpos ? (const void*)k_steps<true, true> : (const void*)k_steps<true, false>)
                                     : (h->cache_bpos ? (const void*)k_steps<false, true> : (const void*)k_steps<false, false>);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, h->stream);
  CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(NTHR), args, h->smem_steps, h->stream));
  ++h->nlaunch;
  cudaEventRecord(e1, h->stream);
  CK(cudaMemcpyAsync(h->h_st, h->rd[0].st, sizeof(PcgState), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->bar_round = h->h_st->counter[3];
  if (ms) *ms = elapsed_ms(e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return TCG_OK;
}

tcg_status tcg_bench_fapply(tcg_handle h, int n, double* ms) {
  if (!h || !ms || n < 1) return h ? fail(h, TCG_EINVAL, "n >= 1 and ms required") : TCG_EINVAL;
  return run_fapply(h, n, ms);
}

tcg_status tcg_fapply(tcg_handle h, const double* lam, double* q, size_t m) {
  if (!h || !lam || !q) return TCG_EINVAL;
  if (!h->setup_done || h->broken) return fail(h, TCG_ESTATE, "setup first");
  if (m != (size_t)h->plan.m) return fail(h, TCG_EINVAL, "need m = " + std::to_string(h->plan.m));
  if (h->world > 1) return fail(h, TCG_EINVAL, "F-apply hooks need a single-process handle");
  CK(cudaSetDevice(h->device));
  // p = lam in every local rank's copy (each reads its own chunk); q gathered from the owners
  for (auto& R : h->rd) CK(cudaMemcpyAsync(R.pk0, lam, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream));
  h->h2d_bytes += (int64_t)(sizeof(double) * m);
  TRY(run_fapply(h, 1, nullptr));
  const int64_t per = (int64_t)h->lam_chunk * h->nbr;  // lambda entries per rank
  for (auto& R : h->rd) {
    const int64_t k0 = std::min<int64_t>((int64_t)m, per * R.r), k1 = std::min<int64_t>((int64_t)m, k0 + per);
    if (k1 > k0) CK(cudaMemcpy(q + k0, R.r1 + k0, sizeof(double) * (k1 - k0), cudaMemcpyDeviceToHost));
  }
  h->d2h_bytes += (int64_t)(sizeof(double) * m);
  return TCG_OK;
}

tcg_status tcg_set_profile(tcg_handle h, int kernel_id) {
  if (!h) return TCG_EINVAL;
  if (kernel_id != 0 && kernel_id != 7) return fail(h, TCG_EINVAL, "kernel id 0 (off) or 7 (k_steps)");
  h->prof_id = kernel_id;
  h->prof_ms = 0;
  h->prof_count = 0;
  h->prof_used = 0;
  return TCG_OK;
}

// Debug readback (not part of the public header; single-rank handles): what 0 = assembled
// augmented matrix of patch `idx` (TCG_DEBUG_KEEP=1), 1 = its current factor/inverse,
// 2 = aug map of patch, 3 = assembled coarse matrix, 4 = Z (rhs-stage vector) of patch,
// 5 = rho weights interleaved, 6 = S_bb tiles of patch, 7 = phase timestamps.
tcg_status tcg_debug_array(tcg_handle h, int what, int idx, double* out, size_t len) {
  if (!h || !h->setup_done) return TCG_ESTATE;
  cudaSetDevice(h->device);
  RankDev& R = h->rd[0];
  const double* src = nullptr;
  size_t n = 0;
  std::vector<double> tmp;
  if (what == 0 || what == 1) {
    src = (what == 0 ? h->dbgA : R.A);
    if (!src) return fail(h, TCG_ESTATE, "TCG_DEBUG_KEEP not set");
    src += h->h_a_off[idx];
    n = tri_tiles(h->h_T[idx]) * TSZ;
  } else if (what == 2) {
    for (int v : h->plan.pp[idx].aug) tmp.push_back((double)v);
  } else if (what == 3) {
    src = h->dbgC;
    if (!src) return fail(h, TCG_ESTATE, "TCG_DEBUG_KEEP not set");
    n = tri_tiles(h->Tc) * TSZ;
  } else if (what == 4) {
    src = R.Z + h->h_vec_off[idx];
    n = (size_t)h->h_T[idx] * TS;
  } else if (what == 5) {
    std::vector<double> wp(h->D.m), wm(h->D.m);
    CK(cudaMemcpy(wp.data(), h->D.wplus, sizeof(double) * h->D.m, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(wm.data(), h->D.wminus, sizeof(double) * h->D.m, cudaMemcpyDeviceToHost));
    for (int64_t k = 0; k < h->D.m; ++k) {
      tmp.push_back(wp[k]);
      tmp.push_back(wm[k]);
    }
  } else if (what == 6) {
    src = R.Sbb + h->h_sbb_off[idx];
    n = tri_tiles(h->plan.pp[idx].Tb) * TSZ;
  } else if (what == 8) {  // sparse coarse solution (by primal group) and forward vectors
    if (!h->sparse) return fail(h, TCG_ESTATE, "dense coarse");
    std::vector<double> a((size_t)h->plan.nc);
    CK(cudaMemcpy(a.data(), h->ndd.Pcs[0], sizeof(double) * a.size(), cudaMemcpyDeviceToHost));
    tmp = a;
  } else if (what == 9) {  // sparse coarse tree: per node (height, n_V, n_B, T_V, T_B)
    for (const auto& n : h->nd.nd) {
      tmp.push_back(n.height);
      tmp.push_back((double)n.V.size());
      tmp.push_back((double)n.B.size());
      tmp.push_back(n.TV);
      tmp.push_back(n.TB);
    }
    if (tmp.empty()) tmp.push_back(0);
  } else if (what == 10 || what == 11) {
    // 10: per-item durations (ns) of phase idx, 11: the items of phase idx as rows
    // (block, s, I, part & 15, gather code, Tb, Tp, nb, np) -- phase-timing builds only
    const int ph = idx;
    if (ph < 0 || ph >= NCACHE) return TCG_EINVAL;
    const auto& items = h->h_items[ph];
    if (what == 10) {
      if (!h->itime) return fail(h, TCG_ESTATE, "TCG_PHASE_TIMING not set");
      std::vector<double> t((size_t)h->itime_stride);
      CK(cudaMemcpy(t.data(), h->itime + (size_t)ph * h->itime_stride, t.size() * sizeof(double), cudaMemcpyDeviceToHost));
      tmp.assign(t.begin(), t.begin() + items.size());
    } else {
      const auto& bo = h->h_boff[ph];
      for (size_t b = 0; b + 1 < bo.size(); ++b)
        for (int j = bo[b]; j < bo[b + 1]; ++j) {
          const ItemDesc& d = items[j];
          for (double v : {(double)b, (double)d.s, (double)d.I, (double)(d.part & 15), (double)((d.part >> 4) & 3),
                           (double)d.Tb, (double)d.Tp, (double)d.nb, (double)d.np})
            tmp.push_back(v);
        }
    }
    if (tmp.empty()) tmp.push_back(0);
  } else if (what == 7) {
    if (!h->tstamp) return fail(h, TCG_ESTATE, "TCG_PHASE_TIMING not set");
    std::vector<unsigned long long> ts(8 * 64 + 16 + 8 * 4096 + 8 * 64);
    CK(cudaMemcpy(ts.data(), h->tstamp, ts.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (auto v : ts) tmp.push_back((double)v);
  } else {
    return TCG_EINVAL;
  }
  if (!tmp.empty()) {
    if (len < tmp.size()) return fail(h, TCG_EINVAL, "need " + std::to_string(tmp.size()));
    std::copy(tmp.begin(), tmp.end(), out);
    return TCG_OK;
  }
  if (len < n) return fail(h, TCG_EINVAL, "need " + std::to_string(n));
  CK(cudaMemcpy(out, src, n * sizeof(double), cudaMemcpyDeviceToHost));
  return TCG_OK;
}

const char* tcg_last_error(tcg_handle h) { return h ? h->err.c_str() : "null handle"; }

void tcg_destroy(tcg_handle h) { delete h; }

}  // extern "C"
