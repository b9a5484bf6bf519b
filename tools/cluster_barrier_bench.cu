// cluster_barrier_bench.cu — grid barrier over a persistent grid built from thread-block
// clusters: cluster-level hardware barrier, one global arrival + poll per cluster, cluster
// barrier to release (optionally with a fixed-order sum of one value per block).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_barrier_bench tools/cluster_barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__global__ void kbar(unsigned* cnt, double* part, int iters, int reduce, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double s_val[32];  // per cluster-rank slots (leader block gathers via DSMEM)
  __shared__ double s_tot;
  const unsigned crank = cl.block_rank(), csize = cl.num_blocks();
  const unsigned ncl = gridDim.x / csize, cid = blockIdx.x / csize;
  unsigned round = 0;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    ++round;
    const double v = (double)(blockIdx.x + it);
    if (reduce && threadIdx.x == 0) {
      double* leader_slots = cl.map_shared_rank(s_val, 0);
      leader_slots[crank] = v;  // DSMEM store into the leader block
    }
    __syncthreads();
    cl_arrive();
    cl_wait();
    if (crank == 0) {
      if (threadIdx.x == 0) {
        if (reduce) {
          double t = 0.0;
          for (unsigned r = 0; r < csize; ++r) t += s_val[r];
          part[cid] = t;
        }
        red_rel(cnt, 1u);
        const unsigned target = round * ncl;
        while ((int)(ld_acq(cnt) - target) < 0) {}
        if (reduce) {
          double t = 0.0;
          for (unsigned c = 0; c < ncl; ++c) t += __ldcg(part + c);
          for (unsigned r = 0; r < csize; ++r) *cl.map_shared_rank(&s_tot, r) = t;
        }
      }
      __syncthreads();
    }
    cl_arrive();
    cl_wait();
    if (reduce) acc += s_tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

int main() {
  unsigned* cnt;
  double *part, *out;
  cudaMalloc(&cnt, 4096);
  cudaMalloc(&part, 8 * 4096);
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(kbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int csz : {2, 4, 8, 16}) {
    for (int per = 1; per <= 2; ++per) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.blockDim = dim3(256);
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.gridDim = dim3(csz);
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, (void*)kbar, &cfg);
      // clusters resident with `per` blocks per SM at most: limit by SM count
      int maxcl = (148 * per) / csz;
      ncl = std::min(ncl, maxcl);
      cfg.gridDim = dim3(ncl * csz);
      for (int reduce = 0; reduce < 2; ++reduce) {
        int iters = 2000;
        cudaMemset(cnt, 0, 4096);
        cudaLaunchKernelEx(&cfg, kbar, cnt, part, 50, reduce, out);
        cudaDeviceSynchronize();
        cudaMemset(cnt, 0, 4096);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, kbar, cnt, part, iters, reduce, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cluster %2d  blocks %3d (%d clusters)  reduce %d  %7.1f ns/barrier  (%s)\n", csz, ncl * csz, ncl, reduce,
               1e6 * ms / iters, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
