// barrier_bench.cu — microbenchmark of grid-barrier variants for the persistent stepper
// (296 co-resident blocks x 256 threads on B200). Prints ns per barrier for each variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ double block_sum(double v, double* red) {
  double w = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  double r = 0;
  for (int i = 0; i < 8; ++i) r += red[i];
  __syncthreads();
  return r;
}

// variant: 0 red.release + acquire poll; 1 red.release + relaxed poll + fence;
// 2 = 0 with nanosleep backoff; 3 = two-level (groups of 16 blocks, group leaders)
__global__ void kbar(unsigned* cnt, double* partials, int nb, int iters, int variant, int reduce, double* out) {
  __shared__ double red[8];
  __shared__ double s_tot;
  unsigned round = 0;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    ++round;
    if (variant <= 2) {
      if (threadIdx.x == 0) {
        if (reduce) partials[blockIdx.x] = (double)(blockIdx.x + it);
        red_rel(cnt, 1u);
        const unsigned target = round * (unsigned)nb;
        if (variant == 0)
          while ((int)(ld_acq(cnt) - target) < 0) {}
        else if (variant == 1) {
          while ((int)(ld_rlx(cnt) - target) < 0) {}
          fence_acqrel();
        } else {
          while ((int)(ld_acq(cnt) - target) < 0) __nanosleep(32);
        }
      }
      __syncthreads();
    } else if (variant == 6) {
      // slot polling: every block writes (value | sentinel-free) into its slot of buffer
      // round % 3; every thread polls its share of the slots until none holds the sentinel;
      // the slot of round - 2 is reset after the round completes (triple buffering)
      const unsigned long long SENT = 0x7ff4deadbeef0000ull;
      unsigned long long* slots = reinterpret_cast<unsigned long long*>(partials + 4096);
      const int buf = round % 3;
      if (threadIdx.x == 0) {
        const double v = (double)(blockIdx.x + it);
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(slots + buf * 4096 + blockIdx.x), "l"(__double_as_longlong(v)) : "memory");
      }
      double t = 0.0;
      for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        unsigned long long v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slots + buf * 4096 + j) : "memory");
        } while (v == SENT);
        t += __longlong_as_double(v);
      }
      const double tot = block_sum(t, red);
      if (reduce) acc += tot;
      if (threadIdx.x == 0) slots[((round + 2) % 3) * 4096 + blockIdx.x] = SENT;  // previous round's slot (read again in round + 2)
      continue;
    } else if (variant == 4 || variant == 5) {
      // master: block 0 watches 8 arrival counters, then writes every block's release slot
      // (triple-buffered, sentinel = NaN payload) carrying the reduced value
      const unsigned long long SENT = 0x7ff4deadbeef0000ull;
      unsigned long long* slots = reinterpret_cast<unsigned long long*>(partials + 4096);
      const int buf = round % 3, nxt = (round + 1) % 3;
      if (threadIdx.x == 0) {
        if (reduce) partials[blockIdx.x] = (double)(blockIdx.x + it);
        red_rel(cnt + 32 * (blockIdx.x & 7), 1u);
      }
      if (blockIdx.x == 0) {
        if (threadIdx.x < 8) {
          const unsigned n_i = (unsigned)((nb - (int)threadIdx.x + 7) / 8);
          const unsigned target = round * n_i;
          while ((int)(ld_acq(cnt + 32 * threadIdx.x) - target) < 0) {
            if (variant == 5) __nanosleep(20);
          }
        }
        __syncthreads();
        double tot = 0.0;
        if (reduce) {
          double t = 0;
          for (int j = threadIdx.x; j < nb; j += blockDim.x) t += __ldcg(partials + j);
          tot = block_sum(t, red);
        }
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
          slots[nxt * 4096 + b] = SENT;
          const unsigned long long v = __double_as_longlong(tot);
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(slots + buf * 4096 + b), "l"(v) : "memory");
        }
        acc += tot;
      } else {
        if (threadIdx.x == 0) {
          unsigned long long v;
          do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slots + buf * 4096 + blockIdx.x) : "memory");
          } while (v == SENT);
          s_tot = __longlong_as_double(v);
        }
        __syncthreads();
        acc += s_tot;
      }
      continue;
    } else {
      // two-level: group g = blockIdx/16 counter cnt[1+g]; last of a group arrives on cnt[0]
      const int g = blockIdx.x / 16, ng = (nb + 15) / 16, gs = min(16, nb - g * 16);
      if (threadIdx.x == 0) {
        if (reduce) partials[blockIdx.x] = (double)(blockIdx.x + it);
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt + 32 * (1 + g)) : "memory");
        if (old + 1 == round * (unsigned)gs) red_rel(cnt, 1u);
        const unsigned target = round * (unsigned)ng;
        while ((int)(ld_acq(cnt) - target) < 0) {}
      }
      __syncthreads();
    }
    if (reduce) {
      double t = 0;
      for (int j = threadIdx.x; j < nb; j += blockDim.x) t += __ldcg(partials + j);
      acc += block_sum(t, red);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

__global__ void kinit(unsigned long long* slots) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * 4096; i += gridDim.x * blockDim.x) slots[i] = 0x7ff4deadbeef0000ull;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* cnt;
  double *partials, *out;
  cudaMalloc(&cnt, 4096);
  cudaMalloc(&partials, 8 * 4096 * 4);
  cudaMalloc(&out, 8);
  const char* names[] = {"red.release + ld.acquire poll", "red.release + relaxed poll + fence", "acquire poll + nanosleep",
                         "two-level (16-block groups)", "master + per-block slots", "master + slots + nanosleep", "slot polling (triple buffer)"};
  for (int per = 1; per <= 2; ++per) {
    const int nb = sms * per;
    for (int reduce = 0; reduce < 2; ++reduce)
      for (int v = 0; v < 7; ++v) {
        int iters = 2000;
        void* args[] = {&cnt, &partials, (void*)&nb, &iters, &v, &reduce, &out};
        cudaMemset(cnt, 0, 4096);
        cudaMemset(partials + 4096, 0xff, 8 * 3 * 4096);  // not the sentinel: overwritten below
        kinit<<<48, 256>>>(reinterpret_cast<unsigned long long*>(partials + 4096));
        cudaLaunchCooperativeKernel((void*)kbar, nb, 256, args, 0, 0);  // warm
        cudaDeviceSynchronize();
        cudaMemset(cnt, 0, 4096);
        kinit<<<48, 256>>>(reinterpret_cast<unsigned long long*>(partials + 4096));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)kbar, nb, 256, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("blocks %3d reduce %d  %-40s %7.1f ns/barrier  (%s)\n", nb, reduce, names[v], 1e6 * ms / iters,
               cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
