// Microbenchmark: FP64 tensor-pipe (DMMA, mma.sync.m8n8k4.f64) and FP64 FMA peak on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double acc[16][2];
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x;
  const double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int bps : {1, 2, 4, 8}) {
      const int blocks = sms * bps, threads = 256, iters = 4096;
      dmma_loop<<<blocks, threads>>>(out, 16);
      cudaEventRecord(e0);
      dmma_loop<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 16.0 * iters * (blocks * threads / 32.0);
      printf("DMMA m8n8k4  blocks/SM %d: %.2f TFLOP/s\n", bps, flops / (ms * 1e-3) / 1e12);
      dfma_loop<<<blocks, threads>>>(out, 16);
      cudaEventRecord(e0);
      dfma_loop<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16.0 * iters * blocks * threads;
      printf("DFMA         blocks/SM %d: %.2f TFLOP/s\n", bps, flops / (ms * 1e-3) / 1e12);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
