// fp64_latency.cu — microbenchmarks behind the tile-POTRF design: dependent DFMA / DMUL /
// rsqrt / sqrt / division chains (1 thread) and a 256-thread loop of 128 __syncthreads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kchain(double* out, long long* cyc, int n, int which) {
  double x = out[0], y = out[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (which == 0) x = fma(x, y, 0.5);
    else if (which == 1) x = x * y;
    else if (which == 2) x = rsqrt(x + 1.5);
    else if (which == 3) x = sqrt(x + 1.5);
    else if (which == 4) x = 1.0 / (x + 1.5);
    else x = __fmul_rn(x, 0.999f) + 1.0f;  // fp32 reference (via double converts)
  }
  long long t1 = clock64();
  out[2] = x;
  cyc[which] = (t1 - t0) / n;
}
__global__ void kbar(long long* cyc, int n) {
  __shared__ double s[256];
  long long t0 = clock64();
  double v = threadIdx.x;
  for (int i = 0; i < n; ++i) {
    s[threadIdx.x] = v;
    __syncthreads();
    v += s[(threadIdx.x + 1) & 255];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / n; s[0] = v; }
  if (v == 12345.0) cyc[1] = 1;
}
int main() {
  double* d; long long* c;
  cudaMalloc(&d, 64); cudaMalloc(&c, 64 * 8);
  double h[3] = {0.7, 0.9, 0}; cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
  const char* nm[] = {"DFMA", "DMUL", "rsqrt(double)", "sqrt(double)", "1/x double", "fp32 fmul+add"};
  for (int w = 0; w < 6; ++w) {
    kchain<<<1, 1>>>(d, c, 4096, w); cudaDeviceSynchronize();
    long long r[6]; cudaMemcpy(r, c, 48, cudaMemcpyDeviceToHost);
    printf("%-16s %lld cycles per dependent op\n", nm[w], r[w]);
  }
  kbar<<<64, 256>>>(c, 1024); cudaDeviceSynchronize();
  long long r; cudaMemcpy(&r, c, 8, cudaMemcpyDeviceToHost);
  printf("2x __syncthreads + smem round trip (256 thr): %lld cycles per iteration\n", r);
  return 0;
}
