// potrf_bench.cu — standalone timing of the tile POTRF+inverse kernel (k_potrf) on random SPD
// tiles: events around launches with 1 and 64 matrices, and a residual check |L X - I|.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_23446_b200/csrc -o tools/potrf_bench tools/potrf_bench.cu
#include <cstdio>
#include <vector>
#include <cmath>
#include <random>
#define POTRF_PROBE_ON
#include "chol.cu"
using namespace tcg;
int main() {
  const int NM = 64;
  std::vector<double> h((size_t)NM * TSZ);
  std::mt19937 g(1);
  std::normal_distribution<double> nd;
  for (int m = 0; m < NM; ++m) {
    std::vector<double> B(TSZ);
    for (auto& v : B) v = nd(g);
    for (int i = 0; i < TS; ++i)
      for (int j = 0; j < TS; ++j) {
        double s = (i == j) ? TS : 0.0;
        for (int q = 0; q < TS; ++q) s += B[i * TS + q] * B[j * TS + q] / TS;
        h[(size_t)m * TSZ + i * TS + j] = s;
      }
  }
  double *dA, *dX;
  cudaMalloc(&dA, h.size() * 8);
  cudaMalloc(&dX, h.size() * 8);
  std::vector<CholDesc> desc(NM);
  for (int m = 0; m < NM; ++m) desc[m] = CholDesc{(int64_t)m * TSZ, (int64_t)m * TSZ, -1, 1, 1, -1, 0};
  CholDesc* dd;
  cudaMalloc(&dd, NM * sizeof(CholDesc));
  cudaMemcpy(dd, desc.data(), NM * sizeof(CholDesc), cudaMemcpyHostToDevice);
  DevError* de;
  cudaMalloc(&de, sizeof(DevError));
  cudaMemset(de, 0, sizeof(DevError));
  cudaFuncSetAttribute(k_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TS * PS * 8);
  for (int nm : {1, 64}) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemcpy(dA, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_potrf<<<nm, 256, 2 * TS * PS * 8>>>(dd, 0, dA, dX, de, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    printf("k_potrf matrices %2d: %.2f us (%s)\n", nm, 1000 * best, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> L(h.size()), X(h.size());
  cudaMemcpy(L.data(), dA, h.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(X.data(), dX, h.size() * 8, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int m = 0; m < NM; ++m)
    for (int i = 0; i < TS; ++i)
      for (int j = 0; j < TS; ++j) {
        double s = 0, r = 0;
        for (int q = 0; q < TS; ++q) {
          s += L[(size_t)m * TSZ + i * TS + q] * X[(size_t)m * TSZ + q * TS + j];
          r += L[(size_t)m * TSZ + i * TS + q] * L[(size_t)m * TSZ + j * TS + q];
        }
        e1 = std::max(e1, std::fabs(s - (i == j)));
        e2 = std::max(e2, std::fabs(r - h[(size_t)m * TSZ + i * TS + j]));
      }
  {
    long long hp[64];
    cudaMemcpyFromSymbol(hp, g_probe, sizeof(hp));
    printf("panel-0 step probes (cycles since step 0 start):\n");
    for (int jj = 0; jj < 16; ++jj) printf("  jj %2d: %6lld %6lld %6lld %6lld\n", jj, hp[jj*4]-hp[0], hp[jj*4+1]-hp[0], hp[jj*4+2]-hp[0], hp[jj*4+3]-hp[0]);
  }
  printf("max |L X - I| = %.3e   max |L L^T - W| = %.3e\n", e1, e2);
  return 0;
}
