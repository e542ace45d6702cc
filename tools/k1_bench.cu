// K1 variants on the cfg2 shape (n = 1000, k = 25, P = 65536), S = 5 chunks, CUDA events.
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_1304_4333_b200/csrc/loglik.cuh"
using namespace sps;
template <typename K>
float run(K kern, LLArgs a, dim3 grid, size_t smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int i = 0; i < 3; ++i) kern<<<grid, 128, smem>>>(a);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) kern<<<grid, 128, smem>>>(a);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 20;
}
int main() {
  const int n = 1000, k = 25, KP = 28; const long P = 65536;
  std::mt19937_64 g(1); std::normal_distribution<double> nd(0, 1);
  std::vector<double> X(n * KP, 0.0), th(P * k);
  for (int t = 0; t < n; ++t) for (int i = 0; i < k; ++i) X[t * KP + i] = (i == 0 ? 1.0 : nd(g)) * (t % 3 ? 1 : -1);
  for (auto& v : th) v = 0.3 * nd(g);
  double *dX, *dth, *dpart; cudaMalloc(&dX, X.size() * 8); cudaMalloc(&dth, th.size() * 8); cudaMalloc(&dpart, 64 * P * 8);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dth, th.data(), th.size() * 8, cudaMemcpyHostToDevice);
  for (int S : {5, 6, 8, 10}) {
    const int chunk = (n + S - 1) / S;
    LLArgs a{dX, nullptr, dth, dpart, k, P, 0, n, chunk}; a.k = k; a.stop = nullptr;
    dim3 grid(P / 128, S);
    size_t smem = 256 * 8 + (size_t)(chunk + 16) * KP * 8;
    float t1 = run(k_loglik_bin_mma<6, 1, 4, 1, 64, 1, 1>, a, grid, smem);
    float t2 = run(k_loglik_bin_mma<6, 1, 4, 1, 64, 2, 1>, a, grid, smem);
    float t3 = run(k_loglik_bin_mma<6, 1, 4, 1, 64, 1, 4>, a, grid, smem);
    float t4 = run(k_loglik_bin_mma<6, 1, 4, 1, 64, 2, 4>, a, grid, smem);
    float t5 = run(k_loglik_bin_mma<6, 1, 2, 1, 64, 2, 6>, a, dim3(P / 64, S), smem);
    dim3 g2(P / 256, S);
    float t6 = run(k_loglik_bin<25, 2>, a, g2, 64 * 8 + (size_t)chunk * KP * 8 + 16);
    printf("S=%d  base %.1f us  ks2 %.1f  minb4 %.1f  ks2+minb4 %.1f  ntw2+ks2+minb6 %.1f  dfma %.1f\n",
           S, 1000 * t1, 1000 * t2, 1000 * t3, 1000 * t4, 1000 * t5, 1000 * t6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
