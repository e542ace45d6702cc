// Dependent-chain latencies (cycles per op) of FP64 and shuffle operations, one warp.
#include <cstdio>
__global__ void k(double x0, int n, long long* out, double* sink) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = fma(x, 0.999999999, 1e-12); t1 = clock64(); out[0] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = x + 1e-12; t1 = clock64(); out[1] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = sqrt(x) + 0.5; t1 = clock64(); out[2] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = rsqrt(x) + 0.5; t1 = clock64(); out[3] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = 1.0 / x + 0.5; t1 = clock64(); out[4] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-12; t1 = clock64(); out[5] = (t1 - t0) / n;
  float f = (float)x;
  t0 = clock64(); for (int i = 0; i < n; ++i) f = fmaf(f, 0.9999f, 1e-6f); t1 = clock64(); out[6] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __drcp_rn(x) + 0.5; t1 = clock64(); out[7] = (t1 - t0) / n;
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __dsqrt_rn(x) + 0.5; t1 = clock64(); out[8] = (t1 - t0) / n;
  sink[threadIdx.x] = x + f;
}
int main() {
  long long* o; double* s; cudaMallocManaged(&o, 16 * 8); cudaMalloc(&s, 1024);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(1.7, 1000, o, s);
  cudaDeviceSynchronize();
  const char* nm[] = {"dfma", "dadd", "sqrt+add", "rsqrt+add", "div+add", "shfl64+add", "ffma32", "drcp_rn+add", "dsqrt_rn+add"};
  for (int i = 0; i < 9; ++i) printf("%-14s %lld cycles\n", nm[i], o[i]);
}
