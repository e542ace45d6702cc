// FP64 pipe microbenchmarks for B200 (sm_100a).
//
// Measures the denominators DESIGN.md needs for the loglik roofline, which
// MEASURED_PEAKS.json does not carry: DFMA throughput, DMMA (mma.sync .f64)
// throughput for every legal f64 shape, whether DMMA and DFMA overlap when
// issued by the same or by different warps, and the cost of CUDA's exp/log1p
// in DFMA-equivalents.  Prints one JSON object on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ unsigned long long g_clk[2];
__device__ unsigned long long g_ns[2];

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

__device__ __forceinline__ void stamp_begin() {
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = clock64(); g_ns[0] = gtimer(); }
}
__device__ __forceinline__ void stamp_end() {
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[1] = clock64(); g_ns[1] = gtimer(); }
}

// ---------------------------------------------------------------- DFMA
__global__ void k_dfma(double* out, int iters, double a, double b) {
  stamp_begin();
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = fma(r[j], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += r[j];
  stamp_end();
  if (s == 12345.678) out[threadIdx.x] = s;
}

// ---------------------------------------------------------------- DMMA
__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double* c, const double* a, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma1688(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>  // 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
__global__ void k_dmma(double* out, int iters) {
  stamp_begin();
  double a[8], b[4], c[4][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1e-3 * (threadIdx.x + j);
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 1e-3 * (threadIdx.x - j);
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[q][j] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (SHAPE == 0) mma884(c[q][0], c[q][1], a[q], b[q]);
        if (SHAPE == 1) mma1684(c[q], a + 2 * (q & 1), b[q]);
        if (SHAPE == 2) mma1688(c[q], a + 4 * (q & 1), b);
        if (SHAPE == 3) mma16816(c[q], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[q][j];
  stamp_end();
  if (s == 12345.678) out[threadIdx.x] = s;
}

// Same warp issues NM m8n8k4 DMMA and NF DFMA (x8 chains) per iteration.
template <int NM, int NF>
__global__ void k_mixed_same(double* out, int iters, double fa, double fb) {
  stamp_begin();
  double a[4], b[4], c[4][2], r[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) { a[j] = 1e-3 * (threadIdx.x + j); b[j] = 1e-3 * j; c[j][0] = c[j][1] = 0; }
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < NM; ++u) mma884(c[u & 3][0], c[u & 3][1], a[u & 3], b[u & 3]);
#pragma unroll
    for (int u = 0; u < NF; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = fma(r[j], fa, fb);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < 8; ++j) s += r[j];
  stamp_end();
  if (s == 12345.678) out[threadIdx.x] = s;
}

// Even warps issue DMMA, odd warps DFMA.
template <int NM, int NF>
__global__ void k_mixed_split(double* out, int iters, double fa, double fb) {
  stamp_begin();
  const int w = threadIdx.x >> 5;
  double s = 0;
  if ((w & 1) == 0) {
    double a[4], b[4], c[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) { a[j] = 1e-3 * (threadIdx.x + j); b[j] = 1e-3 * j; c[j][0] = c[j][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < NM; ++u) mma884(c[u & 3][0], c[u & 3][1], a[u & 3], b[u & 3]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < NF; ++u) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = fma(r[j], fa, fb);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += r[j];
  }
  stamp_end();
  if (s == 12345.678) out[threadIdx.x] = s;
}

// ---------------------------------------------------------------- transcendental cost
template <int OP>  // 0 exp, 1 log1p, 2 log, 3 exp+log1p (softplus tail)
__global__ void k_transc(double* out, int iters) {
  stamp_begin();
  double x[4], s[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { x[j] = -1e-4 * (threadIdx.x + 37 * j) - 0.25; s[j] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double v;
      if (OP == 0) v = exp(x[j]);
      if (OP == 1) v = log1p(-x[j]);
      if (OP == 2) v = log(-x[j]);
      if (OP == 3) v = log1p(exp(x[j]));
      s[j] += v;
      x[j] -= 1e-7;
    }
  }
  stamp_end();
  if (s[0] + s[1] + s[2] + s[3] == 12345.678) out[threadIdx.x] = s[0];
}

struct Res { double ms, mhz; };

template <typename F>
static int timeit(F launch, Res* r) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f; double mhz = 0;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long clk[2], ns[2];
    CK(cudaMemcpyFromSymbol(clk, g_clk, sizeof(clk)));
    CK(cudaMemcpyFromSymbol(ns, g_ns, sizeof(ns)));
    if (ms < best) { best = ms; mhz = (double)(clk[1] - clk[0]) / (double)(ns[1] - ns[0]) * 1e3; }
  }
  r->ms = best; r->mhz = mhz;
  return 0;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int blocks = sms * 8, threads = 256;
  const double nthreads = (double)blocks * threads;
  printf("{\"gpu\": \"%s\", \"sms\": %d", prop.name, sms);

  Res r;
  {  // DFMA
    const int iters = 4096;
    if (timeit([&] { k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9); }, &r)) return 1;
    double fmas = nthreads * iters * 16 * 8;
    printf(", \"dfma\": {\"tflops\": %.3f, \"fma_per_clk_per_sm\": %.2f, \"mhz\": %.0f, \"ms\": %.3f}",
           2 * fmas / r.ms / 1e9, fmas / (r.ms * 1e-3) / (r.mhz * 1e6) / sms, r.mhz, r.ms);
  }
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const int macs[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int s = 0; s < 4; ++s) {
    const int iters = 2048 >> s;
    auto L = [&] {
      if (s == 0) k_dmma<0><<<blocks, threads>>>(out, iters);
      if (s == 1) k_dmma<1><<<blocks, threads>>>(out, iters);
      if (s == 2) k_dmma<2><<<blocks, threads>>>(out, iters);
      if (s == 3) k_dmma<3><<<blocks, threads>>>(out, iters);
    };
    if (timeit(L, &r)) return 1;
    double fmas = (nthreads / 32) * iters * 16.0 * macs[s];
    printf(", \"dmma_%s\": {\"tflops\": %.3f, \"fma_per_clk_per_sm\": %.2f, \"mhz\": %.0f, \"ms\": %.3f}", names[s],
           2 * fmas / r.ms / 1e9, fmas / (r.ms * 1e-3) / (r.mhz * 1e6) / sms, r.mhz, r.ms);
  }
  // Overlap: per iteration 8 DMMA m8n8k4 (2048 FMA/warp... x32 lanes) and NF*8 DFMA per thread.
  {
    const int iters = 1024;
    auto run_same = [&](auto kern, int nm, int nf, const char* tag) -> int {
      if (timeit([&] { kern<<<blocks, threads>>>(out, iters, 0.999999, 1e-9); }, &r)) return 1;
      double fm = (nthreads / 32) * iters * nm * 256.0;
      double ff = nthreads * iters * nf * 8.0;
      printf(", \"%s\": {\"ms\": %.3f, \"dmma_fma\": %.4g, \"dfma_fma\": %.4g, \"total_tflops\": %.3f, \"mhz\": %.0f}", tag,
             r.ms, fm, ff, 2 * (fm + ff) / r.ms / 1e9, r.mhz);
      return 0;
    };
    if (run_same(k_mixed_same<8, 0>, 8, 0, "same_dmma_only")) return 1;
    if (run_same(k_mixed_same<0, 8>, 0, 8, "same_dfma_only")) return 1;
    if (run_same(k_mixed_same<8, 8>, 8, 8, "same_dmma8_dfma8")) return 1;
    if (run_same(k_mixed_same<8, 4>, 8, 4, "same_dmma8_dfma4")) return 1;
    // split: half the warps do each; per-warp work counts halve.
    auto run_split = [&](auto kern, int nm, int nf, const char* tag) -> int {
      if (timeit([&] { kern<<<blocks, threads>>>(out, iters, 0.999999, 1e-9); }, &r)) return 1;
      double fm = (nthreads / 64) * iters * nm * 256.0;
      double ff = (nthreads / 2) * iters * nf * 8.0;
      printf(", \"%s\": {\"ms\": %.3f, \"dmma_fma\": %.4g, \"dfma_fma\": %.4g, \"total_tflops\": %.3f, \"mhz\": %.0f}", tag,
             r.ms, fm, ff, 2 * (fm + ff) / r.ms / 1e9, r.mhz);
      return 0;
    };
    if (run_split(k_mixed_split<16, 16>, 16, 16, "split_dmma16_dfma16")) return 1;
    if (run_split(k_mixed_split<16, 0>, 16, 0, "split_dmma16_idle")) return 1;
    if (run_split(k_mixed_split<0, 16>, 0, 16, "split_idle_dfma16")) return 1;
  }
  {
    const char* tn[4] = {"exp", "log1p", "log", "log1p_exp"};
    for (int op = 0; op < 4; ++op) {
      const int iters = 256;
      auto L = [&] {
        if (op == 0) k_transc<0><<<blocks, threads>>>(out, iters);
        if (op == 1) k_transc<1><<<blocks, threads>>>(out, iters);
        if (op == 2) k_transc<2><<<blocks, threads>>>(out, iters);
        if (op == 3) k_transc<3><<<blocks, threads>>>(out, iters);
      };
      if (timeit(L, &r)) return 1;
      double n = nthreads * iters * 4;
      printf(", \"%s\": {\"gops\": %.3f, \"ns_per_sm_op\": %.5f, \"mhz\": %.0f}", tn[op], n / r.ms / 1e6,
             r.ms * 1e6 / n * sms, r.mhz);
    }
  }
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
