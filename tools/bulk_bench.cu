// Global -> shared copy throughput on B200: TMA bulk copies (one thread per CTA,
// chunk sizes 4..64 KB, up to 4 in flight) vs cp.async 16 B vs plain 16 B loads,
// from an L2-resident (32 MB) and a DRAM-resident (1 GB) source.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k_bulk(const double* src, size_t nbytes, int chunk, int inflight, double* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[4];
  if (threadIdx.x == 0)
    for (int i = 0; i < inflight; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const size_t nchunks = nbytes / chunk;
  unsigned ph[4] = {0, 0, 0, 0};
  double acc = 0;
  for (size_t c0 = (size_t)blockIdx.x * inflight; c0 < nchunks; c0 += (size_t)gridDim.x * inflight) {
    if (threadIdx.x == 0)
      for (int i = 0; i < inflight && c0 + i < nchunks; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(chunk));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + i * chunk)),
                     "l"((const char*)src + (c0 + i) * chunk), "r"(chunk), "r"(smem_u32(&bar[i]))
                     : "memory");
      }
    for (int i = 0; i < inflight && c0 + i < nchunks; ++i) {
      asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                       smem_u32(&bar[i])),
                   "r"(ph[i]));
      ph[i] ^= 1;
      acc += ((const double*)(sm + i * chunk))[threadIdx.x];
    }
    __syncthreads();
  }
  if (acc == 12345.0) sink[0] = acc;
}
__global__ void k_ldg(const double2* src, size_t n2, double* sink) {
  double a = 0, b = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcg(src + i);
    a += v.x;
    b += v.y;
  }
  if (a + b == 12345.0) sink[0] = a;
}
__global__ void k_cpasync(const double2* src, size_t n2, double* sink) {
  extern __shared__ __align__(16) double2 s2[];
  const int per = 8;  // 16 B x 8 per thread in flight
  double acc = 0;
  for (size_t base = (size_t)blockIdx.x * blockDim.x * per; base < n2; base += (size_t)gridDim.x * blockDim.x * per) {
    for (int u = 0; u < per; ++u) {
      const size_t i = base + (size_t)u * blockDim.x + threadIdx.x;
      if (i < n2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&s2[u * blockDim.x + threadIdx.x])),
                     "l"(src + i));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    acc += s2[threadIdx.x].x;
  }
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  double* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (size_t nbytes : {(size_t)32 << 20, (size_t)1 << 30}) {
    double* src;
    cudaMalloc(&src, nbytes);
    cudaMemset(src, 0, nbytes);
    auto timeit = [&](auto fn) {
      fn();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      const int R = nbytes > (64u << 20) ? 3 : 20;
      for (int r = 0; r < R; ++r) fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      return (double)nbytes * R / (ms * 1e-3) / 1e9;
    };
    printf("source %zu MB:\n", nbytes >> 20);
    for (int grid : {148, 296}) {
      for (int chunk : {4096, 16384, 65536}) {
        for (int inflight : {1, 2, 4}) {
          if ((size_t)chunk * inflight > 200 * 1024) continue;
          if (grid == 296 && (size_t)chunk * inflight > 100 * 1024) continue;
          const double gbs = timeit([&] { k_bulk<<<grid, 256, chunk * inflight>>>(src, nbytes, chunk, inflight, sink); });
          printf("  bulk grid %3d chunk %6d inflight %d : %7.0f GB/s\n", grid, chunk, inflight, gbs);
        }
      }
    }
    for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
      const double g1 = timeit([&] { k_ldg<<<grid, 256>>>((const double2*)src, nbytes / 16, sink); });
      printf("  ldg.128 grid %4d : %7.0f GB/s\n", grid, g1);
    }
    for (int grid : {148 * 2, 148 * 4}) {
      const double g2 =
          timeit([&] { k_cpasync<<<grid, 256, 256 * 8 * 16>>>((const double2*)src, nbytes / 16, sink); });
      printf("  cp.async16 x8 grid %4d : %7.0f GB/s\n", grid, g2);
    }
    cudaFree(src);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
