// Microbenchmark: Cholesky variants for the finalize kernel (d = 25), clock64 per call.
#include <cstdio>
#include "../paper_1304_4333_b200/csrc/mstep.cuh"
using namespace sps;

__global__ void kb(const double* V, int d, int variant, long long* out, double* L) {
  extern __shared__ double sm[];
  __shared__ int flag;
  double* sV = sm;
  double* sA = sm + d * d;
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) sV[i] = V[i];
  __syncthreads();
  long long t0 = clock64();
  bool ok = true;
  if (variant == 0) {
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) sA[i] = 0.5 * sV[i];
    __syncthreads();
    ok = block_cholesky(sA, d, &flag);
  } else if (threadIdx.x < 32) {
    __shared__ double colb[33];
    ok = warp_cholesky32(sV, d, 0.5, 0.0, sA, colb);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = ok; }
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) L[i] = sA[i];
}

int main() {
  const int d = 25;
  double h[d * d];
  for (int i = 0; i < d; ++i) for (int j = 0; j < d; ++j) h[i * d + j] = (i == j ? d + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *V, *L; long long* o;
  cudaMalloc(&V, sizeof h); cudaMalloc(&L, sizeof h); cudaMallocManaged(&o, 16);
  cudaMemcpy(V, h, sizeof h, cudaMemcpyHostToDevice);
  for (int v = 0; v < 2; ++v) {
    for (int threads : {32, 256, 512}) {
      if (v == 0 && threads == 32) continue;
      for (int rep = 0; rep < 3; ++rep) kb<<<1, threads, 2 * sizeof h>>>(V, d, v, o, L);
      cudaDeviceSynchronize();
      double hl[d * d]; cudaMemcpy(hl, L, sizeof h, cudaMemcpyDeviceToHost);
      printf("variant %d threads %d cycles %lld ok %lld L00 %.6f L24_23 %.6f err %s\n", v, threads, o[0], o[1], hl[0], hl[24 * d + 23], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
