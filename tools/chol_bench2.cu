#include <cstdio>
// isolate: (1) pivot chain only, (2) full warp cholesky with compile-time D
template <int D, int MODE>
__global__ void kb(const double* V, long long* out, double* L) {
  __shared__ double colbuf[33];
  __shared__ double sV[D * D];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) sV[i] = V[i];
  __syncthreads();
  long long t0 = clock64();
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l) a[l] = lane < D ? sV[lane * D + l] : 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (lane == j) colbuf[32] = rsqrt(a[j]);
    __syncwarp();
    const double r = colbuf[32];
    const double lij = lane >= j ? a[j] * r : 0.0;
    a[j] = lij;
    if (MODE == 1) {
      colbuf[lane] = lij;
      __syncwarp();
#pragma unroll
      for (int l = j + 1; l < D; ++l)
        if (lane >= l) a[l] = fma(-lij, colbuf[l], a[l]);
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (lane < D)
    for (int l = 0; l < D; ++l) L[lane * D + l] = a[l];
}
int main() {
  const int d = 25;
  double h[d * d];
  for (int i = 0; i < d; ++i) for (int j = 0; j < d; ++j) h[i * d + j] = (i == j ? d + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *V, *L; long long* o;
  cudaMalloc(&V, sizeof h); cudaMalloc(&L, sizeof h); cudaMallocManaged(&o, 16);
  cudaMemcpy(V, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) kb<25, 0><<<1, 32>>>(V, o, L);
  cudaDeviceSynchronize(); printf("pivot-chain only: %lld cycles\n", o[0]);
  for (int r = 0; r < 3; ++r) kb<25, 1><<<1, 32>>>(V, o, L);
  cudaDeviceSynchronize(); printf("full, D=25 template: %lld cycles\n", o[0]);
  double hl[d * d]; cudaMemcpy(hl, L, sizeof h, cudaMemcpyDeviceToHost);
  printf("L00 %.6f L24_23 %.6f\n", hl[0], hl[24 * d + 23]);
}
