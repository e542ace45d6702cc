// Cholesky variants for the finalize kernel (one warp of a 256-thread block,
// d = 25): cycles per factorization, cold (first call) and warm.
#include <cstdio>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = fma(y, fma(-h * y, y, 0.5), y);
  y = fma(y, fma(-h * y, y, 0.5), y);
  return y;
}
// V1: smem, lane-divergent trip counts (engine)
__device__ void chol_v1(double* A, int ld, int d) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < d; ++j) {
    const double r = rsqrt_nr(A[j * ld + j]);
    double lij = 0.0;
    if (lane >= j && lane < d) { lij = A[lane * ld + j] * r; A[lane * ld + j] = lij; }
    __syncwarp();
    if (lane > j && lane < d)
#pragma unroll 4
      for (int l = j + 1; l <= lane; ++l) A[lane * ld + l] = fma(-lij, A[l * ld + j], A[lane * ld + l]);
    __syncwarp();
  }
}
// V3: smem, uniform trip count, predicated
__device__ void chol_v3(double* A, int ld, int d) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < d; ++j) {
    const double r = rsqrt_nr(A[j * ld + j]);
    const double lij = (lane >= j && lane < d) ? A[lane * ld + j] * r : 0.0;
    if (lane >= j && lane < d) A[lane * ld + j] = lij;
    __syncwarp();
    const int row = lane < d ? lane : d - 1;
#pragma unroll 4
    for (int l = j + 1; l < d; ++l) {
      const double v = fma(-lij, A[l * ld + j], A[row * ld + l]);
      if (l <= lane && lane < d) A[row * ld + l] = v;
    }
    __syncwarp();
  }
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  return y;
}
// V5: smem rows, column j copied to a separate buffer (no aliasing with the row updates)
__device__ void chol_v5(double* A, int ld, int d, double* colbuf) {
  const int lane = threadIdx.x & 31;
  double* Ar = A + (lane < d ? lane : 0) * ld;
  for (int j = 0; j < d; ++j) {
    const double r = rsqrt_nr(A[j * ld + j]);
    const double lij = (lane >= j && lane < d) ? Ar[j] * r : 0.0;
    colbuf[lane] = lij;
    if (lane >= j && lane < d) Ar[j] = lij;
    __syncwarp();
    if (lane > j && lane < d)
#pragma unroll 4
      for (int l = j + 1; l <= lane; ++l) Ar[l] = fma(-lij, colbuf[l], Ar[l]);
    __syncwarp();
  }
}
// V6: LDL' (reciprocal pivots in the chain), sqrt scaling at the end
__device__ void chol_v6(double* A, int ld, int d, double* colbuf, double* dbuf) {
  const int lane = threadIdx.x & 31;
  double* Ar = A + (lane < d ? lane : 0) * ld;
  for (int j = 0; j < d; ++j) {
    const double Dj = A[j * ld + j];
    const double rj = rcp_nr(Dj);
    const double u = (lane > j && lane < d) ? Ar[j] : 0.0;  // unscaled column entry
    colbuf[lane] = u;
    const double lij = u * rj;
    if (lane > j && lane < d) Ar[j] = lij;
    if (lane == j) dbuf[j] = Dj;
    __syncwarp();
    if (lane > j && lane < d)
#pragma unroll 4
      for (int l = j + 1; l <= lane; ++l) Ar[l] = fma(-lij, colbuf[l], Ar[l]);
    __syncwarp();
  }
  // L = Lunit sqrt(D)
  if (lane < d) {
    for (int l = 0; l < lane; ++l) Ar[l] = Ar[l] * sqrt(dbuf[l]);
    Ar[lane] = sqrt(dbuf[lane]);
  }
  __syncwarp();
}
// V7: registers (A padded to D x D with identity, no load guards); the next
// pivot (column j+1 of lane j+1) uses the lane's own lij (no smem round trip)
template <int D>
__device__ void chol_v7(const double* Ap, double* Lout, int ldo, int d, double* colbuf) {
  const int lane = threadIdx.x & 31;
  const int row = lane < D ? lane : D - 1;
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l) a[l] = Ap[row * D + l];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j < d) {
      const double r = rsqrt_nr(__shfl_sync(0xffffffffu, a[j], j));
      const double lij = lane >= j ? a[j] * r : 0.0;
      a[j] = lij;
      colbuf[lane] = lij;
      __syncwarp();
      if (j + 1 < D) a[j + 1] = fma(-lij, lane == j + 1 ? lij : colbuf[j + 1], a[j + 1]);
#pragma unroll
      for (int l = j + 2; l < D; ++l) a[l] = fma(-lij, colbuf[l], a[l]);
      __syncwarp();
    }
  }
  if (lane < d)
#pragma unroll
    for (int l = 0; l < D; ++l)
      if (l < d) Lout[lane * ldo + l] = l <= lane ? a[l] : 0.0;
}
// V8: registers, column broadcast by shuffles (no shared memory, no warp barriers)
template <int D>
__device__ void chol_v8(const double* Ap, double* Lout, int ldo, int d) {
  const int lane = threadIdx.x & 31;
  const int row = lane < D ? lane : D - 1;
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l) a[l] = Ap[row * D + l];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j < d) {
      const double r = rsqrt_nr(__shfl_sync(0xffffffffu, a[j], j));
      const double lij = lane >= j ? a[j] * r : 0.0;
      a[j] = lij;
#pragma unroll
      for (int l = j + 1; l < D; ++l) a[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l), a[l]);
    }
  }
  if (lane < d)
#pragma unroll
    for (int l = 0; l < D; ++l)
      if (l < d) Lout[lane * ldo + l] = l <= lane ? a[l] : 0.0;
}
// V2: registers, fully unrolled (previous engine)
template <int D>
__device__ void chol_v2(double* A, int ld, int d, double* colbuf) {
  const int lane = threadIdx.x & 31;
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l) a[l] = (lane < d && l < d) ? A[lane * ld + l] : (lane == l ? 1.0 : 0.0);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double r = rsqrt_nr(__shfl_sync(0xffffffffu, a[j], j));
    const double lij = lane >= j ? a[j] * r : 0.0;
    a[j] = lij;
    if (j + 1 < D) {
      colbuf[lane] = lij;
      __syncwarp();
#pragma unroll
      for (int l = j + 1; l < D; ++l) a[l] = fma(-lij, colbuf[l], a[l]);
      __syncwarp();
    }
  }
  if (lane < d)
    for (int l = 0; l < d; ++l) A[lane * ld + l] = a[l];
}
// V4: registers, run-time column loop, predicated static inner loop
template <int D>
__device__ void chol_v4(double* A, int ld, int d, double* colbuf) {
  const int lane = threadIdx.x & 31;
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l) a[l] = (lane < d && l < d) ? A[lane * ld + l] : (lane == l ? 1.0 : 0.0);
  for (int j = 0; j < d; ++j) {
    double ajj = a[0];
#pragma unroll
    for (int l = 1; l < D; ++l) ajj = (l == j) ? a[l] : ajj;
    const double r = rsqrt_nr(__shfl_sync(0xffffffffu, ajj, j));
    const double lij = lane >= j ? ajj * r : 0.0;
    colbuf[lane] = lij;
    __syncwarp();
#pragma unroll
    for (int l = 0; l < D; ++l) {
      if (l == j) a[l] = lij;
      else if (l > j) a[l] = fma(-lij, colbuf[l], a[l]);
    }
    __syncwarp();
  }
  if (lane < d)
    for (int l = 0; l < d; ++l) A[lane * ld + l] = a[l];
}
template <int V>
__global__ void kb(const double* M, int d, long long* out, double* L, int reps) {
  __shared__ double A[32 * 33];
  __shared__ double colbuf[32];
  __shared__ double dbuf[32];
  __shared__ double Ap[28 * 28];
  const int ld = d | 1;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) A[(i / d) * ld + i % d] = M[i];
    for (int i = threadIdx.x; i < 28 * 28; i += blockDim.x) {
      const int r = i / 28, c = i % 28;
      Ap[i] = (r < d && c < d) ? M[r * d + c] : (r == c ? 1.0 : 0.0);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      __syncwarp();
      long long t0 = clock64();
      if (V == 1) chol_v1(A, ld, d);
      if (V == 2) chol_v2<28>(A, ld, d, colbuf);
      if (V == 3) chol_v3(A, ld, d);
      if (V == 4) chol_v4<28>(A, ld, d, colbuf);
      if (V == 5) chol_v5(A, ld, d, colbuf);
      if (V == 6) chol_v6(A, ld, d, colbuf, dbuf);
      if (V == 7) chol_v7<28>(Ap, A, ld, d, colbuf);
      if (V == 8) chol_v8<28>(Ap, A, ld, d);
      __syncwarp();
      long long t1 = clock64();
      if (threadIdx.x == 0) out[r] = t1 - t0;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) L[i] = A[(i / d) * ld + i % d];
}
int main() {
  const int d = 25;
  double h[d * d];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) h[i * d + j] = (i == j ? d + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *M, *L;
  long long* o;
  cudaMalloc(&M, sizeof h);
  cudaMalloc(&L, sizeof h);
  cudaMallocManaged(&o, 64 * 8);
  cudaMemcpy(M, h, sizeof h, cudaMemcpyHostToDevice);
  double ref[d * d];
  for (int v = 1; v <= 8; ++v) {
    if (v == 4) continue;
    for (int launch = 0; launch < 2; ++launch) {
      if (v == 1) kb<1><<<1, 256>>>(M, d, o, L, 5);
      if (v == 2) kb<2><<<1, 256>>>(M, d, o, L, 5);
      if (v == 3) kb<3><<<1, 256>>>(M, d, o, L, 5);
      if (v == 5) kb<5><<<1, 256>>>(M, d, o, L, 5);
      if (v == 6) kb<6><<<1, 256>>>(M, d, o, L, 5);
      if (v == 7) kb<7><<<1, 256>>>(M, d, o, L, 5);
      if (v == 8) kb<8><<<1, 256>>>(M, d, o, L, 5);
      cudaDeviceSynchronize();
      printf("V%d launch %d cycles:", v, launch);
      for (int r = 0; r < 5; ++r) printf(" %lld", o[r]);
      printf("\n");
    }
    double hl[d * d];
    cudaMemcpy(hl, L, sizeof h, cudaMemcpyDeviceToHost);
    if (v == 1) for (int i = 0; i < d * d; ++i) ref[i] = hl[i];
    double md = 0;
    for (int i = 0; i < d; ++i) for (int j = 0; j <= i; ++j) md = fmax(md, fabs(hl[i * d + j] - ref[i * d + j]));
    printf("V%d max |L - L_v1| (lower) = %.3g, L00 %.6f\n", v, md, hl[0]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
