// Launch floor: empty / trivial kernels of various grid and dynamic-smem sizes, back-to-back, CUDA events.
#include <cstdio>
__global__ void kempty(int* flag) {
  extern __shared__ double sm[];
  if (flag && *flag == 12345) sm[threadIdx.x] = 1.0;
}
__global__ void kwork(double* out, int iters) {
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 0.001);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
int main() {
  int* flag; cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaFuncSetAttribute(kempty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int grid, block, smem; } cfgs[] = {{1, 32, 0}, {1, 256, 0}, {148, 256, 0}, {1024, 256, 0}, {1024, 256, 56 * 1024},
                                                 {4096, 256, 0}, {256, 256, 75 * 1024}, {296, 256, 56 * 1024}};
  for (auto c : cfgs) {
    for (int w = 0; w < 10; ++w) kempty<<<c.grid, c.block, c.smem>>>(flag);
    cudaEventRecord(e0);
    const int N = 200;
    for (int i = 0; i < N; ++i) kempty<<<c.grid, c.block, c.smem>>>(flag);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("empty grid %5d block %3d smem %6d : %.2f us/launch\n", c.grid, c.block, c.smem, 1000 * ms / N);
  }
  // event pair overhead
  cudaEvent_t a[400];
  for (int i = 0; i < 400; ++i) cudaEventCreate(&a[i]);
  kwork<<<148, 256>>>(out, 100000);
  for (int i = 0; i < 400; i += 2) { cudaEventRecord(a[i]); cudaEventRecord(a[i + 1]); }
  cudaDeviceSynchronize();
  float tot = 0; for (int i = 0; i < 400; i += 2) { float ms; cudaEventElapsedTime(&ms, a[i], a[i + 1]); tot += ms; }
  printf("empty event pair (queued behind work): %.2f us\n", 1000 * tot / 200);
  // dependent chain of small work kernels
  for (int iters : {10, 1000}) {
    cudaEventRecord(e0);
    for (int i = 0; i < 200; ++i) kwork<<<1024, 256>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("kwork 1024x256 iters %d: %.2f us/launch\n", iters, 1000 * ms / 200);
  }
  return 0;
}
