// Dependent-launch cost on B200: chains of kernels that each read the previous
// kernel's output, launched (A) plainly on a stream, (B) with programmatic
// dependent launch (PDL: the next grid is scheduled while the previous runs and
// waits in griddepcontrol.wait), (C) as a captured CUDA graph, (D) graph of PDL
// launches.  Reports us per kernel for a 1-block and a 296-block grid.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kchain(double* buf, int n, int iters, int pdl) {
  // prologue independent of the predecessor (what PDL overlaps)
  double x = threadIdx.x * 1e-3;
  for (int i = 0; i < 16; ++i) x = fma(x, 0.999, 0.001);
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double v = t < n ? buf[t] : 0.0;
  for (int i = 0; i < iters; ++i) v = fma(v, 0.999, x);
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (t < n) buf[t] = v;
}
int main() {
  double* buf;
  cudaMalloc(&buf, 1 << 24);
  cudaMemset(buf, 0, 1 << 24);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int N = 400;
  struct G { int grid, iters; } gs[] = {{1, 10}, {296, 10}, {296, 2000}};
  for (auto g : gs) {
    const int n = g.grid * 256;
    auto launch = [&](bool pdl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(g.grid);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, kchain, buf, n, g.iters, pdl ? 1 : 0);
    };
    for (int mode = 0; mode < 4; ++mode) {
      const bool pdl = mode == 1 || mode == 3, graph = mode >= 2;
      cudaGraphExec_t ge = nullptr;
      if (graph) {
        cudaGraph_t gr;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) launch(pdl);
        cudaStreamEndCapture(s, &gr);
        if (cudaGraphInstantiate(&ge, gr, 0) != cudaSuccess) {
          printf("instantiate failed mode %d\n", mode);
          continue;
        }
        cudaGraphLaunch(ge, s);  // warm
      } else {
        for (int i = 0; i < 20; ++i) launch(pdl);
      }
      cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      if (graph)
        cudaGraphLaunch(ge, s);
      else
        for (int i = 0; i < N; ++i) launch(pdl);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* nm[] = {"stream", "stream+PDL", "graph", "graph+PDL"};
      printf("grid %4d iters %5d %-11s: %.2f us/kernel  (%s)\n", g.grid, g.iters, nm[mode], 1000 * ms / N,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
