// Probe: device-side WHILE loop over a captured multi-stream body (conditional graph node).
// The body: k_work (main) -> fork -> k_side (aux) ; k_dec (main) sets the condition; join.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_work(double* buf, int iters) {
  double v = buf[threadIdx.x];
  for (int i = 0; i < iters; ++i) v = fma(v, 0.999, 0.001);
  buf[threadIdx.x] = v;
}
__global__ void k_side(int* side_count) { if (threadIdx.x == 0) atomicAdd(side_count, 1); }
__global__ void k_dec(int* counter, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) {
    const int c = --(*counter);
    cudaGraphSetConditional(h, c > 0 ? 1u : 0u);
  }
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)
int main() {
  double* buf; int *counter, *side;
  CK(cudaMalloc(&buf, 8 * 256)); CK(cudaMemset(buf, 0, 8 * 256));
  CK(cudaMallocManaged(&counter, 4)); CK(cudaMallocManaged(&side, 4));
  cudaStream_t s, aux; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
  cudaEvent_t ef, ej; CK(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming)); CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h; CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {}; np.type = cudaGraphNodeTypeConditional; np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile; np.conditional.size = 1;
  cudaGraphNode_t cn; CK(cudaGraphAddNode(&cn, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  k_work<<<1, 256, 0, s>>>(buf, 100);
  CK(cudaEventRecord(ef, s)); CK(cudaStreamWaitEvent(aux, ef, 0));
  k_side<<<1, 32, 0, aux>>>(side);
  CK(cudaEventRecord(ej, aux));
  k_dec<<<1, 32, 0, s>>>(counter, h);
  CK(cudaStreamWaitEvent(s, ej, 0));
  CK(cudaStreamEndCapture(s, &body));
  cudaGraphExec_t ge; CK(cudaGraphInstantiateWithFlags(&ge, g, cudaGraphInstantiateFlagUseNodePriority));
  for (int trial = 0; trial < 3; ++trial) {
    *counter = 1000; *side = 0;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaEventRecord(e0, s)); CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s)); CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("trial %d: counter %d side %d  %.2f us/iteration\n", trial, *counter, *side, 1000 * ms / 1000);
  }
  printf("ok: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
