// Probe: per-kernel cost of a chain of tiny dependent kernels inside a conditional
// WHILE graph body, with and without programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_work(double* v, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = v[i] * 1.0000001 + 1.0;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}
__global__ void k_ctl(cudaGraphConditionalHandle h, int* it, int lim, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int v = ++(*it);
  cudaGraphSetConditional(h, v < lim ? 1 : 0);
}
__global__ void k_reset(cudaGraphConditionalHandle h, int* it) { *it = 0; cudaGraphSetConditional(h, 1); }

int run(int pdl, int nblk) {
  cudaStream_t s0, s1;
  CK(cudaStreamCreate(&s0)); CK(cudaStreamCreate(&s1));
  int* it; double* v;
  int n = nblk * 256;
  CK(cudaMalloc(&it, 4)); CK(cudaMalloc(&v, n * 8)); CK(cudaMemset(v, 0, n * 8));
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* d; size_t nd;
  CK(cudaStreamGetCaptureInfo(s0, &st, nullptr, &g, &d, &nd));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
  k_reset<<<1, 1, 0, s0>>>(h, it);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional; p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaStreamGetCaptureInfo(s0, &st, nullptr, &g, &d, &nd));
  CK(cudaGraphAddNode(&node, g, d, nd, &p));
  CK(cudaStreamUpdateCaptureDependencies(s0, &node, 1, cudaStreamSetCaptureDependencies));
  CK(cudaStreamBeginCaptureToGraph(s1, p.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  for (int k = 0; k < 20; k++) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk); cfg.blockDim = dim3(256); cfg.stream = s1;
    cfg.attrs = pdl ? at : nullptr; cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k_work, v, n, pdl));
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(1); cfg.stream = s1;
    cfg.attrs = pdl ? at : nullptr; cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k_ctl, h, it, 100, pdl));
  }
  CK(cudaStreamEndCapture(s1, nullptr));
  cudaGraph_t graph;
  CK(cudaStreamEndCapture(s0, &graph));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, graph, 0));
  CK(cudaGraphLaunch(ex, s0)); CK(cudaStreamSynchronize(s0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s0);
  for (int r = 0; r < 5; r++) CK(cudaGraphLaunch(ex, s0));
  cudaEventRecord(b, s0);
  CK(cudaStreamSynchronize(s0));
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("pdl=%d blocks=%d: %.3f us per kernel node\n", pdl, nblk, ms * 1e3 / (5 * 100 * 21));
  return 0;
}
int main() {
  for (int nblk : {1, 148, 3168}) { run(0, nblk); run(1, nblk); }
  return 0;
}
