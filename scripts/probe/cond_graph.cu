// Probe: nested conditional WHILE nodes built by stream capture (CUDA 12.4+),
// device-side cudaGraphSetConditional.  Outer loop 3 times, inner loop 5 times;
// counter must be 15 after one graph launch, and 30 after two.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_inc(int* c) { atomicAdd(c, 1); }
__global__ void k_set(cudaGraphConditionalHandle h, int* it, int lim) {
  int v = ++(*it);
  cudaGraphSetConditional(h, v < lim ? 1 : 0);
}
__global__ void k_reset(cudaGraphConditionalHandle h, int* it) { *it = 0; cudaGraphSetConditional(h, 1); }

static cudaGraphNode_t add_while(cudaStream_t s, cudaGraphConditionalHandle* h, cudaGraph_t* body) {
  cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
  cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
  cudaGraphConditionalHandleCreate(h, g, 0, 0);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = *h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, deps, nd, &p);
  if (e != cudaSuccess) printf("add node: %s\n", cudaGetErrorString(e));
  *body = p.conditional.phGraph_out[0];
  cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
  return node;
}

int main() {
  cudaStream_t s0, s1, s2;
  CK(cudaStreamCreate(&s0)); CK(cudaStreamCreate(&s1)); CK(cudaStreamCreate(&s2));
  int *c, *it;
  CK(cudaMalloc(&c, 4)); CK(cudaMalloc(&it, 8));
  CK(cudaMemset(c, 0, 4)); CK(cudaMemset(it, 0, 8));
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  cudaGraphConditionalHandle ho, hi; cudaGraph_t bo, bi;
  // outer: need the handle value 1 on entry: set by a kernel before the node
  cudaStreamCaptureStatus st; cudaGraph_t g0; const cudaGraphNode_t* d; size_t nd;
  CK(cudaStreamGetCaptureInfo(s0, &st, nullptr, &g0, &d, &nd));
  CK(cudaGraphConditionalHandleCreate(&ho, g0, 0, 0));
  k_reset<<<1, 1, 0, s0>>>(ho, it);
  {
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional; p.conditional.handle = ho; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaStreamGetCaptureInfo(s0, &st, nullptr, &g0, &d, &nd));
    CK(cudaGraphAddNode(&node, g0, d, nd, &p));
    bo = p.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(s0, &node, 1, cudaStreamSetCaptureDependencies));
  }
  CK(cudaStreamBeginCaptureToGraph(s1, bo, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  {
    CK(cudaStreamGetCaptureInfo(s1, &st, nullptr, &g0, &d, &nd));
    CK(cudaGraphConditionalHandleCreate(&hi, bo, 0, 0));
    k_reset<<<1, 1, 0, s1>>>(hi, it + 1);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional; p.conditional.handle = hi; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaStreamGetCaptureInfo(s1, &st, nullptr, &g0, &d, &nd));
    CK(cudaGraphAddNode(&node, g0, d, nd, &p));
    bi = p.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(s1, &node, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(s2, bi, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_inc<<<1, 1, 0, s2>>>(c);
    k_set<<<1, 1, 0, s2>>>(hi, it + 1, 5);
    CK(cudaStreamEndCapture(s2, nullptr));
    k_set<<<1, 1, 0, s1>>>(ho, it, 3);
  }
  CK(cudaStreamEndCapture(s1, nullptr));
  cudaGraph_t graph;
  CK(cudaStreamEndCapture(s0, &graph));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, graph, 0));
  CK(cudaGraphLaunch(ex, s0));
  CK(cudaStreamSynchronize(s0));
  int h = 0;
  CK(cudaMemcpy(&h, c, 4, cudaMemcpyDeviceToHost));
  printf("after 1 launch: %d (expect 15)\n", h);
  CK(cudaGraphLaunch(ex, s0));
  CK(cudaStreamSynchronize(s0));
  CK(cudaMemcpy(&h, c, 4, cudaMemcpyDeviceToHost));
  printf("after 2 launches: %d (expect 30)\n", h);
  // timing: empty-ish loop of 1000 iterations of 3 tiny kernels
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s0);
  for (int r = 0; r < 100; r++) cudaGraphLaunch(ex, s0);
  cudaEventRecord(b, s0);
  CK(cudaStreamSynchronize(s0));
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("100 launches x (3 outer x (1 + 5x2 + 1) kernels): %.3f ms -> %.2f us per kernel node\n", ms, ms * 1e3 / (100 * 3 * 12));
  return 0;
}
