#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(int* c, cudaGraphConditionalHandle h) { int v = ++(*c); cudaGraphSetConditional(h, v < 10); }
int main() {
  cudaStream_t s, s2; cudaStreamCreate(&s); cudaStreamCreate(&s2);
  int* c; cudaMalloc(&c, 4); cudaMemset(c, 0, 4);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaStreamCaptureStatus st; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
  cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
  cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional; p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t n; cudaGraphAddNode(&n, cg, deps, nd, &p);
  cudaStreamUpdateCaptureDependencies(s, &n, 1, cudaStreamSetCaptureDependencies);
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  body<<<1,1,0,s2>>>(c, h);
  cudaStreamEndCapture(s2, &bodyg);
  cudaStreamEndCapture(s, &g);
  printf("inst %d\n", (int)cudaGraphInstantiate(&ge, g, 0));
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  int hc; cudaMemcpy(&hc, c, 4, cudaMemcpyDeviceToHost); printf("count %d err %s\n", hc, cudaGetErrorString(cudaGetLastError()));
}
