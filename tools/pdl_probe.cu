#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void prim(int* x) {
  asm volatile("griddepcontrol.launch_dependents;");
  for (int i = 0; i < 1000; ++i) atomicAdd(x, 1);
}
__global__ void dep(int* x, int* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = *x;
}
int main() {
  int *x, *out; cudaMalloc(&x, 4); cudaMalloc(&out, 4); cudaMemset(x, 0, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  auto launch = [&](int pdl) {
    prim<<<148, 128, 0, s>>>(x);
    cudaLaunchConfig_t cfg{}; cfg.gridDim = 148; cfg.blockDim = 256; cfg.stream = s;
    cudaLaunchAttribute a[2]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
    a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization; a[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a; cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, dep, x, out);
  };
  printf("stream pdl: %s\n", cudaGetErrorString(launch(1)));
  printf("sync: %s\n", cudaGetErrorString(cudaStreamSynchronize(s)));
  int h; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost); printf("out %d (expect 148000)\n", h);
  // graph with conditional while body
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle c; printf("cond: %s\n", cudaGetErrorString(cudaGraphConditionalHandleCreate(&c, g, 1, cudaGraphCondAssignDefault)));
  cudaGraphNodeParams cp{}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = c;
  cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t loop; printf("add: %s\n", cudaGetErrorString(cudaGraphAddNode(&loop, g, nullptr, 0, &cp)));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  printf("begin: %s\n", cudaGetErrorString(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)));
  printf("launch in capture: %s\n", cudaGetErrorString(launch(1)));
  cudaGraph_t tmp; printf("end: %s\n", cudaGetErrorString(cudaStreamEndCapture(s, &tmp)));
  cudaGraphExec_t ge; printf("inst: %s\n", cudaGetErrorString(cudaGraphInstantiate(&ge, g, 0)));
  printf("(body loops forever without a condition setter; not launched)\n");
  return 0;
}
