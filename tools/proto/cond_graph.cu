// Feasibility probe: a device-driven loop as a CUDA graph WHILE node whose
// body is [control kernel -> SWITCH(action) {bodies}], with a cooperative
// kernel and a PDL-launched kernel inside a body. Prints per-iteration time.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#ifndef NWORK
#define NWORK (1 << 20)
#endif
namespace cg = cooperative_groups;

struct Ctl { int iter, niter, action; };

__global__ void k_ctl(Ctl* c, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs) {
  c->iter += 1;
  c->action = c->iter & 1;
  cudaGraphSetConditional(hs, (unsigned)c->action);
  cudaGraphSetConditional(hw, c->iter < c->niter ? 1u : 0u);
}
__global__ void k_coop(double* v, int n) {
  cg::grid_group g = cg::this_grid();
  asm volatile("griddepcontrol.launch_dependents;");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] += 1.0;
  g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) v[0] += 1.0;
}
__global__ void k_pdl(double* v, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] *= 1.0000001;
}
__global__ void k_plain(double* v) { if (threadIdx.x == 0) v[1] += 2.0; }

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* v; CK(cudaMalloc(&v, sizeof(double) * 1 << 20)); CK(cudaMemset(v, 0, sizeof(double) * (1 << 20)));
  Ctl* c; CK(cudaMalloc(&c, sizeof(Ctl)));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw, hs;
  CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {}; wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw; wp.conditional.type = cudaGraphCondTypeWhile; wp.conditional.size = 1;
  cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  CK(cudaGraphConditionalHandleCreate(&hs, body, 0, 0));
  // body: ctl kernel -> switch
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_ctl<<<1, 1, 0, s>>>(c, hw, hs);
  cudaGraph_t cap; CK(cudaStreamEndCapture(s, &cap));
  size_t nn = 0; CK(cudaGraphGetNodes(body, nullptr, &nn));
  cudaGraphNode_t ctln; CK(cudaGraphGetNodes(body, &ctln, &nn));
  cudaGraphNodeParams sp = {}; sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = hs; sp.conditional.type = cudaGraphCondTypeSwitch; sp.conditional.size = 2;
  cudaGraphNode_t sn; CK(cudaGraphAddNode(&sn, body, &ctln, 1, &sp));
  // case 0: cooperative kernel -> PDL kernel
  CK(cudaStreamBeginCaptureToGraph(s, sp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  {
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at; at.id = cudaLaunchAttributeCooperative; at.val.cooperative = 1;
    cfg.gridDim = 148; cfg.blockDim = 256; cfg.stream = s; cfg.attrs = &at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_coop, v, NWORK));
    cudaLaunchConfig_t cfg2 = {}; cudaLaunchAttribute a2; a2.id = cudaLaunchAttributeProgrammaticStreamSerialization; a2.val.programmaticStreamSerializationAllowed = 1;
    cfg2.gridDim = 592; cfg2.blockDim = 256; cfg2.stream = s; cfg2.attrs = &a2; cfg2.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg2, k_pdl, v, NWORK));
  }
  CK(cudaStreamEndCapture(s, &cap));
  CK(cudaStreamBeginCaptureToGraph(s, sp.conditional.phGraph_out[1], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  k_plain<<<1, 32, 0, s>>>(v);
  CK(cudaStreamEndCapture(s, &cap));
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
  for (int rep = 0; rep < 3; ++rep) {
    Ctl h{0, 1000, 0}; CK(cudaMemcpy(c, &h, sizeof h, cudaMemcpyHostToDevice));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); CK(cudaGraphLaunch(ex, s)); cudaEventRecord(b, s); CK(cudaStreamSynchronize(s));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double hv[2]; CK(cudaMemcpy(hv, v, sizeof hv, cudaMemcpyDeviceToHost));
    printf("1000 iterations: %.3f ms (%.2f us/iter), v0=%g v1=%g\n", ms, ms, hv[0], hv[1]);
  }
  // reference: the same work as separately launched small graphs from the host
  return 0;
}
