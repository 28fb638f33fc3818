// cond_node_bench.cu — cost of a CUDA-graph conditional IF node on B200
// (skip an untaken arm's GEMM with a conditional node).
// Per step inside one graph (R steps, CUDA events around the replay):
//   base      : producer kernel P (sets nothing)
//   cond-host : P + IF node (handle default 0, never set) with a body kernel
//   cond-dev0 : P sets the handle to 0 (cudaGraphSetConditional) + IF node
//   cond-dev1 : P sets the handle to 1 + IF node (body runs)
//   body      : P + body kernel unconditionally
//   exit      : P + a kernel that reads a flag and exits
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cond_node_bench tools/cond_node_bench.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void producer(float* x, int n, cudaGraphConditionalHandle h, int mode, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.5f + 1.f;
  if (i == 0) {
    if (mode == 1) cudaGraphSetConditional(h, 0);
    if (mode == 2) cudaGraphSetConditional(h, 1);
    if (flag) *flag = 0;
  }
}
__global__ void body(float* x, int n, const int* flag) {
  if (flag && *flag == 0) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 2.f - 1.f;
}

int main() {
  const int n = 1 << 20, R = 50;
  float* x; int* flag;
  CK(cudaMalloc(&x, n * 4)); CK(cudaMemset(x, 0, n * 4)); CK(cudaMalloc(&flag, 4));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto add_cond = [&](int mode) {
    cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
    producer<<<n / 256, 256, 0, s>>>(x, n, h, mode, nullptr);
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    body<<<n / 256, 256, 0, s2>>>(x, n, nullptr);
    CK(cudaStreamEndCapture(s2, &bodyg));
    CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  };
  auto timeit = [&](const char* name, auto&& fn) {
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    for (int r = 0; r < R; ++r) fn();
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    std::vector<float> ts;
    for (int t = 0; t < 9; ++t) {
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e0, s)); CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ts.push_back(ms * 1000.f / R);
    }
    std::sort(ts.begin(), ts.end());
    printf("%-12s %7.2f us/step\n", name, ts[ts.size() / 2]);
    CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
  };
  timeit("base", [&] { producer<<<n / 256, 256, 0, s>>>(x, n, 0, 0, nullptr); });
  timeit("body", [&] { producer<<<n / 256, 256, 0, s>>>(x, n, 0, 0, nullptr); body<<<n / 256, 256, 0, s>>>(x, n, nullptr); });
  timeit("exit", [&] { producer<<<n / 256, 256, 0, s>>>(x, n, 0, 0, flag); body<<<n / 256, 256, 0, s>>>(x, n, flag); });
  timeit("cond-host", [&] { add_cond(0); });
  timeit("cond-dev0", [&] { add_cond(1); });
  timeit("cond-dev1", [&] { add_cond(2); });
  return 0;
}
