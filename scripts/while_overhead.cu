// Microbenchmark: per-iteration cost of a CUDA-graph WHILE conditional node (the device-side loop
// of DESIGN §5) against the same kernels in a plain graph, and with the body unrolled U times.
// Body = U x [k_a (no-op, 148 x 192 threads), k_b (1 block: counts down, sets the condition)].
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/while_overhead scripts/while_overhead.cu -lcuda
// Prints one JSON line per variant: microseconds per kernel pair.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::printf("error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

__global__ void k_a(int* sink) {
  if (threadIdx.x == 0 && blockIdx.x == 100000) *sink = 1;
}
__global__ void k_b(int* cnt, cudaGraphConditionalHandle h, int use_h) {
  if (threadIdx.x == 0) {
    const int c = --cnt[0];
    if (use_h) cudaGraphSetConditional(h, c > 0 ? 1u : 0u);
  }
}
__global__ void k_set(int* cnt, int v) { cnt[0] = v; }

int main() {
  int *cnt, *sink;
  CK(cudaMalloc(&cnt, 4));
  CK(cudaMalloc(&sink, 4));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 2000;
  for (int U : {1, 2, 4}) {
    // WHILE graph
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wn;
    CK(cudaGraphAddNode(&wn, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    for (int u = 0; u < U; ++u) {
      k_a<<<148, 192, 0, st>>>(sink);
      k_b<<<1, 32, 0, st>>>(cnt, h, 1);
    }
    cudaGraph_t cap;
    CK(cudaStreamEndCapture(st, &cap));
    cudaGraphExec_t x;
    CK(cudaGraphInstantiate(&x, g, 0));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      k_set<<<1, 1, 0, st>>>(cnt, iters);
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(x, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    std::printf("{\"variant\": \"while\", \"unroll\": %d, \"pairs\": %d, \"us_per_pair\": %.3f}\n", U, iters,
                best * 1e3f / iters);
    CK(cudaGraphExecDestroy(x));
    CK(cudaGraphDestroy(g));
  }
  {  // plain graph of the same kernel pairs (no conditional)
    const int pairs = 1000;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    for (int u = 0; u < pairs; ++u) {
      k_a<<<148, 192, 0, st>>>(sink);
      k_b<<<1, 32, 0, st>>>(cnt, 0, 0);
    }
    CK(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t x;
    CK(cudaGraphInstantiate(&x, g, 0));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      k_set<<<1, 1, 0, st>>>(cnt, 1 << 30);
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(x, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    std::printf("{\"variant\": \"plain_graph\", \"unroll\": %d, \"pairs\": %d, \"us_per_pair\": %.3f}\n", pairs, pairs,
                best * 1e3f / pairs);
  }
  return 0;
}
