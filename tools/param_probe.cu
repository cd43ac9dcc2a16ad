// param_probe.cu — device time per eager launch vs kernel parameter size (and PDL), back to back
// behind a spin so the host is never the bottleneck. nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/param_probe.cu -o tools/param_probe
#include <cuda_runtime.h>
#include <cstdio>
template <int B> struct Blob { char b[B]; };
template <int B>
__global__ void k(const __grid_constant__ Blob<B> p, int* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[B - 1] == 123) *out = 1;
}
__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
template <int B>
void run(cudaStream_t st, int* out, int grid, bool pdl, bool coop) {
  Blob<B> p{};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(grid);
  c.blockDim = dim3(512);
  c.stream = st;
  cudaLaunchAttribute a2[2];
  int na = 0;
  if (pdl) a2[na++] = attr[0];
  if (coop) a2[na++] = attr[1];
  c.attrs = a2;
  c.numAttrs = na;
  const int K = 2000;
  for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&c, k<B>, p, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStreamSynchronize(st);
  spin<<<1, 1, 0, st>>>(40000000);  // ~20 ms: every launch below is queued before it ends
  cudaEventRecord(e0, st);
  for (int i = 0; i < K; ++i) cudaLaunchKernelEx(&c, k<B>, p, out);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // graph of the same K launches
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
  for (int i = 0; i < K; ++i) cudaLaunchKernelEx(&c, k<B>, p, out);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float gms;
  cudaEventElapsedTime(&gms, e0, e1);
  // one single-kernel graph, launched K times (a per-call graph cache)
  cudaGraph_t g1;
  cudaGraphExec_t ge1;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
  cudaLaunchKernelEx(&c, k<B>, p, out);
  cudaStreamEndCapture(st, &g1);
  cudaGraphInstantiate(&ge1, g1, 0);
  cudaGraphLaunch(ge1, st);
  cudaStreamSynchronize(st);
  spin<<<1, 1, 0, st>>>(40000000);
  cudaEventRecord(e0, st);
  for (int i = 0; i < K; ++i) cudaGraphLaunch(ge1, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float g1ms;
  cudaEventElapsedTime(&g1ms, e0, e1);
  std::printf("{\"param_bytes\": %d, \"grid\": %d, \"pdl\": %d, \"coop\": %d, \"eager_us\": %.3f, \"graph_us\": %.3f, "
              "\"one_node_graph_launches_us\": %.3f}\n", B, grid, pdl, coop, 1e3 * ms / K, 1e3 * gms / K, 1e3 * g1ms / K);
}
int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 4);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int coop = 0; coop < 2; ++coop) {
      run<64>(st, out, 128, pdl, coop);
      run<1536>(st, out, 128, pdl, coop);
    }
  return 0;
}
