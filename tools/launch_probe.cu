// launch_probe.cu — what does a back-to-back collective call cost before any data moves?
// Not part of the product; it decides whether programmatic dependent launch (PDL) is worth
// adding to the transport kernel's launch (fixed cost a = 3.6 us per LL call).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/launch_probe.cu -o tools/launch_probe
//   tools/launch_probe
//
// 1. Graph of K empty kernels (1 x 512), per-kernel time: normal, cooperative, PDL, coop+PDL.
// 3. In-kernel ping-pong of one polled line, 16-byte (LL) vs 32-byte (LL32) lines.
// 2. Exchange: 2 GPUs, each kernel stores one 16-byte LL line {data, flag, data, flag} into the
//    peer and polls its own line for the peer's (the 1-round LL step with no payload), K
//    kernels per graph on each GPU, graphs launched together: per-exchange time, same variants.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

__global__ void empty_kernel(int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// counter[0] (local) = calls so far; flag of call k = k + 1
__global__ void exchange_kernel(uint32_t* counter, uint4* mine, uint4* peer, int pdl, int trigger) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t f = *counter + 1;
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(peer), "r"(f), "r"(f), "r"(f), "r"(f)
                 : "memory");
    uint4 v;
    do {
      asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(mine)
                   : "memory");
    } while (v.y != f || v.w != f);
    *counter = f;
  }
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


// In-kernel ping-pong of one polled line: 16-byte LL line (flag in words 1 and 3) vs 32-byte
// LL32 line (flag in word 7). Leader stores, waits for the echo; returns ns per round trip.
template <int W>
__global__ void line_pingpong(uint32_t* mine, uint32_t* peer, int iters, int leader, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    const uint32_t f = static_cast<uint32_t>(i);
    if (!leader) {  // wait first
      if constexpr (W == 4) {
        uint4 v;
        do asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mine) : "memory");
        while (v.y != f || v.w != f);
      } else {
        uint32_t w[8];
        do asm volatile("ld.volatile.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "l"(mine) : "memory");
        while (w[7] != f);
      }
    }
    if constexpr (W == 4)
      asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(peer), "r"(f), "r"(f), "r"(f), "r"(f) : "memory");
    else
      asm volatile("st.volatile.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(peer), "r"(f), "r"(f), "r"(f), "r"(f), "r"(f), "r"(f), "r"(f), "r"(f) : "memory");
    if (leader) {
      if constexpr (W == 4) {
        uint4 v;
        do asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mine) : "memory");
        while (v.y != f || v.w != f);
      } else {
        uint32_t w[8];
        do asm volatile("ld.volatile.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "l"(mine) : "memory");
        while (w[7] != f);
      }
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (leader) *out = (t1 - t0) / iters;
}

static void launch(void (*k)(int), int pdl, int coop, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(512);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  CK(cudaLaunchKernelEx(&cfg, k, pdl));
}

static void launch_x(uint32_t* c, uint4* m, uint4* p, int pdl, int coop, int trig, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(512);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  CK(cudaLaunchKernelEx(&cfg, exchange_kernel, c, m, p, pdl, trig));
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int K = 200;
  cudaStream_t st[2];
  for (int d = 0; d < (ndev >= 2 ? 2 : 1); ++d) {
    CK(cudaSetDevice(d));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  CK(cudaSetDevice(0));
  std::printf("== graph of %d empty kernels, per kernel (us)\n", K);
  for (int coop : {0, 1})
    for (int pdl : {0, 1}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(st[0], cudaStreamCaptureModeGlobal));
      for (int i = 0; i < K; ++i) launch(empty_kernel, pdl, coop, st[0]);
      CK(cudaStreamEndCapture(st[0], &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(a, st[0]));
        CK(cudaGraphLaunch(ge, st[0]));
        CK(cudaEventRecord(b, st[0]));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep && ms < best) best = ms;
      }
      std::printf("coop %d pdl %d: %.3f us\n", coop, pdl, best * 1e3 / K);
    }
  if (ndev < 2) return 0;
  std::printf("== 2-GPU LL exchange, graph of %d kernels per GPU, per exchange (us)\n", K);
  uint32_t* cnt[2];
  uint4* line[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&cnt[d], 64));
    CK(cudaMalloc(&line[d], 64));
  }
  for (int coop : {0, 1})
    for (int pdl : {0, 1})
      for (int trig : {0, 1}) {
        if (trig && !pdl) continue;
        cudaGraphExec_t ge[2];
        for (int d = 0; d < 2; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaMemset(cnt[d], 0, 64));
          CK(cudaMemset(line[d], 0, 64));
          CK(cudaDeviceSynchronize());
          cudaGraph_t g;
          CK(cudaStreamBeginCapture(st[d], cudaStreamCaptureModeGlobal));
          for (int i = 0; i < K; ++i) launch_x(cnt[d], line[d], line[1 - d], pdl, coop, trig, st[d]);
          CK(cudaStreamEndCapture(st[d], &g));
          CK(cudaGraphInstantiate(&ge[d], g, 0));
        }
        cudaEvent_t a[2], b[2];
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            if (rep == 0) {
              CK(cudaEventCreate(&a[d]));
              CK(cudaEventCreate(&b[d]));
            }
            CK(cudaEventRecord(a[d], st[d]));
            CK(cudaGraphLaunch(ge[d], st[d]));
            CK(cudaEventRecord(b[d], st[d]));
          }
          float worst = 0;
          for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventSynchronize(b[d]));
            float ms;
            CK(cudaEventElapsedTime(&ms, a[d], b[d]));
            worst = ms > worst ? ms : worst;
          }
          if (rep && worst < best) best = worst;
        }
        std::printf("coop %d pdl %d trigger %d: %.3f us\n", coop, pdl, trig, best * 1e3 / K);
      }
  {
    unsigned long long* out;
    CK(cudaMallocManaged(&out, 8));
    for (int W : {4, 8}) {
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMemset(line[d], 0, 64));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 1; d >= 0; --d) {
        CK(cudaSetDevice(d));
        if (W == 4) line_pingpong<4><<<1, 32, 0, st[d]>>>((uint32_t*)line[d], (uint32_t*)line[1 - d], 10000, d == 0, out);
        else line_pingpong<8><<<1, 32, 0, st[d]>>>((uint32_t*)line[d], (uint32_t*)line[1 - d], 10000, d == 0, out);
      }
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      std::printf("line ping-pong %d-byte line: round trip %.3f us\n", W * 4, *out / 1e3);
    }
  }
  std::printf("done\n");
  return 0;
}
