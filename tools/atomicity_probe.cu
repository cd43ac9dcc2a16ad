// atomicity_probe.cu — does one vector store cross NVLink whole? Not part of the product; it
// decides how many flag words a polling line needs. The LL protocol puts a flag in every
// 8-byte half of its 16-byte line (50% payload); if a single 16-byte (or 32-byte) store always
// lands whole, one flag word per line is enough (75% / 87.5% payload). LL128's 128-byte lines,
// written by 8 lanes, tore but only ever between whole 16-byte lane pieces.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/atomicity_probe.cu -o tools/atomicity_probe
//   tools/atomicity_probe [ngpus] [iters]
//
// GPU pairs (0,1), (2,3) exchange: every thread stores LPT lines of W words into the peer
// (flag = call number in the last word, the other words a hash of (flag, line, word)), then
// polls its own incoming lines until the flag matches and checks the data words. Two buffers
// alternate by iteration parity. A line whose flag matched while a data word did not is a
// torn line; the probe counts them. Lines are 16 bytes (st.v4) or 32 bytes (st.v8).
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

__device__ __forceinline__ uint32_t h(uint32_t f, uint32_t line, uint32_t k) {
  uint32_t x = f * 0x9E3779B1u ^ line * 0x85EBCA77u ^ (k + 1) * 0xC2B2AE3Du;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  return x ^ (x >> 12);
}

template <int W>
__device__ __forceinline__ void st_line(uint32_t* p, const uint32_t* v) {
  if constexpr (W == 4)
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
                 : "memory");
  else
    asm volatile("st.volatile.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
template <int W>
__device__ __forceinline__ void ld_line(const uint32_t* p, uint32_t* v) {
  if constexpr (W == 4)
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "l"(p)
                 : "memory");
  else
    asm volatile("ld.volatile.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p)
                 : "memory");
}

// buffers: [2][grid*blockDim*LPT lines][W words]
template <int W, int LPT>
__global__ void __launch_bounds__(512) exchange(uint32_t* mine, uint32_t* peer, int iters, int first,
                                                unsigned long long* torn, unsigned long long* polls) {
  const uint32_t B = gridDim.x * blockDim.x;
  const uint32_t lines = B * LPT;
  unsigned long long bad = 0, spins = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t f = static_cast<uint32_t>(first + it);
    const size_t base = static_cast<size_t>(f & 1u) * lines * W;
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
      const uint32_t line = blockIdx.x * blockDim.x * LPT + k * blockDim.x + threadIdx.x;
      uint32_t v[W];
#pragma unroll
      for (int w = 0; w < W - 1; ++w) v[w] = h(f, line, w);
      v[W - 1] = f;
      st_line<W>(peer + base + static_cast<size_t>(line) * W, v);
    }
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
      const uint32_t line = blockIdx.x * blockDim.x * LPT + k * blockDim.x + threadIdx.x;
      uint32_t v[W];
      do {
        ld_line<W>(mine + base + static_cast<size_t>(line) * W, v);
        ++spins;
      } while (v[W - 1] != f);
#pragma unroll
      for (int w = 0; w < W - 1; ++w) bad += v[w] != h(f, line, w);
    }
  }
  atomicAdd(torn, bad);
  atomicAdd(polls, spins);
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int G = argc > 1 ? std::atoi(argv[1]) : ndev;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 2000;
  if (G < 2 || G > ndev || G % 2) {
    std::printf("need an even number >= 2 of GPUs (have %d)\n", ndev);
    return 0;
  }
  const int grid = 148 * 2, threads = 512;
  constexpr int LPT = 8;
  const size_t lines = static_cast<size_t>(grid) * threads * LPT;
  std::vector<uint32_t*> buf(G);
  std::vector<unsigned long long*> cnt(G);
  std::vector<cudaStream_t> st(G);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(d ^ 1, 0));
    CK(cudaMalloc(&buf[d], 2 * lines * 8 * 4));
    CK(cudaMemset(buf[d], 0, 2 * lines * 8 * 4));
    CK(cudaMalloc(&cnt[d], 16));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  auto run = [&](const char* name, auto launch) {
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(buf[d], 0, 2 * lines * 8 * 4));
      CK(cudaMemset(cnt[d], 0, 16));
      CK(cudaDeviceSynchronize());
    }
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      launch(d);
    }
    unsigned long long total = 0, polls = 0;
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaStreamSynchronize(st[d]));
      CK(cudaGetLastError());
      unsigned long long h2[2];
      CK(cudaMemcpy(h2, cnt[d], 16, cudaMemcpyDeviceToHost));
      total += h2[0];
      polls += h2[1];
    }
    std::printf("%-28s G=%d iters %d lines/iter/GPU %zu: torn data words %llu (polls %llu)\n", name, G, iters, lines,
                total, polls);
    std::fflush(stdout);
  };
  run("16-byte lines, 1 flag word", [&](int d) {
    exchange<4, LPT><<<grid, threads, 0, st[d]>>>(buf[d], buf[d ^ 1], iters, 1, cnt[d], cnt[d] + 1);
  });
  run("32-byte lines, 1 flag word", [&](int d) {
    exchange<8, LPT><<<grid, threads, 0, st[d]>>>(buf[d], buf[d ^ 1], iters, 1, cnt[d], cnt[d] + 1);
  });
  std::printf("done\n");
  return 0;
}
