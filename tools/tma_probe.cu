// tma_probe.cu — can the tensor memory accelerator move more bytes over NVLink than SM
// stores? Not part of the product; it decides whether the SIMPLE transport should push (or pull)
// through bulk copies instead of 16-byte st.global (the SM store path caps
// pushing at ~704 GB/s while the link carries ~774 GB/s with the copy engines).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_probe.cu -o tools/tma_probe
//   tools/tma_probe [ngpus]
//
// Patterns (G GPUs, one process, peer access, 1 GiB per GPU, every GPU sends and receives):
//   v4-push      GPU i stores 16-byte vectors into GPU i+1 (the current transport)
//   v8-push      the same with 32-byte st.global.v8 (sm_100)
//   tma-push     bulk load local tile -> smem, bulk store smem -> peer (cp.async.bulk.global.shared::cta)
//   tma-pull     bulk load peer tile -> smem, bulk store smem -> local
//   mixed        a fraction of each GPU's bytes pushed by the sender, the rest pulled by the receiver
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

template <int U>
__global__ void __launch_bounds__(512) copy_v4(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t B = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * B < n16; i += U * B) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = src[i + k * B];
#pragma unroll
    for (int k = 0; k < U; ++k) dst[i + k * B] = v[k];
  }
}

struct V8 {
  uint32_t w[8];
};
__device__ __forceinline__ V8 ld32(const void* p) {
  V8 v;
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                 "=r"(v.w[7])
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st32(void* p, const V8& v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
               "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
               : "memory");
}

template <int U>
__global__ void __launch_bounds__(512) copy_v8(const char* __restrict__ src, char* __restrict__ dst, size_t n32) {
  size_t B = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * B < n32; i += U * B) {
    V8 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = ld32(src + 32 * (i + k * B));
#pragma unroll
    for (int k = 0; k < U; ++k) st32(dst + 32 * (i + k * B), v[k]);
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// One elected thread per CTA: NS stages of `piece` bytes; tile k of this CTA = blockIdx + k*grid.
__global__ void __launch_bounds__(32) copy_tma(const char* __restrict__ src, char* __restrict__ dst, size_t bytes,
                                               int piece, int NS) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[8];
  if (threadIdx.x != 0) return;
  const int64_t tiles = (bytes + piece - 1) / piece;
  const int64_t mine = tiles > blockIdx.x ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto load = [&](int64_t k) {
    const int64_t off = (blockIdx.x + k * gridDim.x) * (int64_t)piece;
    const int s = static_cast<int>(k % NS);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[s])), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(smem + (int64_t)s * piece)),
                 "l"(src + off), "r"(piece), "r"(sa(&bars[s]))
                 : "memory");
  };
  for (int64_t k = 0; k < mine && k < NS; ++k) load(k);
  uint32_t phase = 0;
  for (int64_t k = 0; k < mine; ++k) {
    const int s = static_cast<int>(k % NS);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                   : "=r"(done)
                   : "r"(sa(&bars[s])), "r"((phase >> s) & 1u)
                   : "memory");
    phase ^= 1u << s;
    const int64_t off = (blockIdx.x + k * gridDim.x) * (int64_t)piece;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(sa(smem + (int64_t)s * piece)), "r"(piece)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (k >= 1 && k - 1 + NS < mine) load(k - 1 + NS);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Push and pull sharing one link direction: blocks [0, gp) push bytes [0, split) of my source
// into my downstream peer; blocks [gp, grid) pull bytes [split, end) of my upstream's source.
__global__ void __launch_bounds__(512) mixed_push_pull(const uint4* __restrict__ mysrc, uint4* __restrict__ down_dst,
                                                       const uint4* __restrict__ up_src, uint4* __restrict__ mydst,
                                                       size_t split16, size_t n16, int gp) {
  const bool push = blockIdx.x < gp;
  const int nb = push ? gp : gridDim.x - gp;
  const int b = push ? blockIdx.x : blockIdx.x - gp;
  const uint4* src = push ? mysrc : up_src;
  uint4* dst = push ? down_dst : mydst;
  const size_t beg = push ? 0 : split16, end = push ? split16 : n16;
  constexpr int U = 8;
  const size_t B = (size_t)nb * blockDim.x;
  size_t i = beg + (size_t)b * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * B < end; i += U * B) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = src[i + k * B];
#pragma unroll
    for (int k = 0; k < U; ++k) dst[i + k * B] = v[k];
  }
  for (; i < end; i += B) dst[i] = src[i];
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int G = argc > 1 ? std::atoi(argv[1]) : ndev;
  if (G < 2 || G > ndev) {
    std::printf("need >= 2 GPUs (have %d)\n", ndev);
    return 0;
  }
  const size_t bytes = 1ull << 30;
  std::vector<char*> src(G), dst(G);
  std::vector<cudaStream_t> st(G);
  std::vector<cudaEvent_t> e0(G), e1(G);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < G; ++p)
      if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&src[d], bytes));
    CK(cudaMalloc(&dst[d], bytes));
    CK(cudaMemset(src[d], d + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    CK(cudaFuncSetAttribute(copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  auto run = [&](const char* name, auto fn) {
    for (int rep = 0; rep < 2; ++rep) {
      for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        for (int r = 0; r < 3; ++r) fn(d);
        CK(cudaEventRecord(e1[d], st[d]));
      }
      if (rep == 0) continue;
      double worst = 1e30;
      for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        const double gbs = 3.0 * bytes / (ms / 1e3) / 1e9;
        worst = gbs < worst ? gbs : worst;
      }
      std::printf("%-40s G=%d: %7.1f GB/s per GPU per direction\n", name, G, worst);
      std::fflush(stdout);
    }
  };
  char nm[96];
  for (int grid : {148, 296}) {
    std::snprintf(nm, sizeof nm, "v4-push grid %d", grid);
    run(nm, [&](int d) { copy_v4<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[d], (uint4*)dst[(d + 1) % G], bytes / 16); });
    std::snprintf(nm, sizeof nm, "v8-push grid %d", grid);
    run(nm, [&](int d) { copy_v8<4><<<grid, 512, 0, st[d]>>>(src[d], dst[(d + 1) % G], bytes / 32); });
    std::snprintf(nm, sizeof nm, "v4-pull grid %d", grid);
    run(nm, [&](int d) { copy_v4<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[(d + G - 1) % G], (uint4*)dst[d], bytes / 16); });
  }
  for (int pct : {40, 50, 60, 70}) {
    for (int grid : {148, 296}) {
      const int gp = grid * pct / 100;
      const size_t n16 = bytes / 16, split = (n16 * pct / 100) & ~size_t(255);
      std::snprintf(nm, sizeof nm, "mixed push %d%% pull rest grid %d", pct, grid);
      run(nm, [&](int d) {
        mixed_push_pull<<<grid, 512, 0, st[d]>>>((const uint4*)src[d], (uint4*)dst[(d + 1) % G],
                                                 (const uint4*)src[(d + G - 1) % G], (uint4*)dst[d], split, n16, gp);
      });
    }
  }
  for (int piece : {8192, 16384, 32768}) {
    for (int NS : {2, 4}) {
      const int sm = piece * NS;
      if (sm > 200 * 1024) continue;
      for (int cps : {1, 2, 4}) {
        if (sm * cps > 220 * 1024) continue;
        const int grid = 148 * cps;
        std::snprintf(nm, sizeof nm, "tma-push piece %d NS %d grid %d", piece, NS, grid);
        run(nm, [&](int d) { copy_tma<<<grid, 32, sm, st[d]>>>(src[d], dst[(d + 1) % G], bytes, piece, NS); });
        std::snprintf(nm, sizeof nm, "tma-pull piece %d NS %d grid %d", piece, NS, grid);
        run(nm, [&](int d) { copy_tma<<<grid, 32, sm, st[d]>>>(src[(d + G - 1) % G], dst[d], bytes, piece, NS); });
      }
    }
  }
  run("ce-ring", [&](int d) { CK(cudaMemcpyPeerAsync(dst[(d + 1) % G], (d + 1) % G, src[d], d, bytes, st[d])); });
  std::printf("done\n");
  return 0;
}
