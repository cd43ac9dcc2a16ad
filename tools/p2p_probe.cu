// p2p_probe.cu — microbenchmarks of the NVLink transport primitives the PAT kernels are
// built from (2 GPUs, one process, peer access). Not part of the product; the numbers it
// prints drive the kernel design.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/p2p_probe.cu -o tools/p2p_probe
//
// 1. push (LDG local -> STG peer), grid x unroll sweep
// 2. pull (LDG peer -> STG local)
// 3. TMA push (cp.async.bulk global->shared, shared->global peer), 1 issuing thread per CTA
// 4. flag ping-pong latency (st.release.sys / ld.acquire.sys)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t B = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * B < n16; i += U * B) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = src[i + k * B];
#pragma unroll
    for (int k = 0; k < U; ++k) dst[i + k * B] = v[k];
  }
  for (; i < n16; i += B) dst[i] = src[i];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Each CTA copies a contiguous range in pieces of `piece` bytes through NS smem stages.
__global__ void tma_copy_kernel(const char* src, char* dst, size_t bytes, int piece, int NS) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x != 0) return;
  const size_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
  const size_t beg = per * blockIdx.x < bytes ? per * blockIdx.x : bytes, end = beg + per < bytes ? beg + per : bytes;
  for (int s = 0; s < NS; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t npieces = (end - beg + piece - 1) / piece;
  uint32_t phase[16] = {0};
  // prologue: issue up to NS loads
  auto issue_load = [&](size_t k) {
    const int s = k % NS;
    const size_t off = beg + k * piece;
    const uint32_t len = (uint32_t)((end - off) < (size_t)piece ? (end - off) : piece);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(len)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (size_t)s * piece)),
        "l"(src + off), "r"(len), "r"(smem_u32(&bars[s]))
        : "memory");
  };
  for (size_t k = 0; k < npieces && k < (size_t)NS; ++k) issue_load(k);
  for (size_t k = 0; k < npieces; ++k) {
    const int s = k % NS;
    // wait for load k
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bars[s])), "r"(phase[s])
          : "memory");
    }
    phase[s] ^= 1;
    const size_t off = beg + k * piece;
    const uint32_t len = (uint32_t)((end - off) < (size_t)piece ? (end - off) : piece);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(smem_u32(smem + (size_t)s * piece)), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (k + NS < npieces) {
      // stage s is re-filled once its store has read smem
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue_load(k + NS);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA variant with store look-ahead: allow NS-1 stores in flight before reusing a stage.
__global__ void tma_copy_kernel2(const char* src, char* dst, size_t bytes, int piece, int NS) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x != 0) return;
  const size_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
  const size_t beg = per * blockIdx.x < bytes ? per * blockIdx.x : bytes, end = beg + per < bytes ? beg + per : bytes;
  for (int s = 0; s < NS; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t npieces = (end - beg + piece - 1) / piece;
  uint32_t phase[16] = {0};
  for (size_t k = 0; k < npieces; ++k) {
    const int s = k % NS;
    const size_t off = beg + k * piece;
    const uint32_t len = (uint32_t)((end - off) < (size_t)piece ? (end - off) : piece);
    if (k >= (size_t)NS) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(len)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (size_t)s * piece)),
        "l"(src + off), "r"(len), "r"(smem_u32(&bars[s]))
        : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bars[s])), "r"(phase[s])
          : "memory");
    }
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(smem_u32(smem + (size_t)s * piece)), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void pingpong(uint64_t* mine, uint64_t* peer, int iters, int leader, unsigned long long* out_ns) {
  if (threadIdx.x != 0) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (leader) {
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer), "l"((uint64_t)i) : "memory");
      uint64_t v = 0;
      do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v < (uint64_t)i);
    } else {
      uint64_t v = 0;
      do { asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v < (uint64_t)i);
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer), "l"((uint64_t)i) : "memory");
    }
  }
  uint64_t t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (leader) *out_ns = t1 - t0;
}

__global__ void empty_kernel() {}

int main(int argc, char** argv) {
  const bool lat_only = argc > 1;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::printf("need 2 GPUs\n");
    return 0;
  }
  const size_t bytes = 1ull << 30;
  char *a0, *b1, *a1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMemset(a1, 2, bytes));
  CK(cudaSetDevice(0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto fn, int reps) {
    fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
  };
  const size_t n16 = bytes / 16;
  if (!lat_only) {
  std::printf("== push LDG local -> STG peer (GB/s, 1 GiB)\n");
  for (int threads : {256, 512, 1024}) {
    for (int grid : {16, 32, 64, 128, 148, 296}) {
      float ms = timeit([&] { copy_kernel<8><<<grid, threads>>>((const uint4*)a0, (uint4*)b1, n16); }, 5);
      std::printf("push grid %4d thr %4d U8: %7.1f\n", grid, threads, bytes / ms / 1e6);
    }
  }
  for (int grid : {32, 64, 148}) {
    float ms = timeit([&] { copy_kernel<4><<<grid, 512>>>((const uint4*)a0, (uint4*)b1, n16); }, 5);
    std::printf("push grid %4d thr 512 U4: %7.1f\n", grid, bytes / ms / 1e6);
    ms = timeit([&] { copy_kernel<16><<<grid, 512>>>((const uint4*)a0, (uint4*)b1, n16); }, 5);
    std::printf("push grid %4d thr 512 U16: %7.1f\n", grid, bytes / ms / 1e6);
  }
  std::printf("== pull LDG peer -> STG local\n");
  for (int grid : {32, 64, 148, 296}) {
    float ms = timeit([&] { copy_kernel<8><<<grid, 512>>>((const uint4*)a1, (uint4*)a0, n16); }, 5);
    std::printf("pull grid %4d thr 512 U8: %7.1f\n", grid, bytes / ms / 1e6);
  }
  std::printf("== local copy (HBM)\n");
  for (int grid : {148, 296, 592}) {
    char* c0;
    CK(cudaMalloc(&c0, bytes));
    float ms = timeit([&] { copy_kernel<8><<<grid, 512>>>((const uint4*)a0, (uint4*)c0, n16); }, 5);
    std::printf("local grid %4d: %7.1f GB/s (read+write %7.1f)\n", grid, bytes / ms / 1e6, 2 * bytes / ms / 1e6);
    CK(cudaFree(c0));
  }
  std::printf("== TMA push (1 thread/CTA): load G->S, store S->G(peer)\n");
  for (int piece : {16384, 32768, 65536}) {
    for (int NS : {2, 4, 6}) {
      const int smem = piece * NS;
      if (smem > 200 * 1024) continue;
      CK(cudaFuncSetAttribute(tma_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      CK(cudaFuncSetAttribute(tma_copy_kernel2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      for (int grid : {16, 32, 64, 128, 148}) {
        float ms = timeit([&] { tma_copy_kernel<<<grid, 32, smem>>>(a0, b1, bytes, piece, NS); }, 5);
        float ms2 = timeit([&] { tma_copy_kernel2<<<grid, 32, smem>>>(a0, b1, bytes, piece, NS); }, 5);
        std::printf("tma piece %6d NS %d grid %4d: %7.1f  (v2 %7.1f)\n", piece, NS, grid, bytes / ms / 1e6,
                    bytes / ms2 / 1e6);
      }
    }
  }
  std::printf("== TMA local copy\n");
  {
    char* c0;
    CK(cudaMalloc(&c0, bytes));
    CK(cudaFuncSetAttribute(tma_copy_kernel2, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
    for (int grid : {74, 148, 296}) {
      float ms = timeit([&] { tma_copy_kernel2<<<grid, 32, 4 * 32768>>>(a0, c0, bytes, 32768, 4); }, 5);
      std::printf("tma local grid %4d: %7.1f GB/s\n", grid, bytes / ms / 1e6);
    }
    CK(cudaFree(c0));
  }
  }
  std::printf("== flag ping-pong (st.release.sys / ld.acquire.sys)\n");
  {
    uint64_t *f0, *f1;
    unsigned long long* out;
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&f0, 64));
    CK(cudaMemset(f0, 0, 64));
    CK(cudaMallocHost(&out, 8));
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&f1, 64));
    CK(cudaMemset(f1, 0, 64));
    const int iters = 10000;
    CK(cudaSetDevice(1));
    pingpong<<<1, 32>>>(f1, f0, iters, 0, out);
    CK(cudaSetDevice(0));
    pingpong<<<1, 32>>>(f0, f1, iters, 1, out);
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(1));
    CK(cudaDeviceSynchronize());
    std::printf("round trip %.3f us (one-way ~%.3f us)\n", *out / 1e3 / iters, *out / 2e3 / iters);
  }
  std::printf("== empty kernel launch (back-to-back, normal vs cooperative)\n");
  {
    CK(cudaSetDevice(0));
    float ms = timeit([&] { empty_kernel<<<1, 32>>>(); }, 1000);
    std::printf("empty launch: %.2f us\n", ms * 1e3);
    void* args[1] = {nullptr};
    ms = timeit([&] { CK(cudaLaunchCooperativeKernel((void*)empty_kernel, dim3(1), dim3(32), args, 0, 0)); }, 1000);
    std::printf("empty cooperative launch: %.2f us\n", ms * 1e3);
    ms = timeit([&] { CK(cudaLaunchCooperativeKernel((void*)empty_kernel, dim3(128), dim3(512), args, 0, 0)); }, 1000);
    std::printf("empty cooperative launch 128x512: %.2f us\n", ms * 1e3);
  }
  std::printf("done\n");
  return 0;
}
