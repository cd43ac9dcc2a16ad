// bidir_probe.cu — NVLink ceilings under the traffic pattern of a collective: every GPU sends
// and receives at the same time. Not part of the product; it sets the roofline the PAT
// transport is judged against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bidir_probe.cu -o tools/bidir_probe -lcuda
//   tools/bidir_probe [ngpus]
//
// Patterns (G GPUs, one process, peer access, 1 GiB per GPU, all GPUs launched together):
//   ring-push  GPU i stores into GPU i+1      (every GPU sends 1 GiB and receives 1 GiB)
//   ring-pull  GPU i loads from GPU i-1
//   spread-push GPU i stores 1/(G-1) of its buffer into each peer
//   ce-ring    cudaMemcpyPeerAsync i -> i+1 (copy engines)
//   uni-push / uni-pull  only GPU 0 -> GPU 1 (the one-directional reference numbers)
#include <cuda.h>
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
__global__ void __launch_bounds__(512) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                   size_t n16) {
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

// Contiguous per-CTA ranges (the transport's slice layout) instead of a grid-stride.
template <int U>
__global__ void __launch_bounds__(512) copy_blocked(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                    size_t n16) {
  const size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const size_t beg = per * blockIdx.x, end = beg + per < n16 ? beg + per : n16;
  const size_t B = blockDim.x;
  size_t i = beg + threadIdx.x;
  for (; i + (U - 1) * B < end; i += U * B) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = src[i + k * B];
#pragma unroll
    for (int k = 0; k < U; ++k) dst[i + k * B] = v[k];
  }
  for (; i < end; i += B) dst[i] = src[i];
}

// A persistent kernel that occupies SMs while polling a local word (what the PAT kernel does
// while the copy engines move leaves): does it slow the copy engines down?
__global__ void __launch_bounds__(512) spin_kernel(const volatile uint64_t* flag, uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    (void)*flag;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int G = argc > 1 ? std::atoi(argv[1]) : ndev;
  if (G < 2 || G > ndev) {
    std::printf("need >= 2 GPUs (have %d)\n", ndev);
    return 0;
  }
  const size_t bytes = 1ull << 30, n16 = bytes / 16;
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
  }
  // run fn(d) on every active device, timed per device; returns GB/s received per GPU (min over GPUs)
  auto run = [&](const char* name, int active, auto fn, size_t per_gpu_bytes) {
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 = warm-up
      for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < active; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        for (int r = 0; r < 3; ++r) fn(d);
        CK(cudaEventRecord(e1[d], st[d]));
      }
      if (rep == 0) continue;
      double worst = 1e30;
      for (int d = 0; d < active; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        const double gbs = 3.0 * per_gpu_bytes / (ms / 1e3) / 1e9;
        worst = gbs < worst ? gbs : worst;
      }
      std::printf("%-34s G=%d: %7.1f GB/s per GPU per direction\n", name, active, worst);
      std::fflush(stdout);
    }
  };
  for (int grid : {128, 148, 296}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "uni-push grid %d", grid);
    run(nm, 1, [&](int d) { copy_kernel<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[0], (uint4*)dst[1], n16); }, bytes);
    std::snprintf(nm, sizeof nm, "uni-pull grid %d", grid);
    run(nm, 1, [&](int d) { copy_kernel<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[1], (uint4*)dst[0], n16); }, bytes);
    std::snprintf(nm, sizeof nm, "ring-push grid %d", grid);
    run(nm, G, [&](int d) {
      copy_kernel<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[d], (uint4*)dst[(d + 1) % G], n16);
    }, bytes);
    std::snprintf(nm, sizeof nm, "ring-push-blocked grid %d", grid);
    run(nm, G, [&](int d) {
      copy_blocked<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[d], (uint4*)dst[(d + 1) % G], n16);
    }, bytes);
    std::snprintf(nm, sizeof nm, "ring-pull grid %d", grid);
    run(nm, G, [&](int d) {
      copy_kernel<8><<<grid, 512, 0, st[d]>>>((const uint4*)src[(d + G - 1) % G], (uint4*)dst[d], n16);
    }, bytes);
    if (G > 2) {
      std::snprintf(nm, sizeof nm, "spread-push grid %d", grid);
      const size_t part = (n16 / (G - 1)) & ~size_t(15);
      run(nm, G, [&](int d) {
        for (int k = 1; k < G; ++k)
          copy_kernel<8><<<grid / (G - 1), 512, 0, st[d]>>>((const uint4*)src[d] + (k - 1) * part,
                                                            (uint4*)dst[(d + k) % G] + (k - 1) * part, part);
      }, part * 16 * (G - 1));
    }
  }
  for (int d = 0; d < G; ++d) {  // copy engines
    CK(cudaSetDevice(d));
  }
  // the copy-engine executor's shapes: 16 slices per call, cudaMemcpyAsync(Default) vs Peer,
  // on the legacy default stream vs a non-blocking stream
  const size_t sl = bytes / 16;
  run("ce-ring-16slices-peer", G, [&](int d) {
    for (int s = 0; s < 16; ++s)
      CK(cudaMemcpyPeerAsync(dst[(d + 1) % G] + s * sl, (d + 1) % G, src[d] + s * sl, d, sl, st[d]));
  }, bytes);
  run("ce-ring-16slices-default", G, [&](int d) {
    for (int s = 0; s < 16; ++s)
      CK(cudaMemcpyAsync(dst[(d + 1) % G] + s * sl, src[d] + s * sl, sl, cudaMemcpyDefault, st[d]));
  }, bytes);
  {
    std::vector<cudaEvent_t> ev(G * 16);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      for (int s = 0; s < 16; ++s) CK(cudaEventCreateWithFlags(&ev[d * 16 + s], cudaEventDisableTiming));
    }
    run("ce-ring-16slices-events", G, [&](int d) {
      for (int s = 0; s < 16; ++s) {
        CK(cudaMemcpyAsync(dst[(d + 1) % G] + s * sl, src[d] + s * sl, sl, cudaMemcpyDefault, st[d]));
        CK(cudaEventRecord(ev[d * 16 + s], st[d]));
        if (s > 0) CK(cudaStreamWaitEvent(st[d], ev[((d + G - 1) % G) * 16 + s - 1], 0));
      }
    }, bytes);
  }
  {  // the same dependency chain through stream memory operations on peer-mapped flags
    std::vector<uint32_t*> flag(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMalloc(&flag[d], 4096));
      CK(cudaMemset(flag[d], 0, 4096));
    }
    std::vector<uint32_t> calls(G, 0);
    run("ce-ring-16slices-streamvalue", G, [&](int d) {
      const uint32_t epoch = ++calls[d];  // the k-th call of every device pairs with its upstream's k-th
      for (int s = 0; s < 16; ++s) {
        CK(cudaMemcpyAsync(dst[(d + 1) % G] + s * sl, src[d] + s * sl, sl, cudaMemcpyDefault, st[d]));
        // tell the downstream GPU slice s landed; wait until my upstream's slice s-1 landed
        if (cuStreamWriteValue32(st[d], (CUdeviceptr)(flag[(d + 1) % G]), epoch * 16 + s + 1, 0) != CUDA_SUCCESS)
          std::printf("writevalue failed\n");
        if (s > 0 &&
            cuStreamWaitValue32(st[d], (CUdeviceptr)(flag[d]), epoch * 16 + s, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
          std::printf("waitvalue failed\n");
      }
    }, bytes);
  }
  {  // copy engines and SM stores sharing the same link: fraction f of every GPU's 1 GiB rides
     // the copy engine (second stream), the rest an SM push kernel, both started together
    std::vector<cudaStream_t> st2(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaStreamCreateWithFlags(&st2[d], cudaStreamNonBlocking));
    }
    std::vector<cudaEvent_t> fork(G), join(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventCreateWithFlags(&fork[d], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&join[d], cudaEventDisableTiming));
    }
    for (int pct : {25, 33, 50, 67}) {
      const size_t ce_bytes = (bytes * pct / 100) & ~size_t(4095);
      const size_t sm16 = (bytes - ce_bytes) / 16;
      char nm[64];
      std::snprintf(nm, sizeof nm, "mixed-ring ce %d%% + sm push", pct);
      run(nm, G, [&](int d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(fork[d], st[d]));
        CK(cudaStreamWaitEvent(st2[d], fork[d], 0));
        CK(cudaMemcpyPeerAsync(dst[(d + 1) % G], (d + 1) % G, src[d], d, ce_bytes, st2[d]));
        copy_kernel<8><<<148, 512, 0, st[d]>>>((const uint4*)(src[d] + ce_bytes), (uint4*)(dst[(d + 1) % G] + ce_bytes), sm16);
        CK(cudaEventRecord(join[d], st2[d]));
        CK(cudaStreamWaitEvent(st[d], join[d], 0));
      }, bytes);
    }
  }
  {
    std::vector<cudaStream_t> st3(G);
    std::vector<uint64_t*> word(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaStreamCreateWithFlags(&st3[d], cudaStreamNonBlocking));
      CK(cudaMalloc(&word[d], 64));
      CK(cudaMemset(word[d], 0, 64));
    }
    for (int ctas : {128, 148}) {
      char nm[64];
      std::snprintf(nm, sizeof nm, "ce-ring + spinning kernel %d CTAs", ctas);
      run(nm, G, [&](int d) {
        spin_kernel<<<ctas, 512, 0, st3[d]>>>(word[d], 1500000);  // 1.5 ms
        CK(cudaMemcpyPeerAsync(dst[(d + 1) % G], (d + 1) % G, src[d], d, bytes, st[d]));
      }, bytes);
    }
  }
  run("ce-uni", 1, [&](int d) { CK(cudaMemcpyPeerAsync(dst[1], 1, src[0], 0, bytes, st[d])); }, bytes);
  run("ce-ring", G, [&](int d) { CK(cudaMemcpyPeerAsync(dst[(d + 1) % G], (d + 1) % G, src[d], d, bytes, st[d])); },
      bytes);
  std::printf("done\n");
  return 0;
}
