// capi_latency.cpp — eager latency of the C ABI from C++ (no Python on the call path): what a
// caller of the reference's C++ API sees after switching to patAllGather / patReduceScatter.
// Not part of the product.
//
//   g++ -O2 -std=c++17 tools/capi_latency.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_2506_20252_b200 -lpatb200 -L/usr/local/cuda/lib64 -lcudart \
//       -Wl,-rpath,$PWD/paper_2506_20252_b200 -o tools/capi_latency
//   tools/capi_latency [ngpus] [bytes_per_rank]
//
// One process drives n ranks on the first n GPUs (n = 1: 8 ranks on GPU 0, fused executor).
// Per collective: 20 warm-up calls, then K = 2000 eager calls back to back; reported: host
// microseconds per call (the C-ABI call's own cost) and device microseconds per call (events
// on every stream around the K calls, max over devices).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pat_b200.h"

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)
#define PK(x)                                                                                 \
  do {                                                                                        \
    patResult_t r = (x);                                                                      \
    if (r != patSuccess) {                                                                    \
      std::printf("PAT error %s at %s:%d\n", patGetErrorString(r), __FILE__, __LINE__);       \
      std::exit(1);                                                                           \
    }                                                                                         \
  } while (0)

int main(int argc, char** argv) {
  int ngpu = 0;
  CK(cudaGetDeviceCount(&ngpu));
  const int g = argc > 1 ? std::atoi(argv[1]) : ngpu;
  const size_t bytes = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 8;
  const int n = g == 1 ? 8 : g;
  std::vector<int> dev(n);
  for (int r = 0; r < n; ++r) dev[r] = g == 1 ? 0 : r;
  patComm_t comm;
  PK(patCommInitAll(&comm, n, dev.data(), nullptr));
  const size_t count = bytes / 4;
  std::vector<void*> ag_s(n), ag_r(n), rs_s(n), rs_r(n);
  std::vector<patStream_t> st(n);
  for (int r = 0; r < n; ++r) {
    CK(cudaSetDevice(dev[r]));
    CK(cudaMalloc(&ag_s[r], bytes));
    CK(cudaMalloc(&ag_r[r], n * bytes));
    CK(cudaMalloc(&rs_s[r], n * bytes));
    CK(cudaMalloc(&rs_r[r], bytes));
    CK(cudaMemset(ag_s[r], 1, bytes));
    CK(cudaMemset(rs_s[r], 1, n * bytes));
    cudaStream_t s;
    if (r == 0 || dev[r] != dev[r - 1]) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    else s = reinterpret_cast<cudaStream_t>(st[r - 1]);
    st[r] = reinterpret_cast<patStream_t>(s);
  }
  std::vector<int> devs;
  for (int r = 0; r < n; ++r)
    if (r == 0 || dev[r] != dev[r - 1]) devs.push_back(r);
  const int K = 2000;
  for (int coll = 0; coll < 2; ++coll) {
    auto call = [&]() {
      if (coll == 0) PK(patAllGather(comm, ag_s.data(), ag_r.data(), count, patFloat32, st.data()));
      else PK(patReduceScatter(comm, rs_s.data(), rs_r.data(), count, patFloat32, patSum, st.data()));
    };
    for (int i = 0; i < 20; ++i) call();
    for (int r : devs) {
      CK(cudaSetDevice(dev[r]));
      CK(cudaDeviceSynchronize());
    }
    std::vector<cudaEvent_t> e0(n), e1(n);
    for (int r : devs) {
      CK(cudaSetDevice(dev[r]));
      CK(cudaEventCreate(&e0[r]));
      CK(cudaEventCreate(&e1[r]));
      CK(cudaEventRecord(e0[r], reinterpret_cast<cudaStream_t>(st[r])));
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < K; ++i) call();
    const auto t1 = std::chrono::steady_clock::now();
    float worst = 0;
    for (int r : devs) {
      CK(cudaSetDevice(dev[r]));
      CK(cudaEventRecord(e1[r], reinterpret_cast<cudaStream_t>(st[r])));
      CK(cudaEventSynchronize(e1[r]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[r], e1[r]));
      worst = ms > worst ? ms : worst;
    }
    const double host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / K;
    std::printf("%s n=%d gpus=%d bytes/rank=%zu: host %.2f us/call, device %.2f us/call (eager, %d calls)\n",
                coll == 0 ? "allgather" : "reducescatter", n, (int)devs.size(), bytes, host_us, worst * 1e3 / K, K);
  }
  PK(patCommDestroy(comm));
  return 0;
}
