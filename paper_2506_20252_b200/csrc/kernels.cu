// kernels.cu — dispatch and launch of the transport kernel (transport.cuh). The kernel
// templates are instantiated per dtype group in rs_*.cu so the build compiles in parallel.
#include <cstdlib>

#include "transport.cuh"

namespace pat {

using KernelFn = void (*)(const KPlan);

extern const KernelFn kRsRowI8[4], kRsRowU8[4], kRsRowI32[4], kRsRowU32[4], kRsRowI64[4], kRsRowU64[4],
    kRsRowF16[4], kRsRowF32[4], kRsRowF64[4], kRsRowBF16[4];

static const KernelFn* const kRsTable[10] = {kRsRowI8,  kRsRowU8,  kRsRowI32, kRsRowU32, kRsRowI64,
                                             kRsRowU64, kRsRowF16, kRsRowF32, kRsRowF64, kRsRowBF16};
static const KernelFn kAgKernel = pat_kernel<kU8, kSum, kAG>;

using GroupFn = void (*)(const KPlan2);
extern const GroupFn kGroupI8, kGroupU8, kGroupI32, kGroupU32, kGroupI64, kGroupU64, kGroupF16, kGroupF32, kGroupF64,
    kGroupBF16;
static const GroupFn* const kGroupTable[10] = {&kGroupI8,  &kGroupU8,  &kGroupI32, &kGroupU32, &kGroupI64,
                                               &kGroupU64, &kGroupF16, &kGroupF32, &kGroupF64, &kGroupBF16};

KernelFn kernel_for(int kind, int dtype, int op) {
  if (kind == kAG) return kAgKernel;
  return kRsTable[dtype][op];
}

cudaError_t max_blocks_per_sm(int kind, int dtype, int op, int threads, int* out) {
  if (kind == 2)  // the grouped all-gather + reduce-scatter kernel
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, *kGroupTable[dtype], threads, 0);
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel_for(kind, dtype, op), threads, 0);
}

bool pdl_for(cudaStream_t stream);  // local.cu

// Pool state for a communicator whose step counters start at `start` instead of 0
// (PAT_ITER_START, tests of the 32-bit flag wrap): every done/credit flag = start, and the LL /
// LL32 lines stamped as epoch_clean leaves them (complete for value uint32(start + 1) - 2^30,
// zero data), which a zeroed pool equals for start = 0.
__global__ void init_pool_kernel(char* pool, int64_t ll_off, int64_t ll_bytes, int64_t ll32_off, int64_t ll32_bytes,
                                 uint64_t start) {
  const uint32_t V = static_cast<uint32_t>(start + 1) - 0x40000000u;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint64_t* flags = reinterpret_cast<uint64_t*>(pool);
  for (int64_t i = tid; i < int64_t{kMaxChannels} * kFlagWords; i += nthr) {
    const int w = static_cast<int>(i % kFlagWords);
    if (w >= 8 && w < 16) flags[i] = start;
  }
  uint4* ll = reinterpret_cast<uint4*>(pool + ll_off);
  for (int64_t i = tid; i < ll_bytes / 16; i += nthr) ll[i] = make_uint4(0, V, 0, V);
  uint4* l32 = reinterpret_cast<uint4*>(pool + ll32_off);
  for (int64_t i = tid; i < ll32_bytes / 16; i += nthr) l32[i] = (i & 1) ? make_uint4(0, 0, 0, V) : make_uint4(0, 0, 0, 0);
}

__global__ void fill_u64_kernel(uint64_t* p, int64_t n, uint64_t v) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

cudaError_t init_pool_state(char* pool, int64_t ll_off, int64_t ll_bytes, int64_t ll32_off, int64_t ll32_bytes,
                            uint64_t start, cudaStream_t stream) {
  init_pool_kernel<<<256, 256, 0, stream>>>(pool, ll_off, ll_bytes, ll32_off, ll32_bytes, start);
  return cudaGetLastError();
}

cudaError_t fill_u64(uint64_t* p, int64_t n, uint64_t v, cudaStream_t stream) {
  fill_u64_kernel<<<64, 256, 0, stream>>>(p, n, v);
  return cudaGetLastError();
}

// Device-side barrier over the ranks of a communicator (patCommBarrier): every local rank
// stores the call's sequence number into word `rank` of every peer's barrier words (release),
// then waits until every peer's word in its own pool reached it (acquire). One CTA per device.
__global__ void barrier_kernel(const __grid_constant__ BPlan b) {
  const int i = threadIdx.x;
  if (i >= b.nlocal * b.n) return;
  const int R = b.rank[i / b.n], q = i % b.n;
  if (q == R) return;
  if (b.gpu) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(b.bar[q] + R), "l"(b.seq) : "memory");
  else asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(b.bar[q] + R), "l"(b.seq) : "memory");
  Waiter w{b.timeout_ns, b.err, false, b.gpu != 0};
  wait_flag(b.bar[R] + q, b.seq, w);
}

cudaError_t launch_barrier(const BPlan& b, cudaStream_t stream) {
  barrier_kernel<<<1, 64, 0, stream>>>(b);
  return cudaGetLastError();
}

// Grouped all-gather (a) + reduce-scatter (b, sum, `dtype`) of one communicator in one launch.
cudaError_t launch_group(const KPlan2& plans, int dtype, int threads, cudaStream_t stream) {
  static const int force_coop = [] {
    const char* e = std::getenv("PAT_COOP");
    return e ? std::atoi(e) : -1;
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plans.a.nlocal * (plans.a.channels + plans.b.channels));
  cfg.blockDim = dim3(threads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = force_coop >= 0 ? (force_coop != 0) : (plans.a.nlocal > 1);
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_for(stream) ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, *kGroupTable[dtype], plans);
}

cudaError_t launch(const KPlan& plan, int dtype, int op, int threads, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.nlocal * plan.channels);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  // Cooperative launch (every CTA co-resident) is needed when several ranks share this grid:
  // their CTAs wait on each other. With one rank per device a CTA waits only on CTAs of other
  // devices, so a plain launch is safe and cheaper on the host (PAT_COOP=1 forces cooperative).
  static const int force_coop = [] {
    const char* e = std::getenv("PAT_COOP");
    return e ? std::atoi(e) : -1;
  }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = force_coop >= 0 ? (force_coop != 0) : (plan.nlocal > 1);
  // programmatic dependent launch: scheduled while the stream's previous kernel drains; the
  // kernel waits (griddepcontrol.wait) before touching memory. tools/launch_probe.cu: a
  // cooperative launch in a graph costs 0.99 us back to back, 0.68 us with this attribute.
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_for(stream) ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel_for(plan.kind, dtype, op), plan);
}

}  // namespace pat
