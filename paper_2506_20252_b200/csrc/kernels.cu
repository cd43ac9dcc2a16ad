// kernels.cu — dispatch and launch of the transport kernel (transport.cuh). The kernel
// templates are instantiated per dtype group in rs_*.cu so the build compiles in parallel.
#include "transport.cuh"

namespace pat {

using KernelFn = void (*)(const KPlan);

extern const KernelFn kRsRowI8[4], kRsRowU8[4], kRsRowI32[4], kRsRowU32[4], kRsRowI64[4], kRsRowU64[4],
    kRsRowF16[4], kRsRowF32[4], kRsRowF64[4], kRsRowBF16[4];

static const KernelFn* const kRsTable[10] = {kRsRowI8,  kRsRowU8,  kRsRowI32, kRsRowU32, kRsRowI64,
                                             kRsRowU64, kRsRowF16, kRsRowF32, kRsRowF64, kRsRowBF16};
static const KernelFn kAgKernel = pat_kernel<kU8, kSum, kAG>;

KernelFn kernel_for(int kind, int dtype, int op) {
  if (kind == kAG) return kAgKernel;
  return kRsTable[dtype][op];
}

cudaError_t max_blocks_per_sm(int kind, int dtype, int op, int threads, int* out) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel_for(kind, dtype, op), threads, 0);
}

bool pdl_enabled();  // local.cu

cudaError_t launch(const KPlan& plan, int dtype, int op, int threads, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.nlocal * plan.channels);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  // programmatic dependent launch: scheduled while the stream's previous kernel drains; the
  // kernel waits (griddepcontrol.wait) before touching memory. tools/launch_probe.cu: a
  // cooperative launch in a graph costs 0.99 us back to back, 0.68 us with this attribute.
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel_for(plan.kind, dtype, op), plan);
}

}  // namespace pat
