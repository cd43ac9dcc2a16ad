// ce_fold.cu — the SM half of the copy-engine executor (ce.cpp): element folds of staged
// arrivals, launched between the copy-engine transfers of a PAT round. Up to kMaxChunks
// independent folds per launch, dst = fold_left(src[0], ..., src[m-1]) with the reference's
// fold_one (simulate.cpp:31-39) generalised by fold.cuh; the caller orders the sources exactly
// as the executor folds them (arrivals in round order, own contribution last / first at the root).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ce.hpp"
#include "fold.cuh"

namespace pat {

__device__ __forceinline__ uint4 ce_ld16(const char* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <int DT, int OP>
__global__ void __launch_bounds__(512) ce_fold_kernel(const __grid_constant__ CeFold f) {
  const int pos = blockIdx.y;
  const CeFold::One& o = f.op[pos];
  if (f.vec == 16) {
    const int64_t nu = f.len >> 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < nu; u += stride) {
      uint4 a = ce_ld16(o.src[0] + 16 * u);
      for (int k = 1; k < o.m; ++k) fold_vec<DT, OP>(a, ce_ld16(o.src[k] + 16 * u));
      *reinterpret_cast<uint4*>(o.dst + 16 * u) = a;
    }
  } else {
    const int64_t ne = f.len / f.esize;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < ne; e += stride) {
      uint64_t a = ld_elem(o.src[0] + e * f.esize, f.esize);
      for (int k = 1; k < o.m; ++k) a = fold_elem_bits<DT, OP>(a, ld_elem(o.src[k] + e * f.esize, f.esize));
      st_elem(o.dst + e * f.esize, a, f.esize);
    }
  }
}

using CeFoldFn = void (*)(const CeFold);
#define PAT_CE_ROW(DT) \
  { ce_fold_kernel<DT, kSum>, ce_fold_kernel<DT, kProd>, ce_fold_kernel<DT, kMax>, ce_fold_kernel<DT, kMin> }
static const CeFoldFn kCeFold[10][4] = {
    PAT_CE_ROW(kI8), PAT_CE_ROW(kU8), PAT_CE_ROW(kI32), PAT_CE_ROW(kU32), PAT_CE_ROW(kI64),
    PAT_CE_ROW(kU64), PAT_CE_ROW(kF16), PAT_CE_ROW(kF32), PAT_CE_ROW(kF64), PAT_CE_ROW(kBF16)};

cudaError_t launch_ce_fold(const CeFold& f, int dtype, int op, int sm_count, cudaStream_t stream) {
  if (f.nop <= 0 || f.len <= 0) return cudaSuccess;
  const int64_t units = f.vec == 16 ? (f.len >> 4) : (f.len / f.esize);
  // HBM-bound; the SMs are otherwise idle while the copy engines move the data
  const int64_t want = (units + 511) / 512;
  const int gx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, std::max(1, sm_count / f.nop))));
  kCeFold[dtype][op]<<<dim3(gx, f.nop), 512, 0, stream>>>(f);
  return cudaGetLastError();
}

}  // namespace pat
