// fold.cuh — element arithmetic shared by the transport (kernels.cu) and the fused
// single-device executor (local.cu): the reference's fold_one (simulate.cpp:31-39)
// generalised to the NCCL datatypes and ops. The left operand is the accumulator; integers
// wrap; fp16/bf16 are computed in fp32 and rounded to nearest even after every fold.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "plan.hpp"

namespace pat {

constexpr int kLocalMaxRanks = kMaxRanks;

template <int B>
__device__ __forceinline__ uint64_t ld_cg_bytes(const char* p) {
  if constexpr (B == 1) {
    unsigned short v;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
    return v & 0xff;
  } else if constexpr (B == 2) {
    unsigned short v;
    asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
    return v;
  } else if constexpr (B == 4) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
  } else {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
  }
}
__device__ __forceinline__ uint64_t ld_elem(const char* p, int esize) {
  switch (esize) {
    case 1: return ld_cg_bytes<1>(p);
    case 2: return ld_cg_bytes<2>(p);
    case 4: return ld_cg_bytes<4>(p);
    default: return ld_cg_bytes<8>(p);
  }
}
__device__ __forceinline__ void st_elem(char* p, uint64_t v, int esize) {
  switch (esize) {
    case 1: *reinterpret_cast<volatile uint8_t*>(p) = static_cast<uint8_t>(v); break;
    case 2: *reinterpret_cast<volatile uint16_t*>(p) = static_cast<uint16_t>(v); break;
    case 4: *reinterpret_cast<volatile uint32_t*>(p) = static_cast<uint32_t>(v); break;
    default: *reinterpret_cast<volatile uint64_t*>(p) = v; break;
  }
}

// ------------------------------------------------------------------------- element folds

enum : int { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };
enum : int { kI8 = 0, kU8 = 1, kI32 = 2, kU32 = 3, kI64 = 4, kU64 = 5, kF16 = 6, kF32 = 7, kF64 = 8, kBF16 = 9 };

template <int DT> struct DType;
template <> struct DType<kI8> { using S = int8_t; using U = uint8_t; static constexpr int cls = 0; };
template <> struct DType<kU8> { using S = uint8_t; using U = uint8_t; static constexpr int cls = 0; };
template <> struct DType<kI32> { using S = int32_t; using U = uint32_t; static constexpr int cls = 0; };
template <> struct DType<kU32> { using S = uint32_t; using U = uint32_t; static constexpr int cls = 0; };
template <> struct DType<kI64> { using S = int64_t; using U = uint64_t; static constexpr int cls = 0; };
template <> struct DType<kU64> { using S = uint64_t; using U = uint64_t; static constexpr int cls = 0; };
template <> struct DType<kF32> { using S = float; using U = float; static constexpr int cls = 1; };
template <> struct DType<kF64> { using S = double; using U = double; static constexpr int cls = 1; };
template <> struct DType<kF16> { using S = uint16_t; using U = uint16_t; static constexpr int cls = 2; };
template <> struct DType<kBF16> { using S = uint16_t; using U = uint16_t; static constexpr int cls = 3; };

template <int OP, typename T>
__device__ __forceinline__ T apply(T x, T y) {
  if constexpr (OP == kSum) return x + y;
  else if constexpr (OP == kProd) return x * y;
  else if constexpr (OP == kMax) return y > x ? y : x;
  else return y < x ? y : x;
}

// a = a (op) b; `a` is the accumulator (left operand), as fold_one in simulate.cpp:31-39.
template <int DT, int OP>
__device__ __forceinline__ typename DType<DT>::S fold1(typename DType<DT>::S a, typename DType<DT>::S b) {
  using D = DType<DT>;
  using S = typename D::S;
  using U = typename D::U;
  if constexpr (D::cls == 0) {
    if constexpr (OP == kSum) return static_cast<S>(static_cast<U>(a) + static_cast<U>(b));
    else if constexpr (OP == kProd) return static_cast<S>(static_cast<U>(a) * static_cast<U>(b));
    else return apply<OP>(a, b);
  } else if constexpr (D::cls == 1) {
    return apply<OP>(a, b);
  } else if constexpr (D::cls == 2) {
    const float r = apply<OP>(__half2float(__ushort_as_half(a)), __half2float(__ushort_as_half(b)));
    return __half_as_ushort(__float2half_rn(r));
  } else {
    const float r = apply<OP>(__bfloat162float(__ushort_as_bfloat16(a)), __bfloat162float(__ushort_as_bfloat16(b)));
    return __bfloat16_as_ushort(__float2bfloat16_rn(r));
  }
}

template <int DT, int OP, typename V>
__device__ __forceinline__ void fold_vec(V& a, const V& b) {
  using S = typename DType<DT>::S;
  constexpr int N = sizeof(V) / sizeof(S);
  union U {
    V v;
    S e[N];
  } x, y;
  x.v = a;
  y.v = b;
#pragma unroll
  for (int i = 0; i < N; ++i) x.e[i] = fold1<DT, OP>(x.e[i], y.e[i]);
  a = x.v;
}

template <int DT, int OP>
__device__ __forceinline__ uint64_t fold_elem_bits(uint64_t a, uint64_t b) {
  using S = typename DType<DT>::S;
  S x, y;
  memcpy(&x, &a, sizeof(S));
  memcpy(&y, &b, sizeof(S));
  x = fold1<DT, OP>(x, y);
  uint64_t r = 0;
  memcpy(&r, &x, sizeof(S));
  return r;
}

// Scalar form of the fused PAT reduction tree (see local.cu), element-granular path.
template <int DT, int OP, int N>
__device__ __forceinline__ typename DType<DT>::S tree_scalar(const typename DType<DT>::S* x) {
  auto f = [](typename DType<DT>::S a, typename DType<DT>::S b) { return fold1<DT, OP>(a, b); };
  if constexpr (N == 1) return x[0];
  else if constexpr (N == 2) return f(x[0], x[1]);
  else if constexpr (N == 3) return f(f(x[0], x[1]), x[2]);
  else if constexpr (N == 4) return f(f(x[0], x[1]), f(x[3], x[2]));
  else if constexpr (N == 5) return f(f(f(x[0], x[1]), f(x[3], x[2])), x[4]);
  else if constexpr (N == 6) return f(f(f(x[0], x[1]), f(x[3], x[2])), f(x[5], x[4]));
  else if constexpr (N == 7) return f(f(f(x[0], x[1]), f(x[3], x[2])), f(f(x[5], x[6]), x[4]));
  else return f(f(f(x[0], x[1]), f(x[3], x[2])), f(f(x[5], f(x[7], x[6])), x[4]));
}

}  // namespace pat
