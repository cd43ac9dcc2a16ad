// local.cu — fused single-device executor: every rank of the communicator lives in this
// GPU's HBM ("local mode", the reference's in-process ranks, simulate.cpp:157-165).
//
// With all ranks' buffers in one HBM the per-round messages of the PAT schedule are pure
// overhead: the result is fixed by the schedule alone. All-gather output is the
// concatenation of the inputs (oracle.cpp:15-24). Reduce-scatter output r is the PAT fold
// tree over x_j = contribution of rank (r + j) mod n, with the executor's operand order
// (accumulator left): the host symbolically executes the compiled schedule (comm.cpp,
// symbolic_reduce_scatter) and only takes this path when the result equals the tree
// compiled in here (T-independent for PAT):
//   n=2  x0+x1
//   n=3  (x0+x1)+x2
//   n=4  (x0+x1)+(x3+x2)
//   n=5  ((x0+x1)+(x3+x2))+x4
//   n=6  ((x0+x1)+(x3+x2))+(x5+x4)
//   n=7  ((x0+x1)+(x3+x2))+((x5+x6)+x4)
//   n=8  ((x0+x1)+(x3+x2))+((x5+(x7+x6))+x4)
// So each kernel reads every input byte once and writes every output byte once: the HBM
// roofline of the collective (n*C read + n^2*C written for AG, n^2*C read + n*C written for RS).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include <algorithm>
#include <cstdlib>

#include "fold.cuh"

namespace pat {

struct LPlan {
  int n, kind, vec, esize;
  int64_t chunk_bytes;
  const char* send[kLocalMaxRanks];  // by rank
  char* recv[kLocalMaxRanks];        // by rank
};

// Programmatic dependent launch (launch_local): wait for the stream's previous kernel before
// touching memory. The successor is released only at exit (no early launch_dependents): these
// grids run in more than one wave, and an early-resident successor would take their registers.
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint4 ld_nc16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs16(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int DT, int OP, int N, typename V>
__device__ __forceinline__ V tree(const V* x) {
  auto f = [](V a, const V& b) {
    fold_vec<DT, OP>(a, b);
    return a;
  };
  if constexpr (N == 1) return x[0];
  else if constexpr (N == 2) return f(x[0], x[1]);
  else if constexpr (N == 3) return f(f(x[0], x[1]), x[2]);
  else if constexpr (N == 4) return f(f(x[0], x[1]), f(x[3], x[2]));
  else if constexpr (N == 5) return f(f(f(x[0], x[1]), f(x[3], x[2])), x[4]);
  else if constexpr (N == 6) return f(f(f(x[0], x[1]), f(x[3], x[2])), f(x[5], x[4]));
  else if constexpr (N == 7) return f(f(f(x[0], x[1]), f(x[3], x[2])), f(f(x[5], x[6]), x[4]));
  else return f(f(f(x[0], x[1]), f(x[3], x[2])), f(f(x[5], f(x[7], x[6])), x[4]));
}

// Grid: n groups of `bpr` blocks; group o (all-gather: origin, reduce-scatter: output rank)
// walks its chunk in 16-byte units with U loads in flight per thread before any store.
constexpr int kLocalThreads = 512;
constexpr int kU = 4;

// All-gather: unit u of origin o is read once and written to all n outputs.
__global__ void __launch_bounds__(kLocalThreads, 2) local_ag_kernel(const __grid_constant__ LPlan p) {
  pdl_enter();
  const int n = p.n;
  const int bpr = gridDim.x / n;
  const int o = blockIdx.x / bpr;
  const int b = blockIdx.x - o * bpr;
  const int64_t Cb = p.chunk_bytes;
  const char* src = p.send[o];
  const int skip = (p.recv[o] + o * Cb == src) ? o : -1;  // in place: rank o's own block is there
  if (p.vec == 16) {
    const int64_t nu = Cb >> 4;
    const int64_t step = static_cast<int64_t>(bpr) * blockDim.x;
    int64_t u = static_cast<int64_t>(b) * blockDim.x + threadIdx.x;
    for (; u + (kU - 1) * step < nu; u += kU * step) {
      uint4 v[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) v[k] = ld_nc16(src + 16 * (u + k * step));
      for (int r = 0; r < n; ++r) {
        if (r == skip) continue;
        char* dst = p.recv[r] + o * Cb + 16 * u;
#pragma unroll
        for (int k = 0; k < kU; ++k) st_cs16(dst + 16 * k * step, v[k]);
      }
    }
    for (; u < nu; u += step) {
      const uint4 v = ld_nc16(src + 16 * u);
      for (int r = 0; r < n; ++r)
        if (r != skip) st_cs16(p.recv[r] + o * Cb + 16 * u, v);
    }
  } else {
    const int es = p.esize;
    const int64_t ne = Cb / es;
    for (int64_t e = static_cast<int64_t>(b) * blockDim.x + threadIdx.x; e < ne;
         e += static_cast<int64_t>(bpr) * blockDim.x) {
      const uint64_t v = ld_elem(src + e * es, es);
      for (int r = 0; r < n; ++r)
        if (r != skip) st_elem(p.recv[r] + o * Cb + e * es, v, es);
    }
  }
}

// All-gather, 32-byte units, one wave: global unit g in [0, n * Cb/32) is unit g % nu of origin
// g / nu; each thread loads kAgU units (256-bit loads) before storing each to the n outputs
// (256-bit stores). The broadcast writes n^2 C and reads n C, so it is bound by HBM write
// bandwidth: tools/local_tune.cu measured 12.5 us at n = 8, 1 MiB against 12.2 us for a
// write-only kernel of the same byte count (the bulk-copy kernel below: 13.0 us).
struct V8 {
  uint32_t w[8];
};
__device__ __forceinline__ V8 ld_nc32(const void* p) {
  V8 v;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                 "=r"(v.w[7])
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st32(void* p, const V8& v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
               "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
               : "memory");
}
constexpr int kFlatThreads = 256;  // flat kernels: 4 CTAs of 256 threads per SM, one wave
constexpr int kFlatCtasPerSm = 4;
constexpr int kAgU = 2;

__device__ __forceinline__ void local_ag32_body(const LPlan& p, int blk, int nblk) {
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const int64_t nu = Cb >> 5;
  const int64_t total = n * nu;
  const int64_t TT = static_cast<int64_t>(nblk) * kFlatThreads;
  for (int64_t g = static_cast<int64_t>(blk) * kFlatThreads + threadIdx.x; g < total; g += kAgU * TT) {
    V8 v[kAgU];
    int o[kAgU];
    int64_t u[kAgU];
#pragma unroll
    for (int k = 0; k < kAgU; ++k) {
      const int64_t gg = g + k * TT;
      o[k] = gg < total ? static_cast<int>(gg / nu) : -1;
      u[k] = gg - static_cast<int64_t>(o[k]) * nu;
      if (o[k] >= 0) v[k] = ld_nc32(p.send[o[k]] + 32 * u[k]);
    }
    for (int r = 0; r < n; ++r)
#pragma unroll
      for (int k = 0; k < kAgU; ++k) {
        if (o[k] < 0) continue;
        char* dst = p.recv[r] + o[k] * Cb + 32 * u[k];
        if (dst != p.send[o[k]] + 32 * u[k]) st32(dst, v[k]);  // in place: rank o's own block is there
      }
  }
}

__global__ void __launch_bounds__(kFlatThreads, kFlatCtasPerSm) local_ag32_kernel(const __grid_constant__ LPlan p) {
  pdl_enter();
  local_ag32_body(p, blockIdx.x, gridDim.x);
}

// All-gather through the tensor memory accelerator: one elected thread per CTA streams tiles of
// the inputs into shared memory with 1-D bulk copies (cp.async.bulk, mbarrier completion) and
// writes each tile to the n outputs with n bulk stores, NS stages deep. Full-line writes and no
// per-element instructions; the broadcast is write-bound (n^2 C written, n C read).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kTmaMaxStages = 8;

__global__ void __launch_bounds__(32) local_ag_tma_kernel(const __grid_constant__ LPlan p, int piece, int NS) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[kTmaMaxStages];
  pdl_enter();
  if (threadIdx.x != 0) return;
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const int64_t per_rank = (Cb + piece - 1) / piece;
  const int64_t total = per_rank * n;
  const int64_t mine = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto tile = [&](int64_t k, int& o, int64_t& off, uint32_t& len) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    o = static_cast<int>(t / per_rank);
    off = (t - static_cast<int64_t>(o) * per_rank) * piece;
    len = static_cast<uint32_t>(Cb - off < piece ? Cb - off : piece);
  };
  auto load = [&](int64_t k) {
    int o;
    int64_t off;
    uint32_t len;
    tile(k, o, off, len);
    const int s = static_cast<int>(k % NS);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bars[s])), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(smem + static_cast<int64_t>(s) * piece)),
                 "l"(p.send[o] + off), "r"(len), "r"(smem_addr(&bars[s]))
                 : "memory");
  };
  for (int64_t k = 0; k < mine && k < NS; ++k) load(k);
  uint32_t phase = 0;  // bit s = parity of stage s
  for (int64_t k = 0; k < mine; ++k) {
    const int s = static_cast<int>(k % NS);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                   : "=r"(done)
                   : "r"(smem_addr(&bars[s])), "r"((phase >> s) & 1u)
                   : "memory");
    phase ^= 1u << s;
    int o;
    int64_t off;
    uint32_t len;
    tile(k, o, off, len);
    const bool inplace = p.recv[o] + o * Cb == p.send[o];
    for (int r = 0; r < n; ++r) {
      if (inplace && r == o) continue;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.recv[r] + o * Cb + off),
                   "r"(smem_addr(smem + static_cast<int64_t>(s) * piece)), "r"(len)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the previous tile's stores have read their stage: refill it NS tiles ahead
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (k >= 1 && k - 1 + NS < mine) load(k - 1 + NS);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Reduce-scatter: out[r] = tree(x_0..x_{n-1}), x_j = send[(r+j) % n] block r.
template <int DT, int OP, int N>
__device__ __forceinline__ void local_rs_body(const LPlan& p) {
  const int bpr = gridDim.x / N;
  const int r = blockIdx.x / bpr;
  const int b = blockIdx.x - r * bpr;
  const int64_t Cb = p.chunk_bytes;
  const char* src[N];
#pragma unroll
  for (int j = 0; j < N; ++j) src[j] = p.send[(r + j) % N] + r * Cb;
  char* dst = p.recv[r];
  if (p.vec == 16) {
    const int64_t nu = Cb >> 4;
    const int64_t step = static_cast<int64_t>(bpr) * blockDim.x;
    for (int64_t u = static_cast<int64_t>(b) * blockDim.x + threadIdx.x; u < nu; u += step) {
      uint4 x[N];
#pragma unroll
      for (int j = 0; j < N; ++j) x[j] = ld_nc16(src[j] + 16 * u);
      st_cs16(dst + 16 * u, tree<DT, OP, N>(x));
    }
  } else {
    using S = typename DType<DT>::S;
    const int64_t ne = Cb / static_cast<int64_t>(sizeof(S));
    for (int64_t e = static_cast<int64_t>(b) * blockDim.x + threadIdx.x; e < ne;
         e += static_cast<int64_t>(bpr) * blockDim.x) {
      S x[N];
#pragma unroll
      for (int j = 0; j < N; ++j) x[j] = *reinterpret_cast<const S*>(src[j] + e * static_cast<int64_t>(sizeof(S)));
      *reinterpret_cast<S*>(dst + e * static_cast<int64_t>(sizeof(S))) = tree_scalar<DT, OP, N>(x);
    }
  }
}

// Reduce-scatter, 16-byte units, one wave: global unit g in [0, n * Cb/16) is unit g % nu of
// output rank g / nu, its N loads in flight before the tree (tools/local_tune.cu: 11.5 us at
// n = 8, 1 MiB fp32, against 11.3-12.3 us for the per-rank two-wave grid, which varies with the
// box; a bulk-copy-staged variant reached only 12.7 us).
template <int DT, int OP, int N>
__device__ __forceinline__ void local_rs_flat(const LPlan& p, int blk, int nblk) {
  const int64_t Cb = p.chunk_bytes;
  const int64_t nu = Cb >> 4;
  const int64_t total = N * nu;
  const int64_t TT = static_cast<int64_t>(nblk) * blockDim.x;
  for (int64_t g = static_cast<int64_t>(blk) * blockDim.x + threadIdx.x; g < total; g += TT) {
    const int r = static_cast<int>(g / nu);
    const int64_t off = r * Cb + 16 * (g - r * nu);
    uint4 x[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      int s = r + j;
      s = s >= N ? s - N : s;
      x[j] = ld_nc16(p.send[s] + off);
    }
    st_cs16(p.recv[r] + (off - r * Cb), tree<DT, OP, N>(x));
  }
}

template <int DT, int OP>
__global__ void __launch_bounds__(kLocalThreads, 2) local_rs_kernel(const __grid_constant__ LPlan p) {
  pdl_enter();
  switch (p.n) {
    case 1: local_rs_body<DT, OP, 1>(p); break;
    case 2: local_rs_body<DT, OP, 2>(p); break;
    case 3: local_rs_body<DT, OP, 3>(p); break;
    case 4: local_rs_body<DT, OP, 4>(p); break;
    case 5: local_rs_body<DT, OP, 5>(p); break;
    case 6: local_rs_body<DT, OP, 6>(p); break;
    case 7: local_rs_body<DT, OP, 7>(p); break;
    default: local_rs_body<DT, OP, 8>(p); break;
  }
}

template <int DT, int OP>
__device__ __forceinline__ void local_rs_flat_any(const LPlan& p, int blk, int nblk) {
  switch (p.n) {
    case 1: local_rs_flat<DT, OP, 1>(p, blk, nblk); break;
    case 2: local_rs_flat<DT, OP, 2>(p, blk, nblk); break;
    case 3: local_rs_flat<DT, OP, 3>(p, blk, nblk); break;
    case 4: local_rs_flat<DT, OP, 4>(p, blk, nblk); break;
    case 5: local_rs_flat<DT, OP, 5>(p, blk, nblk); break;
    case 6: local_rs_flat<DT, OP, 6>(p, blk, nblk); break;
    case 7: local_rs_flat<DT, OP, 7>(p, blk, nblk); break;
    default: local_rs_flat<DT, OP, 8>(p, blk, nblk); break;
  }
}

template <int DT, int OP>
__global__ void __launch_bounds__(kFlatThreads, kFlatCtasPerSm) local_rs_flat_kernel(const __grid_constant__ LPlan p) {
  pdl_enter();
  local_rs_flat_any<DT, OP>(p, blockIdx.x, gridDim.x);
}

// A grouped all-gather (a) + reduce-scatter (b, sum) in one launch (patGroupStart/End): the
// first `ga` CTAs broadcast, the rest fold, at the same time — the write-bound broadcast and the
// read-bound fold share HBM instead of taking turns, and one launch ramps up and drains.
struct LPlan2 {
  LPlan a, b;
  int ga;
};
// Interleaved form (default): every thread does both kinds of work each round — kAgU broadcast
// units, then qB fold units — so the two calls drain together instead of one half of the grid
// idling while the other finishes.
template <int DT, int N>
__device__ __forceinline__ void local_group_interleaved(const LPlan2& p) {
  const int64_t nuA = p.a.chunk_bytes >> 5, totA = N * nuA;
  const int64_t nuB = p.b.chunk_bytes >> 4, totB = N * nuB;
  const int64_t TT = static_cast<int64_t>(gridDim.x) * kFlatThreads;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * kFlatThreads + threadIdx.x;
  const int64_t rounds = std::max<int64_t>(1, (totA + kAgU * TT - 1) / (kAgU * TT));
  const int64_t qB = (totB + rounds * TT - 1) / (rounds * TT);
  const int64_t CbA = p.a.chunk_bytes, CbB = p.b.chunk_bytes;
  for (int64_t rd = 0; rd < rounds; ++rd) {
    V8 v[kAgU];
    int o[kAgU];
    int64_t u[kAgU];
#pragma unroll
    for (int k = 0; k < kAgU; ++k) {  // broadcast loads first: in flight while the folds run
      const int64_t gg = tid + (rd * kAgU + k) * TT;
      o[k] = gg < totA ? static_cast<int>(gg / nuA) : -1;
      u[k] = gg - static_cast<int64_t>(o[k]) * nuA;
      if (o[k] >= 0) v[k] = ld_nc32(p.a.send[o[k]] + 32 * u[k]);
    }
    for (int64_t j = 0; j < qB; ++j) {
      const int64_t g = tid + (rd * qB + j) * TT;
      if (g >= totB) break;
      const int r = static_cast<int>(g / nuB);
      const int64_t off = r * CbB + 16 * (g - r * nuB);
      uint4 x[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        int src = r + i;
        src = src >= N ? src - N : src;
        x[i] = ld_nc16(p.b.send[src] + off);
      }
      st_cs16(p.b.recv[r] + (off - r * CbB), tree<DT, kSum, N>(x));
    }
    for (int dst_r = 0; dst_r < N; ++dst_r)
#pragma unroll
      for (int k = 0; k < kAgU; ++k) {
        if (o[k] < 0) continue;
        char* dst = p.a.recv[dst_r] + o[k] * CbA + 32 * u[k];
        if (dst != p.a.send[o[k]] + 32 * u[k]) st32(dst, v[k]);
      }
  }
}

constexpr int kGroupCtasPerSm = 2;  // interleaved body: ~80 registers; 2 CTAs/SM measured 1% faster than 3 (tools/local_tune.cu group)
template <int DT>
__global__ void __launch_bounds__(kFlatThreads, kGroupCtasPerSm) local_group_kernel(const __grid_constant__ LPlan2 p) {
  pdl_enter();
  if (p.ga < 0) {  // interleaved
    switch (p.a.n) {
      case 1: local_group_interleaved<DT, 1>(p); break;
      case 2: local_group_interleaved<DT, 2>(p); break;
      case 3: local_group_interleaved<DT, 3>(p); break;
      case 4: local_group_interleaved<DT, 4>(p); break;
      case 5: local_group_interleaved<DT, 5>(p); break;
      case 6: local_group_interleaved<DT, 6>(p); break;
      case 7: local_group_interleaved<DT, 7>(p); break;
      default: local_group_interleaved<DT, 8>(p); break;
    }
    return;
  }
  if (static_cast<int>(blockIdx.x) < p.ga) local_ag32_body(p.a, blockIdx.x, p.ga);
  else local_rs_flat_any<DT, kSum>(p.b, blockIdx.x - p.ga, gridDim.x - p.ga);
}
using LocalGroupFn = void (*)(const LPlan2);
static const LocalGroupFn kLocalGroup[10] = {
    local_group_kernel<kI8>, local_group_kernel<kU8>, local_group_kernel<kI32>, local_group_kernel<kU32>,
    local_group_kernel<kI64>, local_group_kernel<kU64>, local_group_kernel<kF16>, local_group_kernel<kF32>,
    local_group_kernel<kF64>, local_group_kernel<kBF16>};

using LocalFn = void (*)(const LPlan);
#define PAT_LRS_ROW(DT) \
  { local_rs_kernel<DT, kSum>, local_rs_kernel<DT, kProd>, local_rs_kernel<DT, kMax>, local_rs_kernel<DT, kMin> }
static const LocalFn kLocalRs[10][4] = {
    PAT_LRS_ROW(kI8), PAT_LRS_ROW(kU8), PAT_LRS_ROW(kI32), PAT_LRS_ROW(kU32), PAT_LRS_ROW(kI64),
    PAT_LRS_ROW(kU64), PAT_LRS_ROW(kF16), PAT_LRS_ROW(kF32), PAT_LRS_ROW(kF64), PAT_LRS_ROW(kBF16)};
#define PAT_LRSF_ROW(DT)                                                                             \
  {                                                                                                  \
    local_rs_flat_kernel<DT, kSum>, local_rs_flat_kernel<DT, kProd>, local_rs_flat_kernel<DT, kMax>, \
        local_rs_flat_kernel<DT, kMin>                                                               \
  }
static const LocalFn kLocalRsFlat[10][4] = {
    PAT_LRSF_ROW(kI8), PAT_LRSF_ROW(kU8), PAT_LRSF_ROW(kI32), PAT_LRSF_ROW(kU32), PAT_LRSF_ROW(kI64),
    PAT_LRSF_ROW(kU64), PAT_LRSF_ROW(kF16), PAT_LRSF_ROW(kF32), PAT_LRSF_ROW(kF64), PAT_LRSF_ROW(kBF16)};

// The tree the fused reduce-scatter evaluates, in the symbolic form comm.cpp produces.
const char* local_tree_string(int n) {
  switch (n) {
    case 1: return "x0";
    case 2: return "(x0+x1)";
    case 3: return "((x0+x1)+x2)";
    case 4: return "((x0+x1)+(x3+x2))";
    case 5: return "(((x0+x1)+(x3+x2))+x4)";
    case 6: return "(((x0+x1)+(x3+x2))+(x5+x4))";
    case 7: return "(((x0+x1)+(x3+x2))+((x5+x6)+x4))";
    case 8: return "(((x0+x1)+(x3+x2))+((x5+(x7+x6))+x4))";
    default: return "";
  }
}

// PAT_PDL=0 launches without programmatic stream serialization (A/B experiments).
// Transport launches: programmatic dependent launch pays off inside CUDA graphs (7.05 vs 7.34 us
// per n = 2 call) but costs eager stream launches 0.4-1 us (10.7 vs 9.7-10.3 us,
// tools/eager_probe_mp.py, profiles/r02_eager_probe_pdl.txt), so it is requested only while the
// stream is being captured. The fused executor's kernels keep it either way (eager 12.9 vs 14.8 us
// per call without it: their launches hide behind the previous kernel's drain).
bool pdl_for(cudaStream_t stream) {
  static const int mode = [] {  // PAT_PDL: 0 never, 1 always, unset: graphs only
    const char* e = std::getenv("PAT_PDL");
    return e ? std::atoi(e) : -1;
  }();
  if (mode >= 0) return mode != 0;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs == cudaStreamCaptureStatusActive;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PAT_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

cudaError_t launch_local(int kind, int n, int dtype, int op, int vec, int esize, int64_t chunk_bytes,
                         const char* const* send_by_rank, char* const* recv_by_rank, int sm_count,
                         cudaStream_t stream) {
  LPlan p{};
  p.n = n;
  p.kind = kind;
  p.vec = vec;
  p.esize = esize;
  p.chunk_bytes = chunk_bytes;
  for (int r = 0; r < n; ++r) {
    p.send[r] = send_by_rank[r];
    p.recv[r] = recv_by_rank[r];
  }
  const int64_t per_rank_units = vec == 16 ? (chunk_bytes >> 4) : (chunk_bytes / esize);
  const int64_t want = (per_rank_units + kLocalThreads - 1) / kLocalThreads;
  // per rank: enough blocks for ~4 resident CTAs on every SM overall, no more than the units
  const int bpr = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, (4LL * sm_count + n - 1) / n)));
  // all-gather: the bulk-copy kernel (8 KiB tiles, 4 stages, 2 CTAs per SM: measured 12.5 us vs
  // 14.0 us for the vector kernel at n=8, 1 MiB; tools/tune_local*.sh). PAT_LOCAL_TMA=0 turns it off.
  static const int tma_piece = [] {
    const char* e = std::getenv("PAT_LOCAL_TMA");
    if (!e) return 8192;
    const int v = std::atoi(e);
    return v >= 1024 ? (v & ~15) : 0;
  }();
  constexpr int kTmaStages = 4;
  cudaLaunchConfig_t cfg = {};
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see pdl_enter
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  // PAT_LOCAL_FLAT=0: the previous kernels (bulk-copy all-gather, per-rank reduce-scatter grid)
  static const bool flat = [] {
    const char* e = std::getenv("PAT_LOCAL_FLAT");
    return !e || std::atoi(e) != 0;
  }();
  bool aligned32 = (chunk_bytes % 32) == 0;
  for (int r = 0; r < n && aligned32; ++r)
    aligned32 = ((reinterpret_cast<uintptr_t>(p.send[r]) | reinterpret_cast<uintptr_t>(p.recv[r])) % 32) == 0;
  const int64_t units = n * (chunk_bytes >> (kind == 0 ? 5 : 4));
  const int flat_grid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(int64_t{kFlatCtasPerSm} * sm_count, (units + kFlatThreads - 1) / kFlatThreads)));
  if (flat && vec == 16 && (kind == 1 || aligned32)) {
    cfg.gridDim = dim3(flat_grid);
    cfg.blockDim = dim3(kFlatThreads);
    if (kind == 0) return cudaLaunchKernelEx(&cfg, local_ag32_kernel, p);
    return cudaLaunchKernelEx(&cfg, kLocalRsFlat[dtype][op], p);
  }
  if (kind == 0 && tma_piece && vec == 16) {
    const int smem = kTmaStages * tma_piece;
    if (smem > 48 * 1024)  // per device; only for tiles set above the default through the env
      cudaFuncSetAttribute(local_ag_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cfg.gridDim = dim3(2 * sm_count);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    return cudaLaunchKernelEx(&cfg, local_ag_tma_kernel, p, tma_piece, kTmaStages);
  }
  cfg.gridDim = dim3(bpr * n);
  cfg.blockDim = dim3(kLocalThreads);
  if (kind == 0) return cudaLaunchKernelEx(&cfg, local_ag_kernel, p);
  return cudaLaunchKernelEx(&cfg, kLocalRs[dtype][op], p);
}

// Grouped all-gather (chunk a_bytes) + reduce-scatter (sum, chunk b_bytes) of one single-device
// communicator in one launch. Returns cudaErrorNotSupported when the flat kernels cannot take
// both (alignment): the caller launches them one after the other instead.
cudaError_t launch_local_group(int n, int dtype, int64_t a_bytes, const char* const* a_send, char* const* a_recv,
                               int64_t b_bytes, const char* const* b_send, char* const* b_recv, int sm_count,
                               cudaStream_t stream) {
  LPlan2 p{};
  p.a.n = p.b.n = n;
  p.a.kind = 0;
  p.b.kind = 1;
  p.a.vec = p.b.vec = 16;
  p.a.chunk_bytes = a_bytes;
  p.b.chunk_bytes = b_bytes;
  bool ok = (a_bytes % 32) == 0 && (b_bytes % 16) == 0;
  for (int r = 0; r < n; ++r) {
    p.a.send[r] = a_send[r];
    p.a.recv[r] = a_recv[r];
    p.b.send[r] = b_send[r];
    p.b.recv[r] = b_recv[r];
    ok = ok && ((reinterpret_cast<uintptr_t>(a_send[r]) | reinterpret_cast<uintptr_t>(a_recv[r])) % 32) == 0 &&
         ((reinterpret_cast<uintptr_t>(b_send[r]) | reinterpret_cast<uintptr_t>(b_recv[r])) % 16) == 0;
  }
  if (!ok) return cudaErrorNotSupported;
  // CTAs split in proportion to each call's HBM bytes ((n^2 + n) C for both)
  const int grid = kGroupCtasPerSm * sm_count;
  const double wa = static_cast<double>(a_bytes), wb = static_cast<double>(b_bytes);
  p.ga = std::max(1, std::min(grid - 1, static_cast<int>(grid * wa / (wa + wb) + 0.5)));
  // PAT_GROUP_LOCAL: 0 = interleaved (default), 1 = the grid split in two halves
  static const int mode = [] {
    const char* e = std::getenv("PAT_GROUP_LOCAL");
    return e ? std::atoi(e) : 0;
  }();
  if (mode == 0) p.ga = -1;
  cudaLaunchConfig_t cfg = {};
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFlatThreads);
  return cudaLaunchKernelEx(&cfg, kLocalGroup[dtype], p);
}

}  // namespace pat
