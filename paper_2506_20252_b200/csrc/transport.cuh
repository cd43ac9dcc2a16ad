// transport.cuh — the sm_100a transport kernel for PAT all-gather and reduce-scatter
// (instantiated in kernels.cu and rs_*.cu).
//
// One cooperative launch per device per collective. CTA (lr, c) runs channel c of local rank
// lr through `iters` pipeline steps; step i moves slice (i*channels + c) of every chunk
// through all PAT rounds. Per round the rank pushes its <= T chunk slices into the inbox of
// peer (r + peer) over NVLink (or HBM in local mode), then signals; receivers fold or copy
// from their own inbox. This replaces the reference executor's send/deliver phases
// (simulate.cpp:180-218 all-gather, :247-296 reduce-scatter) and its Mailbox rendezvous +
// lockstep join (simulate.cpp:49-70, 131-149) with per-step release/acquire flags.
//
// Protocols (the host's calibrated cost model picks one per call, comm.cpp: choose_slicing):
//  * LL32 (512 KiB up to (n-1) C = 48 MiB): like LL below with 32-byte lines and one flag word
//    (87.5% wire efficiency); see ll32_phase.
//  * LL (up to 256 KiB): 16-byte lines {data32, flag, data32, flag} stored with one
//    st.volatile.v4 into the peer's inbox; the receiver polls the line itself, so data and
//    signal travel together and no fence or separate flag is needed. 50% wire efficiency.
//    Every thread owns the same words of every chunk in every round: no CTA barriers.
//  * SIMPLE (bulk): warp-specialised. Sender warps push 16-byte vectors of the slice into the
//    peer (inbox slot, or the peer's recvbuf directly in direct all-gather mode), then one
//    thread issues fence.acq_rel + st.relaxed of the (channel, round) flag at the receiver
//    (NCCL-style: named barrier, then a single release). Receiver warps wait for the flags
//    and deliver (all-gather) or fold the output (reduce-scatter), so step g+1's pushes
//    overlap step g's delivery.
//  * PULL (mid-size reduce-scatter in one process): receivers read the upstream's buffers;
//    see pull_role.
// Inbox slots are `depth`-buffered by step; a rank re-uses a peer's slot buffer only after
// that peer published "done with step g-depth" (credit flags), so the pool is bounded:
// channels * depth * (n-1) slots per rank, independent of the message size.
//
// Reduction order (reduce-scatter) is the reference's exactly: a forwarded offset carries
// fold(arrivals in round order) (+) own contribution (simulate.cpp:257-266, 281-285); the
// output is own (+) offset-0 arrivals in round order (simulate.cpp:239, 278-279). Each fold
// is rounded to the wire dtype (fp16/bf16 computed in fp32, RNE).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "fold.cuh"
#include "plan.hpp"

// PAT_BOUNDS_CHECK builds (tools/build_variant.sh bounds -DPAT_BOUNDS_CHECK=1) trap on any inbox
// slot or user-buffer range outside its allocation: the stand-in for compute-sanitizer's memcheck,
// which is closed on this GPU pool (profiles/r02_sanitizer.txt).
#ifdef PAT_BOUNDS_CHECK
#define PAT_BOUND(cond)                                                                              \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("pat bounds: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x, threadIdx.x); \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define PAT_BOUND(cond) \
  do {                  \
  } while (0)
#endif

#ifndef PAT_EXTRA_BARRIERS  // A/B builds: 1 restores the barriers the r02 prologue / epilogue dropped
#define PAT_EXTRA_BARRIERS 0
#endif

namespace pat {

// ------------------------------------------------------------------------- memory primitives

// Flags and fences at .gpu scope when every rank lives on this device, .sys across GPUs.
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p, bool gpu) {
  uint64_t v;
  if (gpu) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v, bool gpu) {
  if (gpu) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v, bool gpu) {
  if (gpu) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel(bool gpu) {
  if (gpu) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint4 ld16(const void* p) {  // L2-coherent (bypasses a stale L1)
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st16(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_ll(void* p, uint2 v, uint32_t flag) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(flag), "r"(v.y),
               "r"(flag)
               : "memory");
}
__device__ __forceinline__ uint4 ld_volatile16(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
// ------------------------------------------------------------------------- waits

struct Waiter {
  uint64_t timeout_ns;
  int* err;
  bool aborted;
  bool gpu;  // flag scope
  const uint64_t* cred0 = nullptr;  // credits read at kernel entry, per peer (valid for step `base`)
  uint64_t base = 0;
};

// ------------------------------------------------------------------------- device trace
#ifndef PAT_TRACE_POLL
#define PAT_TRACE_POLL 0  // trace events in the LL / LL32 path (diagnostic builds only)
#endif
// Event codes (bits 56..63 event, 40..55 step, 32..39 round); one writer thread per role.
enum TraceEv : uint64_t {
  kEvStart = 1, kEvCredit = 2, kEvPushed = 3, kEvFenced = 4, kEvArrived = 5, kEvDelivered = 6, kEvDone = 7,
  kEvEnd = 8, kEvWaitArr = 9
};

struct Tracer {
  uint64_t* buf = nullptr;
  int cap = 0, n = 0;
  __device__ __forceinline__ void init(const KPlan& p, int role) {
    if (p.trace) {
      buf = p.trace + (static_cast<int64_t>(blockIdx.x) * 2 + role) * p.trace_cap * 2;
      cap = p.trace_cap;
    }
  }
  __device__ __forceinline__ void rec(uint64_t ev, uint64_t step, int round) {
    if (buf && n < cap) {
      buf[2 * n] = globaltimer();
      buf[2 * n + 1] = (ev << 56) | ((step & 0xffff) << 40) | (static_cast<uint64_t>(round & 0xff) << 32);
      ++n;
    }
  }
};

static __device__ __noinline__ void report_timeout(Waiter& w) {
  if (!w.aborted) {
    atomicCAS_system(w.err, 0, 40 /* patTimeout */);
    w.aborted = true;
  }
}

// Spin until *flag >= want (acquire). Thread-level; callers broadcast with a barrier.
__device__ __forceinline__ void wait_flag(const uint64_t* flag, uint64_t want, Waiter& w) {
  if (w.aborted) return;
  uint64_t start = 0;
  uint32_t spins = 0;
  while (ld_acquire(flag, w.gpu) < want) {
    if ((++spins & 1023u) == 0) {
      const uint64_t now = globaltimer();
      if (start == 0) start = now;
      else if (now - start > w.timeout_ns) { report_timeout(w); return; }
    }
  }
}

// Poll one LL line until both flag words carry `flag`; returns its 8 data bytes.
__device__ __forceinline__ uint2 ld_ll(const char* line, uint32_t flag, Waiter& w) {
  uint4 v = ld_volatile16(line);
  if (v.y == flag && v.w == flag) return make_uint2(v.x, v.z);
  uint64_t start = 0;
  uint32_t spins = 0;
  while (!w.aborted) {
    v = ld_volatile16(line);
    if (v.y == flag && v.w == flag) break;
    if ((++spins & 1023u) == 0) {
      const uint64_t now = globaltimer();
      if (start == 0) start = now;
      else if (now - start > w.timeout_ns) report_timeout(w);
    }
  }
  return make_uint2(v.x, v.z);
}

// ------------------------------------------------------------------------- group data movers

// dst = fold_left(src[0], ..., src[m-1]) over `len` bytes (16-byte vectors; len % 16 == 0),
// by the `nthr` threads of one warp group (thread index `tid` within the group).
template <int DT, int OP>
__device__ __forceinline__ void grp_fold16(char* dst, const char* const* src, int m, int64_t len, int tid, int nthr) {
  const int64_t nu = len >> 4;
  const int64_t B = nthr;
  int64_t u = tid;
  if (m == 1) {  // copy: 8 independent 16-byte loads in flight per thread
    const char* s0 = src[0];
    constexpr int U = 8;
    for (; u + (U - 1) * B < nu; u += U * B) {
      uint4 v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) v[k] = ld16(s0 + 16 * (u + k * B));
#pragma unroll
      for (int k = 0; k < U; ++k) st16(dst + 16 * (u + k * B), v[k]);
    }
    for (; u < nu; u += B) st16(dst + 16 * u, ld16(s0 + 16 * u));
    return;
  }
  constexpr int U = 4;
  for (; u + (U - 1) * B < nu; u += U * B) {
    uint4 a[U];
#pragma unroll
    for (int i = 0; i < U; ++i) a[i] = ld16(src[0] + 16 * (u + i * B));
    for (int k = 1; k < m; ++k) {
      uint4 b[U];
#pragma unroll
      for (int i = 0; i < U; ++i) b[i] = ld16(src[k] + 16 * (u + i * B));
#pragma unroll
      for (int i = 0; i < U; ++i) fold_vec<DT, OP>(a[i], b[i]);
    }
#pragma unroll
    for (int i = 0; i < U; ++i) st16(dst + 16 * (u + i * B), a[i]);
  }
  for (; u < nu; u += B) {
    uint4 a = ld16(src[0] + 16 * u);
    for (int k = 1; k < m; ++k) fold_vec<DT, OP>(a, ld16(src[k] + 16 * u));
    st16(dst + 16 * u, a);
  }
}

// Element-granular variant for buffers that are not 16-byte aligned.
template <int DT, int OP>
__device__ __forceinline__ void grp_fold_elems(char* dst, const char* const* src, int m, int64_t len, int esize,
                                               int tid, int nthr) {
  const int64_t ne = len / esize;
  for (int64_t e = tid; e < ne; e += nthr) {
    uint64_t a = ld_elem(src[0] + e * esize, esize);
    for (int k = 1; k < m; ++k) a = fold_elem_bits<DT, OP>(a, ld_elem(src[k] + e * esize, esize));
    st_elem(dst + e * esize, a, esize);
  }
}

template <int DT, int OP>
__device__ __forceinline__ void grp_fold(char* dst, const char* const* src, int m, int64_t len, const KPlan& p,
                                         int tid, int nthr) {
  if (len <= 0) return;
  if (p.vec == 16) grp_fold16<DT, OP>(dst, src, m, len, tid, nthr);
  else grp_fold_elems<DT, OP>(dst, src, m, len, p.esize, tid, nthr);
}

// 8-byte user words for LL (zero padded past `valid`).
__device__ __forceinline__ uint2 load_word(const char* p, int valid, const KPlan& pl) {
  if (valid == 8 && pl.vec >= 8) {  // user buffer, read-only during the call
    const uint64_t v = *reinterpret_cast<const uint64_t*>(p);
    return make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
  }
  uint64_t v = 0;
  for (int b = 0; b < valid; b += pl.esize) v |= ld_elem(p + b, pl.esize) << (8 * b);
  return make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
}
__device__ __forceinline__ void store_word(char* p, uint2 w, int valid, const KPlan& pl) {
  const uint64_t v = static_cast<uint64_t>(w.x) | (static_cast<uint64_t>(w.y) << 32);
  if (valid == 8 && pl.vec >= 8) {
    *reinterpret_cast<uint64_t*>(p) = v;
    return;
  }
  for (int b = 0; b < valid; b += pl.esize) {
    const uint64_t mask = pl.esize == 8 ? ~0ull : ((1ull << (8 * pl.esize)) - 1);
    st_elem(p + b, (v >> (8 * b)) & mask, pl.esize);
  }
}

// ------------------------------------------------------------------------- steps

struct Step {
  uint64_t g;        // absolute pipeline step of this channel
  int64_t off, len;  // byte range of the slice within every chunk
  int R, lr, c, buf;
};

__device__ __forceinline__ Step make_step(const KPlan& p, uint64_t base, int i, int R, int lr, int c) {
  Step s;
  s.g = base + i;
  s.off = (static_cast<int64_t>(i) * p.channels + (c - p.chan_base)) * p.slice_bytes;
  s.len = max(int64_t{0}, min(p.slice_bytes, p.chunk_bytes - s.off));
  s.R = R;
  s.lr = lr;
  s.c = c;
  s.buf = static_cast<int>(s.g % static_cast<uint64_t>(p.depth));
  PAT_BOUND(s.len == 0 || (s.off >= 0 && s.off + s.len <= p.chunk_bytes));
  PAT_BOUND(s.len <= p.slice_bytes);
  return s;
}


__device__ __forceinline__ char* slot_ptr(const KPlan& p, int rank, int c, int buf, int j) {
  PAT_BOUND(rank >= 0 && rank < p.n && c >= p.chan_base && c < p.chan_base + p.channels && buf >= 0 &&
            buf < p.depth && j >= 0 && j < p.nslots);
  PAT_BOUND(c * p.chan_stride + (static_cast<int64_t>(buf) * p.nslots + j + 1) * p.slot_stride <= p.region_bytes);
  return p.inbox[rank] + c * p.chan_stride + (static_cast<int64_t>(buf) * p.nslots + j) * p.slot_stride;
}

// PULL staging: accumulator `a` of buffer `buf` (pull_nacc accumulators per buffer)
__device__ __forceinline__ char* acc_ptr(const KPlan& p, int rank, int c, int buf, int a) {
  PAT_BOUND(rank >= 0 && rank < p.n && a >= 0 && a < p.pull_nacc && buf >= 0 && buf < p.depth);
  PAT_BOUND(c * p.chan_stride + (static_cast<int64_t>(buf) * p.pull_nacc + a + 1) * p.slot_stride <= p.region_bytes);
  return p.inbox[rank] + c * p.chan_stride + (static_cast<int64_t>(buf) * p.pull_nacc + a) * p.slot_stride;
}

__device__ __forceinline__ uint64_t* chan_flags(const KPlan& p, int rank, int c) {
  return p.flags[rank] + c * kFlagWords;
}

// ------------------------------------------------------------------------- flag epochs
// LL and LL32 lines carry the 32-bit value uint32(g + 1) of a 64-bit step counter, so a line
// last written 2^32 steps ago (or never written, at g + 1 = 2^32) would pass for the current
// step. The owner of an inbox therefore re-stamps its polling buffers once per 2^31 steps: the
// receiver of step g, when g + 1 is within depth_poll of an epoch start, rewrites buffer
// g % depth_poll of channel c in its LL and LL32 regions with lines that are complete for step
// value V = uint32(g + 1) - 2^30 and zero data — a value no step polls in the next 3 * 2^30
// steps — after consuming step g and before publishing done(g). A sender writes that buffer
// again only for step g + depth_poll, after done(g), so the re-stamp cannot race a write.
// (NCCL's LL protocol cleans its buffers near the flag wrap the same way.)
__device__ __forceinline__ bool epoch_clean_due(const KPlan& p, uint64_t g) {
  return ((g + 1) & p.epoch_mask) < static_cast<uint64_t>(p.depth_poll);
}
// by threads [tid, nthr) of the receiver; the caller fences before publishing done(g)
static __device__ __noinline__ void epoch_clean(const KPlan& p, int R, int c, uint64_t g, int tid, int nthr) {
  const uint32_t V = static_cast<uint32_t>(g + 1) - 0x40000000u;
  const int b = static_cast<int>(g % static_cast<uint64_t>(p.depth_poll));
  const int64_t per_buf[2] = {static_cast<int64_t>(p.nslots) * p.poll_slot[0],
                              static_cast<int64_t>(p.nslots) * p.poll_slot[1]};
  char* pool = reinterpret_cast<char*>(p.flags[R]);
  if (c < p.poll_channels[0]) {  // LL lines {data, flag, data, flag}
    uint4* q = reinterpret_cast<uint4*>(pool + p.poll_off[0] + (static_cast<int64_t>(c) * p.depth_poll + b) * per_buf[0]);
    for (int64_t i = tid; i < per_buf[0] / 16; i += nthr) q[i] = make_uint4(0, V, 0, V);
  }
  if (c < p.poll_channels[1]) {  // LL32 lines {7 zero words, V ^ hash(0) = V}
    uint4* q = reinterpret_cast<uint4*>(pool + p.poll_off[1] + (static_cast<int64_t>(c) * p.depth_poll + b) * per_buf[1]);
    for (int64_t i = tid; i < per_buf[1] / 16; i += nthr) q[i] = (i & 1) ? make_uint4(0, 0, 0, V) : make_uint4(0, 0, 0, 0);
  }
}

// Symmetric windows: a rank publishes its call's window tag to every peer before its entry
// handshake (release) flag; after acquiring peer Q's handshake it checks Q's tag against its own,
// so a zero-copy access never uses a peer buffer at a different window offset. On a mismatch the
// call reports patInvalidUsage (5) and moves no data.
__device__ __forceinline__ void sym_publish(const KPlan& p, int R, int c, int q, bool gpu) {
  if (p.sym_tag) st_relaxed(p.flags[q] + c * kFlagWords + 24 + R, p.sym_tag, gpu);
}
__device__ __forceinline__ bool sym_check(const KPlan& p, int R, int c, int q, Waiter& w) {
  if (!p.sym_tag || w.aborted) return !w.aborted;
  if (ld_acquire(p.flags[R] + c * kFlagWords + 24 + q, w.gpu) == p.sym_tag) return true;
  atomicCAS_system(w.err, 0, 5 /* patInvalidUsage */);
  w.aborted = true;
  return false;
}

// Credits: before pushing step g into a peer's inbox buffer g % depth, the peer must have
// finished step g - depth (published as done_from[peer] >= g - depth + 1).
__device__ __forceinline__ void wait_credits(const KPlan& p, const Step& s, Waiter& w) {
  if (s.g < static_cast<uint64_t>(p.depth)) return;
  const uint64_t* mine = chan_flags(p, s.R, s.c);
  for (int k = 0; k < p.npeers; ++k) wait_flag(mine + 8 + (s.R + p.peers[k]) % p.n, s.g - p.depth + 1, w);
}
// The same, one peer per thread (threads [0, npeers) of the caller's group, which then barriers):
// the npeers acquire loads overlap instead of following one another (a small call waits on
// ceil(log2 n) distinct peers: 3 at n = 8). PAT_SERIAL_CREDITS builds keep the one-thread form.
__device__ __forceinline__ void wait_credits_par(const KPlan& p, const Step& s, Waiter& w, int tid) {
#ifdef PAT_SERIAL_CREDITS
  if (tid == 0) wait_credits(p, s, w);
#else
  if (tid >= p.npeers || s.g < static_cast<uint64_t>(p.depth)) return;
  const uint64_t want = s.g - p.depth + 1;
  if (w.cred0 && s.g == w.base && w.cred0[tid] >= want) return;  // the entry read already saw it
  wait_flag(chan_flags(p, s.R, s.c) + 8 + (s.R + p.peers[tid]) % p.n, want, w);
#endif
}

// ------------------------------------------------------------------------- live occupancy
// (PAT_STATS) Counted by the device as the step runs: the receiver role, once round t's flag is
// acquired, counts the slots of round t that stay held — all-gather: an arrival a later round
// forwards (brute_force.hpp occupancy_allgather); reduce-scatter: the first arrival toward an
// offset opens its accumulator (occupancy_reduce_scatter). The sender role, after pushing round
// t, counts the slots it released — the last forward of an arrival / the forward that closes an
// accumulator. Occupancy after round t = sum over rounds <= t of held - released (host).
__device__ __forceinline__ bool ag_forwarded_after(const KPlan& p, int j, int t) {
  for (int t2 = t + 1; t2 < p.nrounds; ++t2)
    for (int q = 0; q < p.rounds[t2].nchunks; ++q)
      if (p.rounds[t2].narr[q] && p.rounds[t2].arr[q][0] == j) return true;
  return false;
}
static __device__ __noinline__ void occ_arrived(const KPlan& p, int lr, int t) {
  const KRound& r = p.rounds[t];
  int held = 0;
  for (int pos = 0; pos < r.nchunks; ++pos) {
    const int j = r.slot_base + pos, k = p.slot_offset[j];
    if (k == 0) continue;
    if (p.kind == kAG) {
      held += ag_forwarded_after(p, j, t);
    } else {
      bool first = true;
      for (int j2 = 0; j2 < j; ++j2) first &= p.slot_offset[j2] != k;
      held += first;
    }
  }
  atomicAdd(p.occ + (lr * 2 + 0) * kMaxRounds + t, held);
}
static __device__ __noinline__ void occ_sent(const KPlan& p, int lr, int t) {
  const KRound& r = p.rounds[t];
  int released = 0;
  for (int pos = 0; pos < r.nchunks; ++pos) {
    if (!r.narr[pos]) continue;
    released += p.kind == kAG ? !ag_forwarded_after(p, r.arr[pos][0], t) : 1;
  }
  atomicAdd(p.occ + (lr * 2 + 1) * kMaxRounds + t, released);
}

// SIMPLE sender role, one PAT round of step s (warps [0, send_warps)). `waited` caches which
// rounds' arrivals of this step were already acquired. `part` selects the round's positions:
// kAllPos, kLeafPos (chunks that carry no arrival: the own chunk in all-gather, a bare own
// contribution in reduce-scatter) or kFwdPos (the rest).
enum : int { kAllPos = 0, kLeafPos = 1, kFwdPos = 2 };
template <int DT, int OP, int KIND>
__device__ void send_round(const KPlan& p, const Step& s, int t, uint32_t& waited, Waiter& w, int tid, int nthr,
                           bool signal, int part = kAllPos) {
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const char* snd = p.send[s.lr];
  char* out = p.recv[s.lr];
  const uint64_t* myflags = chan_flags(p, s.R, s.c);
  const bool gpu = p.gpu_scope;
  auto ensure = [&](int tr) {  // arrivals of round tr (needed for forwarding)
    if (!((waited >> tr) & 1u)) {
      if (tid == 0) wait_flag(myflags + tr, s.g + 1, w);
      named_bar(1, nthr);
      waited |= 1u << tr;
    }
  };
  const char* srcs[kMaxArr + 1];
  {
    const KRound& r = p.rounds[t];
    const int P = (s.R + r.peer) % n;
    for (int pos = 0; pos < r.nchunks; ++pos) {
      if (part != kAllPos && (r.narr[pos] == 0) != (part == kLeafPos)) continue;
      int m = 0;
      char* dst;
      if constexpr (KIND == kAG) {
        const int origin = (s.R - r.chunk[pos] + n) % n;
        if (r.narr[pos] == 0) {
          srcs[m++] = snd + s.off;
        } else {
          const int j = r.arr[pos][0];
          ensure(p.slot_round[j]);
          srcs[m++] = p.direct ? out + origin * Cb + s.off : slot_ptr(p, s.R, s.c, s.buf, j);
        }
        dst = p.direct ? p.peer_recv[P] + origin * Cb + s.off : slot_ptr(p, P, s.c, s.buf, r.slot_base + pos);
      } else {
        const int dest = (s.R - r.chunk[pos] + n) % n;
        for (int a = 0; a < r.narr[pos]; ++a) {
          const int j = r.arr[pos][a];
          ensure(p.slot_round[j]);
          srcs[m++] = slot_ptr(p, s.R, s.c, s.buf, j);
        }
        srcs[m++] = snd + dest * Cb + s.off;  // own contribution folded last
        dst = slot_ptr(p, P, s.c, s.buf, r.slot_base + pos);
      }
      grp_fold<DT, OP>(dst, srcs, m, s.len, p, tid, nthr);
    }
    if (signal) {
      named_bar(1, nthr);
      if (tid == 0) {
        fence_acq_rel(gpu);
        st_relaxed(chan_flags(p, P, s.c) + t, s.g + 1, gpu);
      }
    }
  }
}

// SIMPLE sender role over all steps. With p.skew, iteration k runs round t of step k - t
// (oldest step first): a forward of round t waits for arrivals its upstream peer pushed one
// iteration earlier, so the flag latency hides behind the next step's pushes (a wavefront
// through the PAT tree). Needs depth > nrounds - 1 inbox buffers (host guarantees).
template <int DT, int OP, int KIND>
__device__ void send_role(const KPlan& p, uint64_t base, int R, int lr, int c, Waiter& w, int tid, int nthr,
                          volatile uint64_t* sent_steps) {
  const int NR = p.nrounds;
  uint32_t waited[kMaxRounds] = {};
  Tracer tr;
  if (tid == 0) tr.init(p, 0);
  tr.rec(kEvStart, base, 0);
  auto task = [&](int i, int t, bool signal) {
    const Step s = make_step(p, base, i, R, lr, c);
    uint32_t& wm = waited[i % kMaxRounds];
    if (t == 0) {  // first push of step i: the peers' buffers (g % depth) must be free
      wm = 0;
      if (!p.direct) wait_credits_par(p, s, w, tid);
      tr.rec(kEvCredit, s.g, 0);
      named_bar(1, nthr);
      // leaves first: every round's dependency-free chunks go out now, so the link is busy while
      // the forwards of later rounds wait for their arrivals (each round's flag still follows
      // all of its positions: it is published after a later fence)
      if (p.leaves_first)
        for (int t2 = 0; t2 < NR; ++t2) send_round<DT, OP, KIND>(p, s, t2, wm, w, tid, nthr, false, kLeafPos);
    }
    send_round<DT, OP, KIND>(p, s, t, wm, w, tid, nthr, signal, p.leaves_first ? kFwdPos : kAllPos);
    if (p.occ && i == 0 && c == p.chan_base && tid == 0) occ_sent(p, lr, t);
    tr.rec(kEvPushed, s.g, t);
    if (signal && t == NR - 1 && tid == 0) *sent_steps = s.g + 1;  // after the round's barrier
  };
  if (p.skew) {
    // Round t of step k - t*L in iteration k (L = p.skew): the newest step's independent
    // round 0 goes first, forwards of older steps after it, then ONE fence for the iteration
    // and all of its flags.
    const int L = p.skew;
    for (int k = 0; k < p.iters + (NR - 1) * L; ++k) {
      for (int t = 0; t < NR; ++t)
        if (k - t * L >= 0 && k - t * L < p.iters) task(k - t * L, t, false);
      named_bar(1, nthr);
      if (tid == 0) {
        fence_acq_rel(p.gpu_scope);
        tr.rec(kEvFenced, base + k, 0);
        for (int t = NR - 1; t >= 0; --t) {
          const int i = k - t * L;
          if (i < 0 || i >= p.iters) continue;
          st_relaxed(chan_flags(p, (R + p.rounds[t].peer) % p.n, c) + t, base + i + 1, p.gpu_scope);
          if (t == NR - 1) *sent_steps = base + i + 1;
        }
      }
    }
  } else {
    for (int i = 0; i < p.iters; ++i)
      for (int t = 0; t < NR; ++t) task(i, t, true);
  }
  if (NR == 0 && tid == 0) *sent_steps = base + p.iters;
  tr.rec(kEvEnd, base + p.iters, 0);
}

// SIMPLE receiver role: delivers (AG) or folds the output (RS) of step s, then — once the
// sender role is also done with this step's inbox — publishes done(g) to every rank.
template <int DT, int OP, int KIND>
__device__ void recv_step(const KPlan& p, const Step& s, Waiter& w, int tid, int nthr,
                          volatile uint64_t* sent_steps, Tracer& tr, bool first_step) {
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const char* snd = p.send[s.lr];
  char* out = p.recv[s.lr];
  const uint64_t* myflags = chan_flags(p, s.R, s.c);
  const bool gpu = p.gpu_scope;
  const char* srcs[kMaxArr + 1];
  if constexpr (KIND == kAG) {
    if (out + s.R * Cb != snd) {  // own chunk placement (simulate.cpp:160-165); skipped in place
      srcs[0] = snd + s.off;
      grp_fold<DT, OP>(out + s.R * Cb + s.off, srcs, 1, s.len, p, tid, nthr);
    }
  }
  for (int t = 0; t < p.nrounds; ++t) {
    if (tid == 0) {
      wait_flag(myflags + t, s.g + 1, w);
      if (p.occ && first_step && s.c == p.chan_base) occ_arrived(p, s.lr, t);
    }
    tr.rec(kEvArrived, s.g, t);
    named_bar(2, nthr);
    if constexpr (KIND == kAG) {
      if (!p.direct) {
        const KRound& r = p.rounds[t];
        for (int pos = 0; pos < r.nchunks; ++pos) {
          const int j = r.slot_base + pos;
          const int origin = (s.R - p.slot_offset[j] + n) % n;
          srcs[0] = slot_ptr(p, s.R, s.c, s.buf, j);
          grp_fold<DT, OP>(out + origin * Cb + s.off, srcs, 1, s.len, p, tid, nthr);
        }
      }
    }
  }
  if constexpr (KIND == kRS) {
    int m = 0;
    srcs[m++] = snd + s.R * Cb + s.off;  // output starts as own contribution (simulate.cpp:239)
    for (int f = 0; f < p.nfin; ++f) srcs[m++] = slot_ptr(p, s.R, s.c, s.buf, p.fin[f]);
    grp_fold<DT, OP>(out + s.off, srcs, m, s.len, p, tid, nthr);
  }
  if (tid == 0) {  // the sender role must be done reading this step's inbox too
    uint64_t start = 0;
    uint32_t spins = 0;
    while (*sent_steps < s.g + 1 && !w.aborted) {
      if ((++spins & 1023u) == 0) {
        const uint64_t now = globaltimer();
        if (start == 0) start = now;
        else if (now - start > w.timeout_ns) report_timeout(w);
      }
    }
  }
  tr.rec(kEvDelivered, s.g, 0);
  const bool clean = epoch_clean_due(p, s.g);
  if (clean) epoch_clean(p, s.R, s.c, s.g, tid, nthr);
  named_bar(2, nthr);
  if (clean && tid < n) fence_acq_rel(gpu);
  if (tid < n && tid != s.R) st_release(chan_flags(p, tid, s.c) + 8 + s.R, s.g + 1, gpu);
}

// LL: every thread owns the same 8-byte words of the slice in every chunk and round, so it
// only ever waits on lines it polls itself — no CTA barrier inside the step.
template <int DT, int OP, int KIND>
__device__ void step_ll(const KPlan& p, const Step& s, Waiter& w) {
  // leaves first (p.leaves_first): pass 0 pushes every round's chunks that carry no arrival,
  // pass 1 the forwards; otherwise one pass over all positions in round order
  const int passes = p.leaves_first ? 2 : 1;
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const char* snd = p.send[s.lr];
  char* out = p.recv[s.lr];
  const uint32_t flag = static_cast<uint32_t>(s.g + 1);
  const int64_t nlines = (s.len + 7) >> 3;
  const int B = blockDim.x;
  PAT_BOUND(16 * nlines <= p.slot_stride);

  for (int pass = 0; pass < passes; ++pass)
  for (int t = 0; t < p.nrounds; ++t) {
    const KRound& r = p.rounds[t];
    const int P = (s.R + r.peer) % n;
    for (int pos = 0; pos < r.nchunks; ++pos) {
      if (passes == 2 && (r.narr[pos] == 0) != (pass == 0)) continue;
      char* dst = slot_ptr(p, P, s.c, s.buf, r.slot_base + pos);
      if constexpr (KIND == kAG) {
        const char* fwd = r.narr[pos] ? slot_ptr(p, s.R, s.c, s.buf, r.arr[pos][0]) : nullptr;
        for (int64_t q = threadIdx.x; q < nlines; q += B) {
          const int valid = static_cast<int>(min(int64_t{8}, s.len - 8 * q));
          const uint2 v = fwd ? ld_ll(fwd + 16 * q, flag, w) : load_word(snd + s.off + 8 * q, valid, p);
          st_ll(dst + 16 * q, v, flag);
        }
      } else {
        const int dest = (s.R - r.chunk[pos] + n) % n;
        const char* own = snd + dest * Cb + s.off;
        const int na = r.narr[pos];
        for (int64_t q = threadIdx.x; q < nlines; q += B) {
          const int valid = static_cast<int>(min(int64_t{8}, s.len - 8 * q));
          uint2 acc;
          if (na == 0) {
            acc = load_word(own + 8 * q, valid, p);
          } else {
            acc = ld_ll(slot_ptr(p, s.R, s.c, s.buf, r.arr[pos][0]) + 16 * q, flag, w);
            for (int a = 1; a < na; ++a)
              fold_vec<DT, OP>(acc, ld_ll(slot_ptr(p, s.R, s.c, s.buf, r.arr[pos][a]) + 16 * q, flag, w));
            fold_vec<DT, OP>(acc, load_word(own + 8 * q, valid, p));
          }
          st_ll(dst + 16 * q, acc, flag);
        }
      }
    }
  }
  if constexpr (KIND == kAG) {
    // own chunk placement (simulate.cpp:160-165) after every send: local work that would
    // otherwise delay the first line onto the link
    if (out + s.R * Cb != snd)
      for (int64_t q = threadIdx.x; q < nlines; q += B) {
        const int valid = static_cast<int>(min(int64_t{8}, s.len - 8 * q));
        store_word(out + s.R * Cb + s.off + 8 * q, load_word(snd + s.off + 8 * q, valid, p), valid, p);
      }
    for (int j = 0; j < p.nslots; ++j) {
      const int origin = (s.R - p.slot_offset[j] + n) % n;
      const char* slot = slot_ptr(p, s.R, s.c, s.buf, j);
      for (int64_t q = threadIdx.x; q < nlines; q += B) {
        const int valid = static_cast<int>(min(int64_t{8}, s.len - 8 * q));
        store_word(out + origin * Cb + s.off + 8 * q, ld_ll(slot + 16 * q, flag, w), valid, p);
      }
    }
  } else {
    for (int64_t q = threadIdx.x; q < nlines; q += B) {
      const int valid = static_cast<int>(min(int64_t{8}, s.len - 8 * q));
      uint2 acc = load_word(snd + s.R * Cb + s.off + 8 * q, valid, p);
      for (int f = 0; f < p.nfin; ++f)
        fold_vec<DT, OP>(acc, ld_ll(slot_ptr(p, s.R, s.c, s.buf, p.fin[f]) + 16 * q, flag, w));
      store_word(out + s.off + 8 * q, acc, valid, p);
    }
  }
}

// ------------------------------------------------------------------------- LL32 protocol
// 32-byte lines {7 payload words, check word} written with ONE st.volatile.v8 (STG.256) and
// polled with one ld.volatile.v8. The check word is the step's flag XOR a hash of the 7 payload
// words, so a line counts as arrived only when the flag AND the data it was written with are
// both visible: a line that lands in pieces (the flag's 16-byte sector before the data sector —
// PTX promises single-copy atomicity per element, not per 32-byte vector, and LL128's one flag
// per 128 bytes was observed to tear on this fabric) fails the check and is
// polled again instead of being consumed. tools/atomicity_probe.cu never saw a 32-byte store
// land torn (0 of 7.3e9 lines, profiles/r01f_atomicity_g*.txt); the check makes correctness
// independent of that observation. The reference's executor consumes a message only when it is
// complete (Mailbox::incoming, simulate.cpp:131-149); this is that rule per line.
//
// Payload units: a line holds R units of U bytes (U = 4, R = 7; U = 8 for 8-byte reductions so
// every unit is a whole element, R = 3). Lines go in groups of 32 (one per lane): unit r of
// lane l's line is slice bytes [U (32 r + l), +U) of the group, so every row r of a warp's
// loads and stores is one contiguous 32 U-byte access. Lines whose first unit lies past the
// slice end are empty; sender and receiver skip the same ones.
struct Line32 {
  uint32_t w[8];  // w[7] = check word
};

// Hash of a line's payload words: a sum of distinct odd multiples (7 IMADs), so a change of any
// single word always changes it and the all-zero line (a zeroed or re-stamped pool) hashes to 0.
__host__ __device__ __forceinline__ uint32_t line_hash(const Line32& v) {
#ifdef PAT_LL32_NOHASH  // A/B builds only (tools/build_variant.sh): the flag alone, no integrity check
  return 0 * v.w[0];
#endif
  return v.w[0] * 0x9E3779B1u + v.w[1] * 0x85EBCA77u + v.w[2] * 0xC2B2AE3Du + v.w[3] * 0x27D4EB2Fu +
         v.w[4] * 0x165667B1u + v.w[5] * 0xD3A2646Du + v.w[6] * 0xFD7046C5u;
}

__device__ __forceinline__ void st_line32(void* p, const Line32& v) {
  asm volatile("st.volatile.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
               "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
               : "memory");
}
// Seal a line for step flag `flag` and store it.
__device__ __forceinline__ void put_line32(void* p, Line32& v, uint32_t flag) {
  v.w[7] = flag ^ line_hash(v);
  st_line32(p, v);
}
__device__ __forceinline__ Line32 ld_volatile32(const void* p) {
  Line32 v;
  asm volatile("ld.volatile.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                 "=r"(v.w[7])
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ bool line32_ok(const Line32& v, uint32_t flag) { return v.w[7] == (flag ^ line_hash(v)); }
// Poll one line until it is complete for step flag `flag` (check word matches its payload).
__device__ __forceinline__ Line32 ld_line32(const char* line, uint32_t flag, Waiter& w) {
  Line32 v = ld_volatile32(line);
  if (line32_ok(v, flag)) return v;
  uint64_t start = 0;
  uint32_t spins = 0;
  while (!w.aborted) {
    v = ld_volatile32(line);
    if (line32_ok(v, flag)) break;
    if ((++spins & 1023u) == 0) {
      const uint64_t now = globaltimer();
      if (start == 0) start = now;
      else if (now - start > w.timeout_ns) report_timeout(w);
    }
  }
  return v;
}

template <int U>
struct LL32Shape {
  static constexpr int R = U == 4 ? 7 : 3;  // units per line
  static constexpr int G = 32 * R * U;      // payload bytes per group of 32 lines
};

// Units of line (group base `gb`, lane) from a user buffer `p` (slice start). With an aligned
// buffer every unit that starts before `len` is one aligned U-byte load (each row a contiguous
// warp access); the chunk's last unit may extend past `len`, but an aligned unit never crosses a
// page, and those bytes are never stored (store_units) — a fold of them is discarded. Unaligned
// buffers go byte by byte.
template <int U>
__device__ __forceinline__ Line32 load_units(const char* p, int64_t gb, int lane, int64_t len, const KPlan& pl) {
  constexpr int R = LL32Shape<U>::R;
  Line32 v;
#pragma unroll
  for (int k = 0; k < 8; ++k) v.w[k] = 0;
  if (pl.vec >= U) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t off = gb + static_cast<int64_t>(U) * (32 * r + lane);
      if (off < len) {
        if constexpr (U == 4) {
          v.w[r] = *reinterpret_cast<const uint32_t*>(p + off);
        } else {
          const uint2 x = *reinterpret_cast<const uint2*>(p + off);
          v.w[2 * r] = x.x;
          v.w[2 * r + 1] = x.y;
        }
      }
    }
    return v;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t off = gb + static_cast<int64_t>(U) * (32 * r + lane);
    if (off < len) {
      const int valid = static_cast<int>(min(static_cast<int64_t>(U), len - off));
      uint64_t x = 0;
#pragma unroll
      for (int b = 0; b < U; ++b)
        if (b < valid) x |= static_cast<uint64_t>(static_cast<uint8_t>(p[off + b])) << (8 * b);
      if constexpr (U == 4) {
        v.w[r] = static_cast<uint32_t>(x);
      } else {
        v.w[2 * r] = static_cast<uint32_t>(x);
        v.w[2 * r + 1] = static_cast<uint32_t>(x >> 32);
      }
    }
  }
  return v;
}

// Units of a line into a user buffer: whole aligned units as one store, the chunk's last
// partial unit (or an unaligned buffer) byte by byte, never past `len`.
template <int U>
__device__ __forceinline__ void store_units(char* p, const Line32& v, int64_t gb, int lane, int64_t len,
                                            const KPlan& pl) {
  constexpr int R = LL32Shape<U>::R;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t off = gb + static_cast<int64_t>(U) * (32 * r + lane);
    if (off + U <= len && pl.vec >= U) {
      if constexpr (U == 4) *reinterpret_cast<uint32_t*>(p + off) = v.w[r];
      else *reinterpret_cast<uint2*>(p + off) = make_uint2(v.w[2 * r], v.w[2 * r + 1]);
    } else if (off < len) {
      const int valid = static_cast<int>(min(static_cast<int64_t>(U), len - off));
      const uint64_t x = U == 4 ? v.w[r] : (static_cast<uint64_t>(v.w[2 * r + 1]) << 32 | v.w[2 * r]);
#pragma unroll
      for (int b = 0; b < U; ++b)
        if (b < valid) p[off + b] = static_cast<char>((x >> (8 * b)) & 0xff);
    }
  }
}

// a = a (op) b, unit by unit (every unit holds whole elements).
template <int DT, int OP, int U>
__device__ __forceinline__ void fold_line32(Line32& a, const Line32& b) {
  if constexpr (U == 4) {
#pragma unroll
    for (int r = 0; r < 7; ++r) fold_vec<DT, OP>(a.w[r], b.w[r]);
  } else {
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      uint2 x = make_uint2(a.w[2 * r], a.w[2 * r + 1]);
      fold_vec<DT, OP>(x, make_uint2(b.w[2 * r], b.w[2 * r + 1]));
      a.w[2 * r] = x.x;
      a.w[2 * r + 1] = x.y;
    }
  }
}

// One phase of an LL32 pipeline step: phase t in [0, nrounds) sends round t; phase nrounds
// finishes the step (all-gather: own chunk placement and delivery of every slot; reduce-scatter:
// the output fold). The same rounds, slots and fold order as step_ll.
template <int DT, int OP, int KIND, int U>
__device__ void ll32_phase(const KPlan& p, const Step& s, int t, Waiter& w, int part = kAllPos) {
  constexpr int G = LL32Shape<U>::G;
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const char* snd = p.send[s.lr] + s.off;
  char* out = p.recv[s.lr];
  const uint32_t flag = static_cast<uint32_t>(s.g + 1);
  const int64_t nlines = (s.len + G - 1) / G * 32;
  const int B = blockDim.x;
  PAT_BOUND(32 * nlines <= p.slot_stride);
  const int lane = threadIdx.x & 31;

  // lines inner: a round's stores are all in flight before the next round polls its first arrival
#define PAT_LL32_LINES                                       \
  for (int64_t q = threadIdx.x; q < nlines; q += B)          \
    if (const int64_t gb = (q >> 5) * G; gb + U * lane < s.len)
  if (t < p.nrounds) {
    const KRound& r = p.rounds[t];
    const int P = (s.R + r.peer) % n;
    for (int pos = 0; pos < r.nchunks; ++pos) {
      if (part != kAllPos && (r.narr[pos] == 0) != (part == kLeafPos)) continue;
      char* dst = slot_ptr(p, P, s.c, s.buf, r.slot_base + pos);
      if constexpr (KIND == kAG) {
        const char* fwd = r.narr[pos] ? slot_ptr(p, s.R, s.c, s.buf, r.arr[pos][0]) : nullptr;
        PAT_LL32_LINES {
          Line32 v = fwd ? ld_line32(fwd + 32 * q, flag, w) : load_units<U>(snd, gb, lane, s.len, p);
          put_line32(dst + 32 * q, v, flag);
        }
      } else {
        const char* own = snd + ((s.R - r.chunk[pos] + n) % n) * Cb;
        const int na = r.narr[pos];
        PAT_LL32_LINES {
          const Line32 mine = load_units<U>(own, gb, lane, s.len, p);
          Line32 v;
          if (na == 0) {
            v = mine;
          } else {  // fold(arrivals in round order) (+) own (simulate.cpp:257-266, 281-285)
            v = ld_line32(slot_ptr(p, s.R, s.c, s.buf, r.arr[pos][0]) + 32 * q, flag, w);
            for (int a = 1; a < na; ++a)
              fold_line32<DT, OP, U>(v, ld_line32(slot_ptr(p, s.R, s.c, s.buf, r.arr[pos][a]) + 32 * q, flag, w));
            fold_line32<DT, OP, U>(v, mine);
          }
          put_line32(dst + 32 * q, v, flag);
        }
      }
    }
  } else if constexpr (KIND == kAG) {
    if (out + s.R * Cb != p.send[s.lr])  // own chunk placement (simulate.cpp:160-165)
      PAT_LL32_LINES store_units<U>(out + s.R * Cb + s.off, load_units<U>(snd, gb, lane, s.len, p), gb, lane, s.len, p);
    for (int j = 0; j < p.nslots; ++j) {
      const char* slot = slot_ptr(p, s.R, s.c, s.buf, j);
      char* o = out + ((s.R - p.slot_offset[j] + n) % n) * Cb + s.off;
      PAT_LL32_LINES store_units<U>(o, ld_line32(slot + 32 * q, flag, w), gb, lane, s.len, p);
    }
  } else {  // output = own (+) offset-0 arrivals in round order (simulate.cpp:239, 278-279)
    PAT_LL32_LINES {
      Line32 acc = load_units<U>(snd + s.R * Cb, gb, lane, s.len, p);
      for (int f = 0; f < p.nfin; ++f)
        fold_line32<DT, OP, U>(acc, ld_line32(slot_ptr(p, s.R, s.c, s.buf, p.fin[f]) + 32 * q, flag, w));
      store_units<U>(out + s.off, acc, gb, lane, s.len, p);
    }
  }
#undef PAT_LL32_LINES
}

// ------------------------------------------------------------------------- PULL protocol
// The receiver reads. In round t rank R pulls the chunks K_t from its upstream Q = R - peer_t
// (the rank that pushes to it in the reference's send/deliver, simulate.cpp:186-212, 252-290):
//  * all-gather: a leaf chunk comes straight from Q's sendbuf, a forwarded one from Q's recvbuf
//    (where Q itself delivered it) — zero copy on both sides, no staging at all;
//  * reduce-scatter: a leaf is Q's own contribution (Q's sendbuf); a forwarded offset is Q's
//    staged message fold(arrivals) (+) own, which Q finalised when it pulled the last arrival.
//    R folds what it pulls into its output or into its own staging slot (PullAct).
// Every NVLink byte is a read of the peer's HBM (measured 775 GB/s vs 714 GB/s for pushed
// stores, profiles/r01_p2p_probe_*.txt). Flags: after finishing round tr of a step, Q tells each
// reader whose round t'' depends on round tr (sig_after) by a store into the reader's flags;
// readers publish done(step) to every rank, which is the staging credit (RS) and the exit
// condition: a rank leaves the call only once its readers are done with its buffers.

template <int DT, int OP, int KIND>
__device__ __forceinline__ void pull_task(const KPlan& p, const Step& s, int t, int tid, int nthr) {
  const int n = p.n;
  const int64_t Cb = p.chunk_bytes;
  const KRound& r = p.rounds[t];
  const int Q = (s.R - r.peer + n) % n;
  char* out = p.recv[s.lr];
  const char* own = p.send[s.lr];
  const char* srcs[3];
  for (int pos = 0; pos < r.nchunks; ++pos) {
    const int k = r.chunk[pos];              // offset at the sender Q
    const int at = (Q - k + n) % n;          // AG: origin; RS: destination of the contribution
    if constexpr (KIND == kAG) {
      srcs[0] = r.narr[pos] == 0 ? p.peer_send[Q] + s.off : p.peer_recv[Q] + at * Cb + s.off;
      grp_fold<DT, OP>(out + at * Cb + s.off, srcs, 1, s.len, p, tid, nthr);
    } else {
      const char* m = r.narr[pos] == 0 ? p.peer_send[Q] + at * Cb + s.off
                                       : acc_ptr(p, Q, s.c, s.buf, p.pull_dst[r.arr[pos][r.narr[pos] - 1]]);
      const int j = r.slot_base + pos;
      const int kr = p.slot_offset[j];                  // received offset at R
      const char* mine = own + ((s.R - kr + n) % n) * Cb + s.off;
      char* stage = p.pull_dst[j] >= 0 ? acc_ptr(p, s.R, s.c, s.buf, p.pull_dst[j]) : nullptr;
      char* dst = stage;
      int cnt = 2;
      switch (p.pull_act[j]) {
        case kOutFirst: dst = out + s.off; srcs[0] = mine; srcs[1] = m; break;
        case kOutNext: dst = out + s.off; srcs[0] = dst; srcs[1] = m; break;
        case kAccOnly: srcs[0] = m; srcs[1] = mine; break;
        case kAccFirst: srcs[0] = m; cnt = 1; break;
        case kAccMid: srcs[0] = stage; srcs[1] = m; break;
        default: srcs[0] = stage; srcs[1] = m; srcs[2] = mine; cnt = 3; break;  // kAccLast
      }
      grp_fold<DT, OP>(dst, srcs, cnt, s.len, p, tid, nthr);
    }
  }
}

template <int DT, int OP, int KIND>
__device__ void pull_role(const KPlan& p, uint64_t base, int R, int lr, int c, Waiter& w) {
  const int n = p.n, NR = p.nrounds, L = p.skew;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool gpu = p.gpu_scope != 0;
  uint64_t* myflags = chan_flags(p, R, c);
  __shared__ int s_abort;
  // entry: my sendbuf (and, for AG, recvbuf) are final once this stream reached the call
  if (tid < n && tid != R) {
    sym_publish(p, R, c, tid, gpu);
    st_release(chan_flags(p, tid, c) + 16 + R, base + 1, gpu);
  }
  if (tid == 0) {
    bool ok = true;
    for (int t = 0; t < NR; ++t) {
      const int Q = (R - p.rounds[t].peer + n) % n;
      wait_flag(myflags + 16 + Q, base + 1, w);
      ok = sym_check(p, R, c, Q, w) && ok;
    }
    s_abort = !ok;
  }
  __syncthreads();
  if (s_abort) return;
  auto task = [&](int i, int t) {
    const Step s = make_step(p, base, i, R, lr, c);
    if (tid == 0) {
      // RS: staging buffer s.buf is free once every reader finished step g - depth
      if (KIND == kRS && ((p.stage_rounds >> t) & 1) && s.g >= static_cast<uint64_t>(p.depth))
        for (int q = 0; q < n; ++q)
          if (q != R) wait_flag(myflags + 8 + q, s.g - p.depth + 1, w);
      if (p.round_dep[t] >= 0) wait_flag(myflags + t, s.g + 1, w);
    }
    if constexpr (KIND == kAG) {  // own chunk placement (simulate.cpp:160-165), skipped in place
      if (t == 0 && p.recv[lr] + R * p.chunk_bytes != p.send[lr]) {
        const char* src[1] = {p.send[lr] + s.off};
        grp_fold<DT, OP>(p.recv[lr] + R * p.chunk_bytes + s.off, src, 1, s.len, p, tid, nthr);
      }
    }
    __syncthreads();
    pull_task<DT, OP, KIND>(p, s, t, tid, nthr);
  };
  // after the fence: readers of round t (sig_after) and, after the last round, done(step)
  auto signal = [&](int i, int t) {
    const uint64_t g1 = base + i + 1;
    for (int t2 = 0; t2 < NR; ++t2)
      if ((p.sig_after[t] >> t2) & 1) st_relaxed(chan_flags(p, (R + p.rounds[t2].peer) % n, c) + t2, g1, gpu);
    if (t == NR - 1)
      for (int q = 0; q < n; ++q)
        if (q != R) st_relaxed(chan_flags(p, q, c) + 8 + R, g1, gpu);
  };
  // before done(step i) (signal of the last round): the step's epoch re-stamp, if due
  auto clean = [&](int i) {
    if (epoch_clean_due(p, base + i)) epoch_clean(p, R, c, base + i, tid, nthr);
  };
  if (L > 0) {  // skewed: round t of step k - t*L in iteration k, one fence per iteration
    for (int k = 0; k < p.iters + (NR - 1) * L; ++k) {
      for (int t = 0; t < NR; ++t)
        if (k - t * L >= 0 && k - t * L < p.iters) task(k - t * L, t);
      if (k - (NR - 1) * L >= 0 && k - (NR - 1) * L < p.iters) clean(k - (NR - 1) * L);
      __syncthreads();
      if (tid == 0) {
        fence_acq_rel(gpu);
        for (int t = NR - 1; t >= 0; --t)
          if (k - t * L >= 0 && k - t * L < p.iters) signal(k - t * L, t);
      }
    }
  } else {
    for (int i = 0; i < p.iters; ++i)
      for (int t = 0; t < NR; ++t) {
        task(i, t);
        if (t == NR - 1) clean(i);
        __syncthreads();
        if (tid == 0) {
          fence_acq_rel(gpu);
          signal(i, t);
        }
      }
  }
  // exit: every reader is done with my buffers (sendbuf, recvbuf, staging) for this call
  if (tid < n && tid != R) wait_flag(myflags + 8 + tid, base + p.iters, w);
}

// One CTA of a call: virtual block vb in [0, nlocal * channels) runs channel chan_base + vb %
// channels of local rank vb / channels.
template <int DT, int OP, int KIND>
__device__ __forceinline__ void pat_body(const KPlan& p, int vb) {
  const int lr = vb / p.channels;
  const int c = p.chan_base + (vb - lr * p.channels);
  const int R = p.rank[lr];
  __shared__ uint64_t s_base;
  __shared__ volatile uint64_t s_sent;
  // programmatic dependent launch (kernels.cu): this grid may be scheduled while its
  // predecessor on the stream drains; it touches memory only once that grid completed and
  // flushed. No early launch_dependents: a successor made resident early would take registers
  // from this grid's later CTAs (measured: the fused reduce-scatter lost half its occupancy).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the step counter and the first step's credits are read at the same time (threads 0 and
  // 1..npeers): the credit loads' addresses do not depend on the counter, only the comparison does
  __shared__ uint64_t s_cred[kMaxRounds];
  if (threadIdx.x == 0) {
    s_base = p.iter_state[lr][c];
    s_sent = 0;
  } else if (static_cast<int>(threadIdx.x) <= p.npeers) {
    const int k = threadIdx.x - 1;
    s_cred[k] = ld_acquire(chan_flags(p, R, c) + 8 + (R + p.peers[k]) % p.n, p.gpu_scope != 0);
  }
  __syncthreads();
  const uint64_t base = s_base;
  Waiter w{p.timeout_ns, p.err, false, p.gpu_scope != 0};
#ifndef PAT_NO_CRED0  // A/B builds: the first step's credits waited for as every later step's
  w.cred0 = s_cred;
#endif
  w.base = base;

  // done(step) for the previous call's last step on this channel: a polling-protocol call defers
  // it from its exit (below), and EVERY protocol publishes it here — a bulk call that follows a
  // polling one needs it, or its sender's credit for step base + depth - 1 (which the skew allows
  // to wait on step base - 1) would wait on the peer's receiver, itself waiting on this sender.
  // Every step before `base` finished: the previous kernel completed before this one started.
  if (threadIdx.x < p.n && static_cast<int>(threadIdx.x) != R)
    st_relaxed(chan_flags(p, threadIdx.x, c) + 8 + R, base, w.gpu);
  // SIMPLE / PULL publish later done values from other threads: a barrier orders this store before
  // them (release cumulativity). The polling protocols' later done stores come from these same
  // threads (program order), and their first barrier follows the credit wait.
  const bool polling = p.proto == kProtoLL || p.proto == kProtoLL32;
  if (!polling || PAT_EXTRA_BARRIERS) __syncthreads();

  if (p.direct && KIND == kAG) {
    // entry handshake: a peer may be written directly only once it entered this call
    __shared__ int s_abort;
    if (threadIdx.x < p.n && static_cast<int>(threadIdx.x) != R) {
      sym_publish(p, R, c, threadIdx.x, w.gpu);
      st_release(chan_flags(p, threadIdx.x, c) + 16 + R, base + 1, w.gpu);
    }
    if (threadIdx.x == 0) {
      bool ok = true;
      for (int k = 0; k < p.npeers; ++k) {
        const int P = (R + p.peers[k]) % p.n;
        wait_flag(chan_flags(p, R, c) + 16 + P, base + 1, w);
        ok = sym_check(p, R, c, P, w) && ok;
      }
      s_abort = !ok;
    }
    __syncthreads();
    if (s_abort) return;
  }

  if (p.proto == kProtoPull) {
    pull_role<DT, OP, KIND>(p, base, R, lr, c, w);
  } else if (p.proto == kProtoLL || p.proto == kProtoLL32) {
    // 8-byte reductions use 8-byte LL32 units (whole elements); everything else 4-byte units
    constexpr int U = KIND == kRS && sizeof(typename DType<DT>::S) == 8 ? 8 : 4;
    // Steps in order. (A wavefront — phase t of step k - t in iteration k, as send_role — was
    // built and measured slower: LL32 is bound by the polled lines' bandwidth, not by flight
    // times; profiles/r01f_ll32_{skew,noskew}_n*.jsonl.)
    // PAT_TRACE in a -DPAT_TRACE_POLL=1 build (tools/build_variant.sh; compiled out by default, so
    // the polling path's code is unchanged): thread 0's view (role 1): start, credits in, each LL32
    // phase done (round t: its lines sent and, for t > 0, its arrivals of round t-1 consumed), end
    Tracer tr;
    if (PAT_TRACE_POLL && threadIdx.x == 0) tr.init(p, 1);
    tr.rec(kEvStart, base, 0);
    for (int i = 0; i < p.iters; ++i) {
      const Step s = make_step(p, base, i, R, lr, c);
      wait_credits_par(p, s, w, threadIdx.x);
      __syncthreads();
      tr.rec(kEvCredit, s.g, 0);
      if (p.proto == kProtoLL) {
        step_ll<DT, OP, KIND>(p, s, w);
        tr.rec(kEvDelivered, s.g, 0);
      } else {
        if (p.leaves_first) {  // every round's leaf lines, then the forwards, then the finish
          for (int t = 0; t < p.nrounds; ++t) ll32_phase<DT, OP, KIND, U>(p, s, t, w, kLeafPos);
          for (int t = 0; t < p.nrounds; ++t) ll32_phase<DT, OP, KIND, U>(p, s, t, w, kFwdPos);
          ll32_phase<DT, OP, KIND, U>(p, s, p.nrounds, w);
          tr.rec(kEvDelivered, s.g, p.nrounds);
        } else {
          for (int t = 0; t <= p.nrounds; ++t) {
            ll32_phase<DT, OP, KIND, U>(p, s, t, w);
            tr.rec(t < p.nrounds ? kEvPushed : kEvDelivered, s.g, t);
          }
        }
      }
      const bool clean = epoch_clean_due(p, s.g);
      if (clean) {  // every load of this step's lines returned before the barrier above it
        __syncthreads();
        epoch_clean(p, R, c, s.g, threadIdx.x, blockDim.x);
      }
      __syncthreads();
      if (clean && threadIdx.x < p.n) fence_acq_rel(w.gpu);
      // done(step): every load of this step's inbox has returned (its value was consumed before
      // the barrier), so a relaxed store suffices to hand the buffers back. The last step's is
      // published by the next call's kernel (above): a remote store at exit would hold the
      // grid's completion for its NVLink acknowledgement, and no sender needs it earlier — the
      // first step of the next call waits for step base - depth + 1 <= base - 1 (depth >= 2).
      if (i + 1 < p.iters && threadIdx.x < p.n && static_cast<int>(threadIdx.x) != R)
        st_relaxed(chan_flags(p, threadIdx.x, c) + 8 + R, s.g + 1, w.gpu);
    }
    tr.rec(kEvEnd, base + p.iters, 0);
  } else {
    const int nsend = p.send_warps * 32;
    if (static_cast<int>(threadIdx.x) < nsend) {
      send_role<DT, OP, KIND>(p, base, R, lr, c, w, threadIdx.x, nsend, &s_sent);
    } else {
      const int tid = threadIdx.x - nsend, nrecv = blockDim.x - nsend;
      Tracer tr;
      if (tid == 0) tr.init(p, 1);
      tr.rec(kEvStart, base, 0);
      for (int i = 0; i < p.iters; ++i) {
        const Step s = make_step(p, base, i, R, lr, c);
        recv_step<DT, OP, KIND>(p, s, w, tid, nrecv, &s_sent, tr, i == 0);
      }
      tr.rec(kEvEnd, base + p.iters, 0);
    }
  }
  // thread 0 advances the step counter; the next call reads it only after this grid completed, so
  // no barrier is needed before it
  if (PAT_EXTRA_BARRIERS) __syncthreads();
  if (threadIdx.x == 0) p.iter_state[lr][c] = base + p.iters;
}

template <int DT, int OP, int KIND>
__global__ void __launch_bounds__(kMaxThreads) pat_kernel(const __grid_constant__ KPlan p) {
  pat_body<DT, OP, KIND>(p, blockIdx.x);
}

// A grouped all-gather + reduce-scatter (patGroupStart/End) in one launch: the two calls run
// side by side on disjoint channels, so their latencies overlap instead of adding up.
template <int DT>
__global__ void __launch_bounds__(kMaxThreads) pat_group_kernel(const __grid_constant__ KPlan2 p) {
  const int na = p.a.nlocal * p.a.channels;
  if (static_cast<int>(blockIdx.x) < na) pat_body<kU8, kSum, kAG>(p.a, blockIdx.x);
  else pat_body<DT, kSum, kRS>(p.b, blockIdx.x - na);
}

}  // namespace pat
