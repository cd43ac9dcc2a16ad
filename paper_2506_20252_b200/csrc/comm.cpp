// comm.cpp — host runtime behind include/pat_b200.h.
//
// A communicator owns, for every rank it drives, one inbox pool in that rank's HBM
// (flags + channels * 2 * (n-1) slots) and maps every other rank's pool into each of its
// devices' address spaces: legacy peer access between devices of this process
// (patCommInitAll) or CUDA IPC between processes (patCommInitRank*). A collective compiles
// the PAT schedule for (kind, T) once, picks the protocol and slicing from the chunk size,
// and launches ONE cooperative kernel per device covering all ranks on that device.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <unistd.h>
#include <vector>

#include "../../include/pat_b200.h"
#include "launch_worker.hpp"
#include "plan.hpp"
#include "schedule.hpp"

namespace pat {
using KernelFn = void (*)(const KPlan);
cudaError_t launch(const KPlan& plan, int dtype, int op, int threads, cudaStream_t stream);
cudaError_t launch_barrier(const BPlan& b, cudaStream_t stream);
cudaError_t launch_group(const KPlan2& plans, int dtype, int threads, cudaStream_t stream);
cudaError_t launch_local_group(int n, int dtype, int64_t a_bytes, const char* const* a_send, char* const* a_recv,
                               int64_t b_bytes, const char* const* b_send, char* const* b_recv, int sm_count,
                               cudaStream_t stream);
cudaError_t max_blocks_per_sm(int kind, int dtype, int op, int threads, int* out);
cudaError_t init_pool_state(char* pool, int64_t ll_off, int64_t ll_bytes, int64_t ll32_off, int64_t ll32_bytes,
                            uint64_t start, cudaStream_t stream);
cudaError_t fill_u64(uint64_t* p, int64_t n, uint64_t v, cudaStream_t stream);
cudaError_t launch_local(int kind, int n, int dtype, int op, int vec, int esize, int64_t chunk_bytes,
                         const char* const* send_by_rank, char* const* recv_by_rank, int sm_count,
                         cudaStream_t stream);
const char* local_tree_string(int n);
}  // namespace pat

using namespace pat;

namespace {

// per pool: channel flags (8 KiB), then the barrier words (patCommBarrier), padded so the
// inbox regions stay 4 KiB aligned
constexpr size_t kChanFlagBytes = sizeof(uint64_t) * kMaxChannels * kFlagWords;  // 40 KiB
constexpr size_t kBarrierOff = kChanFlagBytes;
constexpr size_t kFlagBytes = kChanFlagBytes + 4096;
constexpr uint32_t kMagic = 0x50415442;                                       // "PATB"
constexpr size_t kDefaultPoolBytes = 512ull << 20;  // inbox pool budget per rank (all channels)
constexpr size_t kMaxSlice = 256 << 10;
constexpr size_t kCapMinSlice = 32 << 10;  // smallest bulk slice a staging cap shrinks to before channels
constexpr int kDefaultChannels = 148;            // one CTA per SM of a B200; clamped to co-residency at launch
// LL32 vs bulk is chosen by the calibrated cost model below (choose_slicing).
constexpr int64_t kPullMaxRS = 128 << 20;  // PULL reduce-scatter below this chunk size
constexpr int64_t kPullMinRS = 1 << 20;    // ... and above this one (LL wins below anyway)
constexpr size_t kLLSlotBytes = 32 << 10;  // LL slot: 16 KiB payload per channel-step
// LL32 slot (28/32 of it payload per channel-step); PAT_LL32_SLOT overrides (experiments)
size_t ll32_slot_default() {
  static const size_t v = [] {
    const char* e = std::getenv("PAT_LL32_SLOT");
    const long long x = e ? std::atoll(e) : 0;
    return x >= 1024 ? static_cast<size_t>(x) & ~size_t(1023) : size_t(32) << 10;
  }();
  return v;
}
constexpr int kDefaultTimeoutMs = 20000;

struct Compiled {
  Schedule sched;
  KPlan proto;  // schedule part of the plan (rounds, slots, fin, peers)
  int peak_slots = 0;
  bool fused_ok = false;  // the fused single-device executor computes exactly this schedule
};

struct DevGroup {
  int device = 0;
  std::vector<int> lidx;           // local indices on this device
  uint64_t* iter_state = nullptr;  // [lidx.size()][kMaxChannels]
  uint64_t* trace = nullptr;       // PAT_TRACE: [lidx.size() * kMaxChannels][2 roles][cap][2]
  int trace_cap = 0;
  int trace_ctas = 0;              // CTAs of the last traced launch
  int* occ = nullptr;              // PAT_STATS: [lidx.size()][2][kMaxRounds] live occupancy counters
  int occ_rounds = -1;             // rounds of the last SIMPLE launch that filled them
  int sm_count = 0;
  std::array<char*, kMaxRanks> pool_view{};  // every rank's pool as seen from this device
  // calls of one communicator run in issue order on each device even across streams (NCCL's
  // guarantee; concurrent calls would share channels): recorded after every eager launch, waited
  // on by the next call when it comes on another stream
  cudaEvent_t order_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
};

struct Handle {
  uint32_t magic, version;
  int32_t nranks, rank, device, channels, pid, pad;
  uint64_t pool_bytes, slot_bytes;
  uint64_t config_hash;  // every resolved setting that decides a call's protocol, slicing or layout
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(Handle) <= PAT_HANDLE_BYTES, "handle too large");

// Registration blob of one symmetric window (patCommRegisterPrepare).
struct RegHandle {
  uint32_t magic, version;
  int32_t nranks, rank;
  uint64_t bytes;   // window size (equal on every rank)
  uint64_t offset;  // window start within its allocation (the IPC handle names the allocation)
  uint64_t config_hash;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(RegHandle) <= PAT_HANDLE_BYTES, "registration handle too large");

bool env_int(const char* name, long long* out) {
  const char* v = std::getenv(name);
  if (!v || !*v) return false;
  *out = std::atoll(v);
  return true;
}

}  // namespace

struct patComm {
  // PAT_HOST_PROFILE=1: host nanoseconds spent planning vs submitting calls (printed at destroy)
  bool host_profile = false;
  uint64_t hp_calls = 0, hp_plan_ns = 0, hp_submit_ns = 0;
  int n = 0;
  patConfig_t cfg{};
  bool multiprocess = false;
  bool finished = false;
  std::vector<int> lranks, ldevs;    // per local index
  std::vector<char*> owned_pool;     // per local index
  std::vector<DevGroup> groups;
  std::vector<void*> ipc_opened;
  // symmetric windows (multi-process zero copy): local range, the peers' matching ranges
  struct Window {
    char* local = nullptr;
    size_t bytes = 0;
    uint32_t id = 0;
    std::array<char*, kMaxRanks> peer{};
    std::array<std::string, kMaxRanks> key{};  // ipc_cache key of each peer's mapping
  };
  std::vector<Window> windows;
  uint32_t next_window = 1;
  std::map<std::string, std::pair<char*, int>> ipc_cache;  // IPC handle bytes -> (base, refs)
  size_t slot_bytes = 0, pool_bytes = 0;
  size_t ll_slot_bytes = 0;                // LL inbox slot (own region, common_init)
  size_t ll32_slot_bytes = 0;              // LL32 inbox slot (own region)
  size_t region_off[kNumProtoSlots] = {};  // inbox region of each protocol within a pool
  size_t region_bytes[kNumProtoSlots] = {};
  int region_channels[kNumProtoSlots] = {};  // channels each protocol region is laid out for
  int depth_poll = 0;                        // inbox buffers per channel of the LL / LL32 regions
  // Pools are allocated lazily for one-process communicators: a communicator whose ranks all
  // sit on one device runs PAT calls through the fused executor (local.cu), which needs no
  // inbox, so its pools appear only if a transport launch ever happens.
  bool pools_ready = false;
  size_t pools_allocated = 0;  // bytes of inbox pool this process allocated (all its ranks)
  int64_t pull_slice = 0;  // all-gather PULL slice (no staging, so not bounded by the slots)
  int skew = 1;            // SIMPLE / PULL sender skew distance (PAT_SKEW; 0 = rounds in order)
  int leaves_first = -1;   // push senders send every round's leaf chunks first (PAT_LEAVES_FIRST:
                           // 1 always, 0 never, default: single-step SIMPLE calls only)
  uint64_t epoch_mask = (1ull << 31) - 1;  // LL / LL32 flag epochs (PAT_EPOCH_SHIFT, tests)
  uint64_t iter_start = 0;                 // first pipeline step of every channel (PAT_ITER_START, tests)
  uint64_t barrier_seq = 0;                // patCommBarrier calls so far
  int channels = 0;
  uint64_t config_hash = 0;  // config_fingerprint(): must be equal on every process of a comm
  int* err_host = nullptr;
  int* err_dev = nullptr;
  std::map<std::vector<int32_t>, Compiled> compiled;  // keyed by schedule encoding
  std::map<int, Compiled*> pat_cache;                  // kind*64 + trees -> compiled PAT
  std::map<std::array<int, 5>, int> occupancy;
  std::vector<cudaEvent_t> events;   // per local index
  std::vector<std::unique_ptr<LaunchWorker>> workers;  // groups[1..] of a one-process comm
  std::mutex mu;
};

namespace {

#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::fprintf(stderr, "pat_b200: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(e_), \
                   __FILE__, __LINE__);                                                    \
      return patUnhandledCudaError;                                                        \
    }                                                                                      \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

patResult_t to_result(Err e) { return static_cast<patResult_t>(e); }

// cudaMalloc (legacy) allocations are reachable from every peer-enabled device; VMM /
// stream-ordered pool memory is not, so zero-copy is only auto-enabled for the former.
bool legacy_ipc_capable(const void* ptr) {
  using Fn = int (*)(void*, int, unsigned long long);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<Fn>(nullptr);
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) return false;
  int v = 0;
  constexpr int kIsLegacyIpcCapable = 10;  // CU_POINTER_ATTRIBUTE_IS_LEGACY_CUDA_IPC_CAPABLE
  if (fn(&v, kIsLegacyIpcCapable, reinterpret_cast<unsigned long long>(ptr)) != 0) return false;
  return v != 0;
}

// Base of the allocation holding `ptr` (cuMemGetAddressRange through the runtime's driver
// entry point, so the library links no libcuda).
bool allocation_base(const void* ptr, char** base, size_t* size) {
  using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<Fn>(nullptr);
    return reinterpret_cast<Fn>(f);
  }();
  unsigned long long b = 0;
  size_t sz = 0;
  if (!fn || fn(&b, &sz, reinterpret_cast<unsigned long long>(ptr)) != 0) return false;
  *base = reinterpret_cast<char*>(b);
  *size = sz;
  return true;
}

size_t dtype_size(int dt) {
  switch (dt) {
    case patInt8: case patUint8: return 1;
    case patFloat16: case patBfloat16: return 2;
    case patInt32: case patUint32: case patFloat32: return 4;
    case patInt64: case patUint64: case patFloat64: return 8;
    default: return 0;
  }
}

// Pool layout. Each protocol has its own inbox region, laid out [channel][buffer][slot]:
//   SIMPLE  channels x depth x (n-1) landing slots x slice     (one slot per arrival of a step)
//   PULL    the SIMPLE region re-cut as channels x depth x A x pslice, A = accumulators of the
//           schedule (internal nodes of the PAT reduction tree: 3 at n = 8) — the reference's
//           intermediate slots; leaves are read straight from the peers' sendbufs
//   LL      ll_channels x depth x (n-1) x 32 KiB              (16-byte lines, half payload)
//   LL32    channels x depth x (n-1) x 32 KiB                 (32-byte lines, 28/32 payload)
// The polling protocols poll their lines, so each has its own memory: a stale payload word left
// by another protocol could otherwise pass for a flag. Without a cap the bulk region takes
// kDefaultPoolBytes; under patConfig_t::staging_bytes (the whole pool, flags aside) the polling
// regions get at most a quarter and the bulk region the rest, with fewer channels rather than
// slices below kCapMinSlice (large slices amortise the per-round fence and flag).
constexpr int kLLChannels = 32;  // LL runs to 256 KiB chunks: 32 x 16 KiB payload per step covers them
struct Layout {
  int ch[kNumProtoSlots] = {};
  size_t slot[kNumProtoSlots] = {};
  size_t bytes[kNumProtoSlots] = {};
};

// Channels and slot size for a region of `budget` bytes: `slot_pref` per slot if it fits with
// `ch_max` channels, else smaller slots down to `slot_min`, then fewer channels.
void fit_region(size_t budget, int ch_max, size_t per_ch_slots, size_t slot_pref, size_t slot_min, size_t align,
                int* ch, size_t* slot) {
  size_t s = budget / (static_cast<size_t>(ch_max) * per_ch_slots);
  s = std::min(s, slot_pref) / align * align;
  if (s >= slot_min) {
    *ch = ch_max;
    *slot = s;
    return;
  }
  const size_t c = budget / (per_ch_slots * slot_min);
  if (c >= 1) {
    *ch = static_cast<int>(std::min<size_t>(c, ch_max));
    *slot = std::min(slot_pref, budget / (static_cast<size_t>(*ch) * per_ch_slots)) / align * align;
    return;
  }
  *ch = 1;
  *slot = std::max(align, budget / per_ch_slots / align * align);
}

Layout plan_layout(const patConfig_t& c, int n, int depth_poll, bool explicit_slice) {
  Layout L;
  const size_t slots = static_cast<size_t>(std::max(n - 1, 1));
  const size_t ll_pref = kLLSlotBytes, ll32_pref = ll32_slot_default();
  const int ch_ll = std::min(c.max_channels, kLLChannels);
  const size_t poll_default = static_cast<size_t>(ch_ll) * depth_poll * slots * ll_pref +
                              static_cast<size_t>(c.max_channels) * depth_poll * slots * ll32_pref;
  size_t bulk_budget = kDefaultPoolBytes, poll_budget = poll_default;
  if (c.staging_bytes != 0) {
    const size_t B = c.staging_bytes > kFlagBytes + 3 * 4096 ? c.staging_bytes - kFlagBytes - 3 * 4096 : 0;
    // Under a cap the polling regions get up to 90% of the pool (never more than their uncapped
    // size), the bulk region the rest: with a small pool LL32 — no fence per step — sustains far
    // more than SIMPLE, whose per-iteration fence stalls the few channels a small pool leaves it
    // (n = 4, ZeRO-3 shape, 12 / 32 / 64 MiB caps: LL32 325 / 530 / 523 GB/s busbw against SIMPLE
    // 177 / 408 / 489, profiles/r02_capped_ll32_vs_simple.jsonl). PAT_POLL_SHARE overrides (percent).
    long long pct = 90;
    if (env_int("PAT_POLL_SHARE", &pct)) pct = std::min(95LL, std::max(5LL, pct));
    poll_budget = std::min(poll_default, B / 100 * static_cast<size_t>(pct));
    bulk_budget = B - poll_budget;
  }
  // LL gets a fifth of the polling budget (it serves chunks up to 256 KiB), LL32 the rest (LL32
  // carries up to 48 MiB per call uncapped, any size under a cap)
  const size_t ll_budget = c.staging_bytes != 0 ? poll_budget / 5 : poll_budget / 4;
  fit_region(ll_budget, ch_ll, depth_poll * slots, ll_pref, 1024, 1024, &L.ch[kProtoLL], &L.slot[kProtoLL]);
  fit_region(poll_budget - ll_budget, c.max_channels, depth_poll * slots, ll32_pref, 1024, 1024,
             &L.ch[kProtoLL32], &L.slot[kProtoLL32]);
  if (explicit_slice && c.staging_bytes == 0) {
    L.ch[kProtoSimple] = c.max_channels;
    L.slot[kProtoSimple] = c.slice_bytes;
  } else {
    // under a cap, slices shrink to kCapMinSlice before channels are dropped (PAT_MIN_SLICE)
    long long ms = 0;
    const size_t min_slice = env_int("PAT_MIN_SLICE", &ms) && ms >= 1024 ? static_cast<size_t>(ms) : kCapMinSlice;
    fit_region(bulk_budget, c.max_channels, c.depth * slots, kMaxSlice, std::min(min_slice, kMaxSlice), 128,
               &L.ch[kProtoSimple], &L.slot[kProtoSimple]);
  }
  L.ch[kProtoPull] = L.ch[kProtoSimple];
  L.slot[kProtoPull] = L.slot[kProtoSimple];  // re-cut per call by the schedule's accumulator count
  L.bytes[kProtoSimple] = L.bytes[kProtoPull] = static_cast<size_t>(L.ch[kProtoSimple]) * c.depth * slots * L.slot[kProtoSimple];
  for (int p : {kProtoLL, kProtoLL32})
    L.bytes[p] = static_cast<size_t>(L.ch[p]) * depth_poll * slots * L.slot[p];
  return L;
}

void fill_defaults(patConfig_t* c, int n) {
  long long v;
  if (c->max_channels <= 0) c->max_channels = env_int("PAT_CHANNELS", &v) ? (int)v : kDefaultChannels;
  c->max_channels = std::min(std::max(c->max_channels, 1), kMaxChannels);
  // one inbox buffer per PAT round of the full-aggregation schedule, plus one: the skewed
  // sender keeps ceil(log2 n) steps in flight (kernels.cu, send_role)
  if (c->depth <= 0) c->depth = env_int("PAT_DEPTH", &v) ? (int)v : ceil_log2(std::max(n, 2)) + 1;
  // at least 2: the polling protocols publish a call's last done(step) only when the next call
  // starts (transport.cuh), which a first step waiting for step base - depth + 1 must not need
  c->depth = std::min(std::max(c->depth, 2), 16);
  // SIMPLE slice: explicit (config or PAT_SLICE_BYTES), else sized from the pool budget by
  // plan_layout (large slices amortise the per-round fence + flag: 85 KiB -> 256 KiB slices
  // lifted n=4 all-gather from ~460 to ~660 GB/s)
  if (c->slice_bytes == 0 && env_int("PAT_SLICE_BYTES", &v) && v > 0) c->slice_bytes = (size_t)v;
  if (c->slice_bytes) c->slice_bytes = std::max<size_t>(256, c->slice_bytes & ~size_t(127));
  if (c->ll_threshold == 0 && env_int("PAT_LL_THRESHOLD", &v)) c->ll_threshold = (size_t)v;  // 0: cost model
  if (c->timeout_ms <= 0) c->timeout_ms = env_int("PAT_TIMEOUT_MS", &v) ? (int)v : kDefaultTimeoutMs;
  if (c->protocol == patProtoAuto && env_int("PAT_PROTOCOL", &v)) c->protocol = (int)v;
  if (c->threads <= 0) c->threads = env_int("PAT_THREADS", &v) ? (int)v : 512;
  c->threads = std::min(std::max(c->threads / 32 * 32, 64), kMaxThreads);
  if (c->direct == 0 && env_int("PAT_DIRECT", &v)) c->direct = (int)v;
  if (c->fused == 0 && env_int("PAT_FUSED", &v)) c->fused = (int)v;
  if (c->send_warps <= 0) c->send_warps = env_int("PAT_SEND_WARPS", &v) ? (int)v : c->threads / 64;
  c->send_warps = std::min(std::max(c->send_warps, 1), c->threads / 32 - 1);
}

// Symbolic run of a reduce-scatter schedule with the executor's fold rules
// (simulate.cpp:237-290): returns rank 0's output as an expression over x_j = contribution of
// rank j, accumulator as left operand, e.g. "((x0+x1)+(x3+x2))" for PAT at n = 4. Rank 0
// stands for every rank: schedules are translation invariant (schedule.hpp:56-63).
std::string symbolic_reduce_scatter(const Schedule& s) {
  const int n = s.n;
  // expressions over absolute contributions c(src, dest) -> only dest == rank-local matter;
  // track every rank, then read rank 0 where c(src, 0) = x_src.
  std::vector<std::string> out(n);
  std::vector<std::map<int, std::string>> acc(n);
  auto own = [&](int src, int dest) { return "c" + std::to_string(src) + "_" + std::to_string(dest); };
  for (int r = 0; r < n; ++r) out[r] = own(r, r);
  for (const Round& rd : s.rounds) {
    if (rd.exchange) return "";
    std::vector<std::vector<std::string>> msgs(n);
    for (int r = 0; r < n; ++r)
      for (int k : rd.chunks) {
        const int dest = mod_ranks(int64_t{r} - k, n);
        auto it = acc[r].find(k);
        msgs[r].push_back(it == acc[r].end() ? own(r, dest) : "(" + it->second + "+" + own(r, dest) + ")");
      }
    for (int r = 0; r < n; ++r) {
      const int src = mod_ranks(int64_t{r} - rd.peer, n);
      for (size_t i = 0; i < rd.chunks.size(); ++i) {
        const int k = received_offset(rd, rd.chunks[i], n);
        const std::string& m = msgs[src][i];
        if (k == 0) out[r] = "(" + out[r] + "+" + m + ")";
        else if (!acc[r].count(k)) acc[r][k] = m;
        else acc[r][k] = "(" + acc[r][k] + "+" + m + ")";
      }
      for (int k : rd.chunks) acc[r].erase(k);
    }
  }
  std::string e = out[0], res;  // c<src>_0 -> x<src>
  for (size_t i = 0; i < e.size();) {
    if (e[i] == 'c') {
      size_t j = e.find('_', i);
      res += "x" + e.substr(i + 1, j - i - 1);
      i = j + 2;  // skip "_0"
    } else {
      res += e[i++];
    }
  }
  return res;
}

// Compile a validated schedule into the schedule part of a KPlan (arrival slots, fold lists).
patResult_t compile_schedule(patComm* comm, const Schedule& given, Compiled** out) {
  std::vector<int32_t> key = encode(given);
  auto it = comm->compiled.find(key);
  if (it != comm->compiled.end()) {
    *out = &it->second;
    return patSuccess;
  }
  Compiled c;
  c.sched = given;
  if (c.sched.n != comm->n) return patPayloadShape;
  std::string why;
  if (validate(c.sched, &why) != 0) {
    std::fprintf(stderr, "pat_b200: invalid schedule: %s\n", why.c_str());
    return patInvalidSchedule;
  }
  const Schedule& s = c.sched;
  const int kind = static_cast<int>(s.kind);
  const int n = s.n;
  if (static_cast<int>(s.rounds.size()) > kMaxRounds) return patInvalidArgument;
  KPlan& p = c.proto;
  std::memset(&p, 0, sizeof(p));
  p.n = n;
  p.kind = kind;
  p.nrounds = static_cast<int>(s.rounds.size());
  int slot = 0;
  std::vector<int> slot_of_round_pos;  // flattened
  for (int t = 0; t < p.nrounds; ++t) {
    const Round& r = s.rounds[t];
    if (static_cast<int>(r.chunks.size()) > kMaxChunks || r.exchange) return patInvalidArgument;
    KRound& kr = p.rounds[t];
    kr.peer = static_cast<int8_t>(mod_ranks(r.peer, n));
    kr.nchunks = static_cast<int8_t>(r.chunks.size());
    kr.slot_base = static_cast<int8_t>(slot);
    for (size_t pos = 0; pos < r.chunks.size(); ++pos) {
      if (slot >= kMaxSlots) return patInvalidArgument;
      kr.chunk[pos] = static_cast<int8_t>(r.chunks[pos]);
      p.slot_round[slot] = static_cast<int8_t>(t);
      p.slot_offset[slot] = static_cast<int8_t>(received_offset(r, r.chunks[pos], n));
      ++slot;
    }
  }
  p.nslots = slot;
  // sources of every send, in reference order
  for (int t = 0; t < p.nrounds; ++t) {
    KRound& kr = p.rounds[t];
    for (int pos = 0; pos < kr.nchunks; ++pos) {
      const int k = kr.chunk[pos];
      int na = 0;
      for (int j = 0; j < kr.slot_base; ++j) {  // slots filled by earlier rounds, round order
        if (p.slot_offset[j] != k) continue;
        if (na >= kMaxArr) return patInvalidArgument;
        kr.arr[pos][na++] = static_cast<int8_t>(j);
      }
      if (kind == kAG) {
        if ((k == 0) != (na == 0)) return patInternalError;  // AG: own chunk or a held arrival
        na = std::min(na, 1);
      }
      kr.narr[pos] = static_cast<int8_t>(na);
    }
  }
  for (int j = 0; j < p.nslots; ++j)
    if (p.slot_offset[j] == 0) p.fin[p.nfin++] = static_cast<int8_t>(j);
  // PULL protocol tables (kernels: pull_task / pull_role)
  for (int j = 0; j < p.nslots; ++j) p.pull_dst[j] = -1;
  for (int f = 0; f < p.nfin; ++f) p.pull_act[p.fin[f]] = f == 0 ? kOutFirst : kOutNext;
  for (int t = 0; t < p.nrounds; ++t) {
    const KRound& kr = p.rounds[t];
    int dep = -1;
    for (int pos = 0; pos < kr.nchunks; ++pos) {
      const int na = kr.narr[pos];
      if (na == 0) continue;
      dep = std::max(dep, static_cast<int>(p.slot_round[kr.arr[pos][na - 1]]));
      for (int a = 0; a < na; ++a) {  // arrivals of the forwarded offset, round order
        const int j = kr.arr[pos][a];
        p.pull_dst[j] = kr.arr[pos][na - 1];
        p.pull_act[j] = na == 1 ? kAccOnly : a == 0 ? kAccFirst : a == na - 1 ? kAccLast : kAccMid;
      }
    }
    p.round_dep[t] = static_cast<int8_t>(dep);
  }
  for (int t = 0; t < p.nrounds; ++t) {
    if (p.round_dep[t] >= 0) p.sig_after[p.round_dep[t]] |= static_cast<uint8_t>(1u << t);
    for (int pos = 0; pos < p.rounds[t].nchunks; ++pos) {
      const int j = p.rounds[t].slot_base + pos;
      if (p.slot_offset[j] != 0) {
        p.stage_rounds |= static_cast<uint8_t>(1u << t);
        if (kind == kRS && p.pull_dst[j] < 0) return patInternalError;  // arrival never forwarded
      }
    }
  }
  // PULL staging holds accumulators only (fold of a forwarded offset's arrivals, finalised with
  // the own contribution): number them compactly, one slot per forwarded offset with arrivals
  // (the internal nodes of the reduction tree, the reference's intermediate slots). Ids are not
  // reused within a step: a reader may still be pulling an accumulator while its owner opens the
  // next one, and slots return only with done(step).
  {
    int8_t id_of[kMaxSlots];
    for (int j = 0; j < kMaxSlots; ++j) id_of[j] = -1;
    int na = 0;
    for (int j = 0; j < p.nslots; ++j) {
      const int d = p.pull_dst[j];
      if (d < 0) continue;
      if (id_of[d] < 0) id_of[d] = static_cast<int8_t>(na++);
      p.pull_dst[j] = id_of[d];
    }
    p.pull_nacc = static_cast<int8_t>(na);
  }
  for (int t = 0; t < p.nrounds; ++t) {
    bool seen = false;
    for (int k = 0; k < p.npeers; ++k) seen |= p.peers[k] == p.rounds[t].peer;
    if (!seen) p.peers[p.npeers++] = p.rounds[t].peer;
  }
  c.peak_slots = schedule_stats(s, 1).peak;
  c.fused_ok = kind == kAG || symbolic_reduce_scatter(s) == local_tree_string(n);
  auto ins = comm->compiled.emplace(std::move(key), std::move(c));
  *out = &ins.first->second;
  return patSuccess;
}

// The PAT schedule for (kind, trees) (algorithms.cpp:191-249), compiled once per communicator.
patResult_t compile(patComm* comm, int kind, int trees, Compiled** out) {
  const int key = kind * 64 + trees;
  auto it = comm->pat_cache.find(key);
  if (it != comm->pat_cache.end()) {
    *out = it->second;
    return patSuccess;
  }
  Schedule s;
  if (Err e = build(static_cast<Kind>(kind), Algo::Pat, comm->n, trees, &s)) return to_result(e);
  if (patResult_t e = compile_schedule(comm, s, out)) return e;
  comm->pat_cache[key] = *out;
  return patSuccess;
}

struct Slicing {
  int proto, channels, iters;
  int64_t slice;
};

// Alpha-beta model of one call (the reference's costmodel.cpp:70-104 prices a
// schedule as rounds x (alpha + beta x bytes)), calibrated on B200 by tools/fit_costmodel.py
// from forced-protocol sweeps at n = 2, 3, 4 (profiles/r01f_costmodel_fit.json):
//   t = steps x (a + b x R) + wire x (n-1) x C / B        (LL, LL32: one fixed cost per step)
//   t = a + b x R + (n-1) x C / B                          (SIMPLE / PULL: steps pipelined)
// R = PAT rounds. (n-1) x C does not depend on T, so T = max_trees (fewest rounds) is optimal.
struct CostRow {
  double a_us, b_us, gbs, wire;
};
constexpr CostRow kCostLL{3.41, 1.40, 565.0, 2.0};
constexpr CostRow kCostLL32{3.07, 2.42, 608.0, 32.0 / 28.0};  // one fixed cost per call (below)
// LL32 is eligible while a rank moves at most this much payload per call: measured against
// SIMPLE, LL32 wins up to (n-1) C = 48 MiB at n = 2 and 4 (n = 4, 16 MiB: 106 vs 110 us graph
// mode; loop mode SIMPLE is 0.95x NCCL there) and is within 6% at n = 3, 16 MiB
// (profiles/r01f_ll32_noskew_n*.jsonl, r01f_forced_n*_p2.jsonl, r01f_loopmid_n*.jsonl); the
// linear model alone would keep it far beyond, where SIMPLE's pipelined pushes reach 670 GB/s.
constexpr int64_t kLL32MaxPayload = 48ll << 20;
constexpr int64_t kLLMaxChunk = 256 << 10;  // auto mode sends chunks from here up with LL32 or bulk, never LL
constexpr double kCappedIterUs = 10.0;  // per extra bulk iteration under a staging cap (fence + flag)
constexpr size_t kCappedSmallSlot = 64 << 10;  // bulk slots below this make the fence dominate
constexpr CostRow kCostBulk{5.99, 6.11, 560.0, 1.0};

double predict_us(int proto, int n, int rounds, int64_t chunk_bytes, int iters) {
  // LL pays its fixed cost per step; LL32's extra steps cost nothing measurable (fit over
  // 1-10 steps, profiles/r01f_ll32_noskew_n*.jsonl), SIMPLE / PULL pipeline theirs
  const CostRow& c = proto == kProtoLL ? kCostLL : proto == kProtoLL32 ? kCostLL32 : kCostBulk;
  const double fixed = (proto == kProtoLL ? std::max(iters, 1) : 1) * (c.a_us + c.b_us * rounds);
  return fixed + c.wire * (n - 1) * static_cast<double>(chunk_bytes) / (c.gbs * 1e3);
}

// LL32 payload bytes per group of 32 lines (transport.cuh, LL32Shape): 28-byte lines, 24 for
// 8-byte reductions.
int64_t ll32_group(int kind, int64_t es) { return kind == kRS && es == 8 ? 768 : 896; }

// PULL staging slot for a schedule with `nacc` accumulators per step: the bulk region re-cut
// into region_channels x depth x nacc slots (at most kMaxSlice x 4 each)
int64_t pull_slot_bytes(const patComm* comm, int nacc) {
  const int64_t per = static_cast<int64_t>(comm->region_bytes[kProtoPull]) /
                      (int64_t{comm->region_channels[kProtoPull]} * comm->cfg.depth * std::max(nacc, 1));
  return std::min<int64_t>(per, 4 * kMaxSlice) & ~int64_t(127);
}

Slicing shape(const patComm* comm, int proto, int kind, int64_t chunk_bytes, int max_channels, int64_t es,
              int nacc, bool direct_ag = false) {
  Slicing s{};
  s.proto = proto;
  // a direct all-gather pushes into the peers' recvbufs: no inbox slots, so neither the slot size
  // nor the SIMPLE region's channel count (both shrink under a staging cap) bound its slicing
  const bool unstaged = direct_ag && proto == kProtoSimple;
  const int channels = std::max(1, std::min(unstaged ? comm->channels : comm->region_channels[proto], max_channels));
  int64_t cap = static_cast<int64_t>(comm->slot_bytes);
  if (unstaged) cap = std::max<int64_t>(cap, comm->pull_slice);
  int64_t minslice = 16 << 10;
  if (proto == kProtoLL) {
    cap = static_cast<int64_t>(comm->ll_slot_bytes / 2);
    minslice = 512;
  } else if (proto == kProtoLL32) {
    cap = static_cast<int64_t>(comm->ll32_slot_bytes / 1024) * ll32_group(kind, es);
    minslice = ll32_group(kind, es);
  } else if (proto == kProtoPull) {
    // RS stages only accumulators; AG pull stages nothing
    cap = kind == kAG ? std::max<int64_t>(cap, comm->pull_slice) : pull_slot_bytes(comm, nacc);
  }
  int64_t per = (chunk_bytes + channels - 1) / channels;
  per = (per + 15) & ~int64_t(15);
  per = std::max<int64_t>(per, std::min<int64_t>(minslice, cap));
  per = std::min<int64_t>(per, cap);
  s.slice = std::max<int64_t>(per, 16);
  const int64_t nslices = std::max<int64_t>(1, (chunk_bytes + s.slice - 1) / s.slice);
  s.channels = static_cast<int>(std::min<int64_t>(channels, nslices));
  s.iters = static_cast<int>((nslices + s.channels - 1) / s.channels);
  if (proto == kProtoLL32 && s.iters > 1) {
    // equal steps: every channel runs `iters` steps of the same size (no short last wave)
    const int64_t even = (chunk_bytes + int64_t{s.channels} * s.iters - 1) / (int64_t{s.channels} * s.iters);
    s.slice = std::min(s.slice, (even + 15) & ~int64_t(15));
  }
  return s;
}

Slicing choose_slicing(const patComm* comm, int kind, int64_t chunk_bytes, int max_channels, bool pull_ok,
                       int rounds, int64_t es, int nacc, bool direct_ag = false) {
  const int channels = std::max(1, std::min(comm->channels, max_channels));
  int proto = comm->cfg.protocol;
  if (proto == patProtoAuto) {
    // reduce-scatter reads faster than it pushes between 4 and 128 MiB in one process (the
    // receiver folds what it pulls, no inbox round trip); beyond that, and for all-gather,
    // pushed stores win (profiles/r01_sp_simple_vs_pull.jsonl)
    const int bulk = pull_ok && kind == kRS && chunk_bytes < kPullMaxRS ? kProtoPull : kProtoSimple;
    if (comm->cfg.ll_threshold) {  // explicit threshold
      proto = chunk_bytes <= static_cast<int64_t>(comm->cfg.ll_threshold) ? kProtoLL32 : bulk;
    } else {  // the cost model picks the fastest of LL, LL32 and the bulk protocol
      double best = 0;
      bool have = false;
      for (const int cand : std::array<int, 3>{kProtoLL, kProtoLL32, bulk}) {
        // from 256 KiB chunks LL32 beats LL at n = 2, 3, 4 by 5-20% (r02 forced sweeps,
        // profiles/r02_forced_n*_p{1,5}.jsonl), where the fitted model still favoured LL
        if (cand == kProtoLL && chunk_bytes >= kLLMaxChunk) continue;
        // uncapped, SIMPLE's pipelined pushes beat LL32's polled lines beyond 48 MiB of payload;
        // under a cap that shrank the bulk slots every size is a candidate for LL32
        const bool capped = comm->slot_bytes < kMaxSlice;
        if (cand == kProtoLL32 && !capped && static_cast<int64_t>(comm->n - 1) * chunk_bytes > kLL32MaxPayload)
          continue;
        const Slicing sh = shape(comm, cand, kind, chunk_bytes, channels, es, nacc, direct_ag);
        double t = predict_us(cand, comm->n, rounds, chunk_bytes, sh.iters);
        if (capped && comm->slot_bytes < kCappedSmallSlot && (cand == kProtoSimple || cand == kProtoPull) &&
            !(direct_ag && cand == kProtoSimple)) {
          // a bulk region shrunk to small slots: fewer channels push (each SM pushes ~5 GB/s) and
          // every iteration pays a fence for little data (profiles/r02_zero3_*: ~10 us per iteration)
          t += (static_cast<double>(kDefaultChannels) / std::max(sh.channels, 1) - 1.0) *
                   (comm->n - 1) * static_cast<double>(chunk_bytes) / (kCostBulk.gbs * 1e3) +
               kCappedIterUs * std::max(sh.iters - 1, 0);
        }
        if (!have || t < best) {
          best = t;
          proto = cand;
          have = true;
        }
      }
    }
  }
  if (proto == kProtoPull && !pull_ok) proto = kProtoSimple;
  return shape(comm, proto, kind, chunk_bytes, channels, es, nacc, direct_ag);
}

// Channels per rank such that every device's launch stays co-resident (cooperative launch).
patResult_t channel_cap(patComm* comm, int kind, int dtype, int op, int* cap) {
  *cap = kMaxChannels;
  const int threads = comm->cfg.threads;
  for (DevGroup& g : comm->groups) {
    const std::array<int, 5> okey{kind, dtype, op, threads, g.device};
    auto oit = comm->occupancy.find(okey);
    if (oit == comm->occupancy.end()) {
      int nb = 0;
      CUDA_TRY(cudaSetDevice(g.device));
      CUDA_TRY(max_blocks_per_sm(kind, dtype, op, threads, &nb));
      oit = comm->occupancy.emplace(okey, nb).first;
    }
    *cap = std::min(*cap, oit->second * g.sm_count / static_cast<int>(g.lidx.size()));
  }
  if (*cap < 1) return patInvalidUsage;
  return patSuccess;
}

patResult_t alloc_pool(patComm* comm, int device, char** pool) {
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaMalloc(pool, comm->pool_bytes));
  CUDA_TRY(cudaMemset(*pool, 0, comm->pool_bytes));
  comm->pools_allocated += comm->pool_bytes;
  return patSuccess;
}

// One-process communicators allocate every rank's pool on the first transport launch. A
// launch may be under stream capture: the allocation is not a stream operation, so it runs in
// relaxed capture mode for this thread and zeroes the pools synchronously before returning.
patResult_t ensure_pools(patComm* comm) {
  if (comm->pools_ready) return patSuccess;
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  CUDA_TRY(cudaThreadExchangeStreamCaptureMode(&mode));
  patResult_t rc = patSuccess;
  for (size_t l = comm->owned_pool.size(); l < comm->ldevs.size() && rc == patSuccess; ++l) {
    char* pool = nullptr;
    rc = alloc_pool(comm, comm->ldevs[l], &pool);
    if (rc == patSuccess) comm->owned_pool.push_back(pool);
  }
  if (rc == patSuccess)
    for (size_t l = 0; l < comm->ldevs.size(); ++l) {  // the memsets ran on the legacy stream
      cudaSetDevice(comm->ldevs[l]);
      if (cudaDeviceSynchronize() != cudaSuccess) rc = patUnhandledCudaError;
    }
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (rc != patSuccess) return rc;
  for (DevGroup& g : comm->groups)
    for (int r = 0; r < comm->n; ++r) g.pool_view[r] = comm->owned_pool[r];
  comm->pools_ready = true;
  return patSuccess;
}

patResult_t common_init(patComm* comm, int nranks, const patConfig_t* config) {
  if (nranks < 1 || nranks > PAT_MAX_RANKS) return patInvalidArgument;
  comm->n = nranks;
  patConfig_t c{};
  if (config) std::memcpy(&c, config, std::min(sizeof(c), config->size ? config->size : sizeof(c)));
  c.size = sizeof(c);
  fill_defaults(&c, nranks);
  if (c.trees != 0) {
    if (!is_pow2(c.trees) || c.trees > max_trees(nranks)) return patInvalidTreeCount;
  }
  if (c.protocol != patProtoAuto && c.protocol != patProtoLL && c.protocol != patProtoLL32 &&
      c.protocol != patProtoSimple && c.protocol != patProtoPull)
    return patInvalidArgument;
  comm->cfg = c;
  comm->channels = c.max_channels;
  {
    long long hp = 0;
    comm->host_profile = env_int("PAT_HOST_PROFILE", &hp) && hp != 0;
  }
  {
    long long v = 0;
    comm->pull_slice = env_int("PAT_PULL_SLICE", &v) && v >= 256 ? (v & ~15LL) : (512 << 10);
    comm->skew = env_int("PAT_SKEW", &v) ? static_cast<int>(std::max(0LL, v)) : 1;
    comm->leaves_first = env_int("PAT_LEAVES_FIRST", &v) ? static_cast<int>(v != 0) : -1;
    // the polling protocols need depth >= 2 (deferred credit, transport.cuh); they do not skew
    // a small cap (< 24 MiB) buys larger LL32 slots with two buffers per channel instead of depth:
    // 12 MiB, n = 4: 455 vs 326 GB/s busbw (profiles/r02_capped_poll_depth.jsonl)
    comm->depth_poll = env_int("PAT_POLL_DEPTH", &v)                         ? static_cast<int>(v)
                       : (c.staging_bytes != 0 && c.staging_bytes < (24u << 20)) ? 2
                                                                                  : c.depth;
    comm->depth_poll = std::min(std::max(comm->depth_poll, 2), c.depth);
    if (env_int("PAT_EPOCH_SHIFT", &v) && v >= 3 && v <= 31 && (1ll << v) > 2 * comm->depth_poll)
      comm->epoch_mask = (1ull << v) - 1;
    if (env_int("PAT_ITER_START", &v) && v > 0) comm->iter_start = static_cast<uint64_t>(v);
  }
  const Layout lay = plan_layout(c, nranks, comm->depth_poll, c.slice_bytes != 0);
  for (int p = 0; p < kNumProtoSlots; ++p) {
    comm->region_channels[p] = lay.ch[p];
    comm->region_bytes[p] = lay.bytes[p];
  }
  comm->slot_bytes = lay.slot[kProtoSimple];
  comm->ll_slot_bytes = lay.slot[kProtoLL];
  comm->ll32_slot_bytes = lay.slot[kProtoLL32];
  auto align = [](size_t x) { return (x + 4095) & ~size_t(4095); };
  comm->region_off[kProtoSimple] = comm->region_off[kProtoPull] = 0;
  comm->region_off[kProtoLL] = align(lay.bytes[kProtoSimple]);
  comm->region_off[kProtoLL32] = comm->region_off[kProtoLL] + align(lay.bytes[kProtoLL]);
  comm->pool_bytes = kFlagBytes + comm->region_off[kProtoLL32] + lay.bytes[kProtoLL32];
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&comm->err_host), sizeof(int),
                         cudaHostAllocMapped | cudaHostAllocPortable));
  *comm->err_host = 0;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&comm->err_dev), comm->err_host, 0));
  return patSuccess;
}

patResult_t setup_groups(patComm* comm) {
  std::map<int, int> gi;
  for (size_t l = 0; l < comm->ldevs.size(); ++l) {
    const int d = comm->ldevs[l];
    if (!gi.count(d)) {
      gi[d] = static_cast<int>(comm->groups.size());
      DevGroup g;
      g.device = d;
      comm->groups.push_back(g);
    }
    comm->groups[gi[d]].lidx.push_back(static_cast<int>(l));
  }
  for (DevGroup& g : comm->groups) {
    if (g.lidx.size() > static_cast<size_t>(kMaxLocal)) return patInvalidArgument;
    CUDA_TRY(cudaSetDevice(g.device));
    CUDA_TRY(cudaDeviceGetAttribute(&g.sm_count, cudaDevAttrMultiProcessorCount, g.device));
    const size_t bytes = sizeof(uint64_t) * kMaxChannels * g.lidx.size();
    CUDA_TRY(cudaMalloc(&g.iter_state, bytes));
    CUDA_TRY(cudaMemset(g.iter_state, 0, bytes));
    if (comm->iter_start) {
      CUDA_TRY(fill_u64(g.iter_state, static_cast<int64_t>(kMaxChannels * g.lidx.size()), comm->iter_start, nullptr));
      CUDA_TRY(cudaDeviceSynchronize());
    }
    long long stats = 0;
    if (env_int("PAT_STATS", &stats) && stats > 0) {  // device-counted occupancy (patCommStatsRead)
      const size_t ob = sizeof(int) * 2 * kMaxRounds * g.lidx.size();
      CUDA_TRY(cudaMalloc(&g.occ, ob));
      CUDA_TRY(cudaMemset(g.occ, 0, ob));
    }
    long long tcap = 0;
    if (env_int("PAT_TRACE", &tcap) && tcap > 0) {  // device event trace for tools/trace.py
      g.trace_cap = static_cast<int>(std::min<long long>(tcap, 4096));
      const size_t tb = sizeof(uint64_t) * 2 * 2 * g.trace_cap * kMaxChannels * g.lidx.size();
      CUDA_TRY(cudaMalloc(&g.trace, tb));
      CUDA_TRY(cudaMemset(g.trace, 0, tb));
    }
  }
  comm->events.resize(comm->lranks.size());
  for (size_t l = 0; l < comm->lranks.size(); ++l) {
    CUDA_TRY(cudaSetDevice(comm->ldevs[l]));
    CUDA_TRY(cudaEventCreateWithFlags(&comm->events[l], cudaEventDisableTiming));
  }
  for (DevGroup& g : comm->groups) {
    CUDA_TRY(cudaSetDevice(g.device));
    CUDA_TRY(cudaEventCreateWithFlags(&g.order_ev, cudaEventDisableTiming));
  }
  return patSuccess;
}

patResult_t check_async(patComm* comm) {
  const int e = *reinterpret_cast<volatile int*>(comm->err_host);
  return e ? static_cast<patResult_t>(e) : patSuccess;
}

// FNV-1a over every resolved setting that decides a call's protocol, slicing, channel count or
// pool layout. The processes of a multi-process communicator each resolve their own config (env
// knobs included); one that differs would slice differently or read another region, so
// patCommInitRankFinish refuses the communicator instead of hanging or corrupting data.
uint64_t config_fingerprint(const patComm* comm) {
  const patConfig_t& c = comm->cfg;
  const uint64_t v[] = {c.staging_bytes, c.slice_bytes, c.ll_threshold, uint64_t(c.trees), uint64_t(c.max_channels),
                        uint64_t(c.protocol), uint64_t(c.threads), uint64_t(c.depth), uint64_t(c.direct),
                        uint64_t(c.send_warps), uint64_t(c.fused), uint64_t(comm->skew), uint64_t(comm->leaves_first), uint64_t(comm->pull_slice),
                        comm->slot_bytes, comm->ll_slot_bytes, comm->ll32_slot_bytes, comm->pool_bytes,
                        comm->region_off[kProtoLL], comm->region_off[kProtoLL32], comm->epoch_mask,
                        comm->iter_start, uint64_t(comm->depth_poll)};
  uint64_t h = 1469598103934665603ull;
  for (uint64_t x : v)
    for (int b = 0; b < 8; ++b) h = (h ^ ((x >> (8 * b)) & 0xff)) * 1099511628211ull;
  return h;
}

// Every rank on one device and the compiled schedule is the tree local.cu evaluates: the
// fused single-device executor runs the call, no transport.
bool fused_path(const patComm* comm, const Compiled* cp) {
  return !comm->multiprocess && comm->groups.size() == 1 && comm->cfg.fused >= 0 && cp->fused_ok &&
         static_cast<int>(comm->groups[0].lidx.size()) == comm->n;
}

// The symmetric window holding [ptr, ptr + bytes), if any.
const patComm::Window* find_window(const patComm* comm, const void* ptr, int64_t bytes) {
  const char* q = static_cast<const char*>(ptr);
  for (const auto& w : comm->windows)
    if (q >= w.local && q + bytes <= w.local + w.bytes) return &w;
  return nullptr;
}

// Inbox slots one pipeline step occupies at a receiver.
int staged_slots(int proto, int kind, bool direct, const KPlan& p) {
  if (proto == kProtoPull) return kind == kRS ? p.pull_nacc : 0;
  if (direct) return 0;
  return p.nslots;
}

int64_t proto_slot_stride(const patComm* comm, int proto, int nacc) {
  return static_cast<int64_t>(proto == kProtoLL     ? comm->ll_slot_bytes
                              : proto == kProtoLL32 ? comm->ll32_slot_bytes
                              : proto == kProtoPull ? pull_slot_bytes(comm, nacc)
                                                    : comm->slot_bytes);
}

// A collective ready to launch: per device group the KPlan (or, fused, the local executor's args).
struct Prepared {
  bool fused = false;
  int kind = 0, dtype = 0, op = 0;
  int64_t chunk_bytes = 0;
  size_t es = 0;
  bool aligned16 = false;
  std::vector<KPlan> plans;  // per device group
};

patResult_t submit_prepared(patComm* comm, const Prepared& a, const Prepared* b, const patStream_t* streams);

// split: 0 = the call alone; 1 / 2 = first / second half of the channels of its protocol's region
// (a grouped pair sharing one launch, patGroupEnd). prep != nullptr: build the plans, do not launch.
patResult_t run_collective(patComm* comm, int kind, const void* const* sendbuffs, void* const* recvbuffs,
                           size_t count, int dtype, int op, const patStream_t* streams,
                           const Schedule* explicit_sched = nullptr, int split = 0, Prepared* prep = nullptr) {
  if (!comm || !comm->finished) return patInvalidUsage;
  const size_t es = dtype_size(dtype);
  if (!es) return patInvalidArgument;
  if (op < 0 || op >= patNumOps) return patUnsupportedOp;
  if (count == 0) return patSuccess;
  if (!sendbuffs || !recvbuffs) return patInvalidArgument;
  // n * count * es bytes (the all-gather output, the reduce-scatter input) must fit in int64
  if (count > static_cast<size_t>(INT64_MAX) / es / static_cast<size_t>(comm->n)) return patInvalidArgument;
  for (size_t l = 0; l < comm->lranks.size(); ++l)
    if (!sendbuffs[l] || !recvbuffs[l]) return patInvalidArgument;
  if (patResult_t e = check_async(comm)) return e;
  std::lock_guard<std::mutex> lock(comm->mu);
  const auto hp_t0 = comm->host_profile ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
  const int n = comm->n;
  const int trees = comm->cfg.trees ? comm->cfg.trees : max_trees(n);
  Compiled* cp = nullptr;
  if (explicit_sched) {
    if (static_cast<int>(explicit_sched->kind) != kind) return patSimulationError;
    if (patResult_t e = compile_schedule(comm, *explicit_sched, &cp)) return e;
  } else if (patResult_t e = compile(comm, kind, trees, &cp)) {
    return e;
  }
  const int64_t chunk_bytes = static_cast<int64_t>(count * es);
  DeviceGuard guard;
  int cap = 0;
  if (patResult_t e = channel_cap(comm, kind, dtype, op, &cap)) return e;
  // one device holds every rank: .gpu-scope flags; zero-copy all-gather is always safe
  const bool single_device = !comm->multiprocess && comm->groups.size() == 1;
  // PULL reads the peers' user buffers: they must be mapped into every device of this process.
  // Auto mode only pulls mid-size reduce-scatters, so small calls skip the pointer queries.
  // One process per rank: zero copy needs the user buffers inside symmetric windows
  // (patCommRegister*); the peers' buffers are then at the same window offset.
  const patComm::Window* wsend = nullptr;
  const patComm::Window* wrecv = nullptr;
  if (comm->multiprocess && !comm->windows.empty()) {
    const int64_t sb = kind == kAG ? chunk_bytes : n * chunk_bytes, rb = kind == kAG ? n * chunk_bytes : chunk_bytes;
    wsend = find_window(comm, sendbuffs[0], sb);
    wrecv = find_window(comm, recvbuffs[0], rb);
  }
  bool pull_ok = (!comm->multiprocess || (wsend && (kind == kRS || wrecv))) && comm->cfg.protocol != patProtoSimple &&
                 (comm->cfg.protocol == patProtoPull || (kind == kRS && chunk_bytes > kPullMinRS));
  for (size_t l = 0; l < comm->lranks.size() && pull_ok && !single_device && !comm->multiprocess; ++l)
    pull_ok = legacy_ipc_capable(sendbuffs[l]) && (kind == kRS || legacy_ipc_capable(recvbuffs[l]));
  // zero-copy all-gather (SIMPLE pushes straight into the peers' recvbufs) where they are
  // reachable: one device; cudaMalloc'd buffers under peer access (one process); symmetric windows
  // (one process per rank). Only bulk calls can take SIMPLE, so small calls skip the queries.
  bool direct_ok = kind == kAG && comm->cfg.direct >= 0 && comm->cfg.protocol != patProtoLL &&
                   comm->cfg.protocol != patProtoLL32 && comm->cfg.protocol != patProtoPull &&
                   (comm->cfg.protocol == patProtoSimple || static_cast<int64_t>(n - 1) * chunk_bytes > (4 << 20));
  if (direct_ok) {
    if (comm->multiprocess) {
      direct_ok = wrecv != nullptr;
    } else if (!single_device && comm->cfg.direct == 0) {  // auto: every recvbuf reachable through peer access
      for (size_t l = 0; l < comm->lranks.size() && direct_ok; ++l) direct_ok = legacy_ipc_capable(recvbuffs[l]);
    }
  }
  if (split) {  // a grouped pair: both halves of one launch must be co-resident together
    int gcap = 0;
    if (patResult_t e = channel_cap(comm, 2, dtype, op, &gcap)) return e;
    cap = std::min(cap, gcap / 2);
  }
  Slicing sl = choose_slicing(comm, kind, chunk_bytes, split ? std::max(cap, 1) : cap, pull_ok, cp->proto.nrounds,
                              static_cast<int64_t>(es), cp->proto.pull_nacc, direct_ok);
  int chan_base = 0;
  if (split) {  // half of the protocol's channel region each, so the two ranges never overlap
    const int region = (direct_ok && sl.proto == kProtoSimple) ? comm->channels : comm->region_channels[sl.proto];
    const int half = std::max(region / 2, 1);
    if (region < 2) return patInvalidUsage;
    sl = shape(comm, sl.proto, kind, chunk_bytes, std::min(std::max(cap, 1), half), static_cast<int64_t>(es),
               cp->proto.pull_nacc, direct_ok);
    chan_base = split == 2 ? half : 0;
  }
  int vec = 16;
  bool aligned4 = (chunk_bytes % 4) == 0, aligned8 = (chunk_bytes % 8) == 0, aligned16 = (chunk_bytes % 16) == 0;
  for (size_t l = 0; l < comm->lranks.size(); ++l) {
    if (!sendbuffs[l] || !recvbuffs[l]) return patInvalidArgument;
    const uintptr_t a = reinterpret_cast<uintptr_t>(sendbuffs[l]) | reinterpret_cast<uintptr_t>(recvbuffs[l]);
    aligned16 &= (a % 16) == 0;
    aligned8 &= (a % 8) == 0;
    aligned4 &= (a % 4) == 0;
  }
  vec = aligned16 ? 16 : (aligned8 ? 8 : 0);
  if (sl.proto == kProtoLL32 && vec == 0 && aligned4) vec = 4;  // LL32 moves 4-byte units
  if (sl.proto == kProtoSimple && vec == 8) vec = 0;  // SIMPLE vectors are 16 bytes
  const bool fused = fused_path(comm, cp);
  if (!fused)
    if (patResult_t e = ensure_pools(comm)) return e;
  const bool direct = direct_ok && sl.proto == kProtoSimple;
  // window tag the kernels compare at entry (transport.cuh: sym_check)
  uint64_t sym_tag = 0;
  // an in-place all-gather (sendbuf = recvbuf + rank * count, NCCL's form) has its send buffer at a
  // rank-dependent window offset: the peers' send buffers are found through their recv windows
  const bool inplace_ag = comm->multiprocess && kind == kAG && wrecv &&
                          static_cast<const char*>(sendbuffs[0]) ==
                              static_cast<const char*>(recvbuffs[0]) + comm->lranks[0] * chunk_bytes;
  if (comm->multiprocess && (direct || sl.proto == kProtoPull)) {
    auto mix = [](uint64_t h, uint64_t x) { return (h ^ x) * 0x100000001B3ull + (h >> 29); };
    uint64_t h = 0xcbf29ce484222325ull;
    if (sl.proto == kProtoPull && inplace_ag)
      h = mix(h, 0x1b9ace0000000000ull);  // every rank must call in place
    else if (sl.proto == kProtoPull)
      h = mix(mix(h, wsend->id), static_cast<uint64_t>(static_cast<const char*>(sendbuffs[0]) - wsend->local));
    if (direct || (sl.proto == kProtoPull && kind == kAG))
      h = mix(mix(h, wrecv->id + 0x10000ull), static_cast<uint64_t>(static_cast<char*>(recvbuffs[0]) - wrecv->local));
    sym_tag = h | 1;
  }
  std::vector<KPlan> plans(comm->groups.size());
  for (size_t gi = 0; gi < comm->groups.size(); ++gi) {
    DevGroup& g = comm->groups[gi];
    KPlan& p = plans[gi];
    p = cp->proto;
    p.nlocal = static_cast<int>(g.lidx.size());
    p.proto = sl.proto;
    p.vec = vec;
    p.esize = static_cast<int>(es);
    p.channels = sl.channels;
    p.chan_base = chan_base;
    p.iters = sl.iters;
    p.chunk_bytes = chunk_bytes;
    p.slice_bytes = sl.slice;
    p.slot_stride = proto_slot_stride(comm, sl.proto, p.pull_nacc);
    const bool polling = sl.proto == kProtoLL || sl.proto == kProtoLL32;
    p.depth = polling ? comm->depth_poll : comm->cfg.depth;
    {
      // skew distance L: the sender keeps (nrounds-1)*L+1 steps in flight -> needs that many buffers
      const int L = comm->skew;
      if (p.proto == kProtoPull)  // all-gather pull stages nothing: no credit bound on the skew
        p.skew = (L > 0 && p.nrounds > 1 && (kind == kAG || p.depth >= (p.nrounds - 1) * L + 1)) ? L : 0;
      else
        p.skew = (L > 0 && p.proto == kProtoSimple && p.nrounds > 1 && p.depth >= (p.nrounds - 1) * L + 1 &&
                  (p.nrounds - 1) * L + 1 <= kMaxRounds)
                     ? L
                     : 0;
    }
    // region layout [channel][buffer][slot]: n-1 landing slots per step, PULL's accumulators
    p.chan_stride = static_cast<int64_t>(p.depth) * (sl.proto == kProtoPull ? std::max<int>(p.pull_nacc, 1) : std::max(n - 1, 1)) *
                    p.slot_stride;
    p.send_warps = comm->cfg.send_warps;
    p.region_bytes = static_cast<int64_t>(comm->region_bytes[sl.proto]);
    // leaves first (r02 A/B, n = 4 all-gather, profiles/r02_leaves_first_n4.jsonl): +7% for a
    // one-step SIMPLE call (32 MiB), -1 to -5% for LL32 and multi-step SIMPLE (the skewed
    // wavefront already keeps the link busy), so by default only single-step SIMPLE calls
    p.leaves_first = sl.proto == kProtoPull ? 0
                     : comm->leaves_first >= 0 ? comm->leaves_first
                                                : (sl.proto == kProtoSimple && sl.iters == 1 ? 1 : 0);
    p.gpu_scope = single_device ? 1 : 0;
    p.direct = direct && sl.proto != kProtoPull ? 1 : 0;
    if (sl.proto == kProtoPull)
      for (size_t l = 0; l < comm->lranks.size(); ++l) {
        p.peer_send[comm->lranks[l]] = static_cast<const char*>(sendbuffs[l]);
        p.peer_recv[comm->lranks[l]] = static_cast<char*>(recvbuffs[l]);
      }
    if (direct)
      for (size_t l = 0; l < comm->lranks.size(); ++l) p.peer_recv[comm->lranks[l]] = static_cast<char*>(recvbuffs[l]);
    p.sym_tag = sym_tag;
    if (sym_tag) {  // the peers' buffers through their windows
      const int me = comm->lranks[0];
      for (int r = 0; r < n; ++r) {
        if (r == me) continue;
        if (sl.proto == kProtoPull && inplace_ag)
          p.peer_send[r] = wrecv->peer[r] + (static_cast<char*>(recvbuffs[0]) - wrecv->local) + r * chunk_bytes;
        else if (wsend && sl.proto == kProtoPull)
          p.peer_send[r] = wsend->peer[r] + (static_cast<const char*>(sendbuffs[0]) - wsend->local);
        if (wrecv && (direct || kind == kAG))
          p.peer_recv[r] = wrecv->peer[r] + (static_cast<char*>(recvbuffs[0]) - wrecv->local);
      }
    }
    p.timeout_ns = static_cast<uint64_t>(comm->cfg.timeout_ms) * 1000000ull;
    p.epoch_mask = comm->epoch_mask;
    p.depth_poll = comm->depth_poll;
    p.poll_channels[0] = comm->region_channels[kProtoLL];
    p.poll_channels[1] = comm->region_channels[kProtoLL32];
    p.poll_off[0] = static_cast<int64_t>(kFlagBytes + comm->region_off[kProtoLL]);
    p.poll_off[1] = static_cast<int64_t>(kFlagBytes + comm->region_off[kProtoLL32]);
    p.poll_slot[0] = static_cast<int64_t>(comm->ll_slot_bytes);
    p.poll_slot[1] = static_cast<int64_t>(comm->ll32_slot_bytes);
    p.err = comm->err_dev;
    p.occ = nullptr;
    if (g.occ && sl.proto == kProtoSimple && !split) {
      p.occ = g.occ;
      g.occ_rounds = p.nrounds;
      CUDA_TRY(cudaSetDevice(g.device));
      CUDA_TRY(cudaMemsetAsync(g.occ, 0, sizeof(int) * 2 * kMaxRounds * g.lidx.size(),
                               streams ? reinterpret_cast<cudaStream_t>(streams[g.lidx[0]]) : nullptr));
    }
    p.trace = split ? nullptr : g.trace;  // the trace indexes CTAs by blockIdx: single calls only
    p.trace_cap = g.trace_cap;
    if (p.trace) {
      g.trace_ctas = p.nlocal * p.channels;
      CUDA_TRY(cudaMemsetAsync(g.trace, 0, sizeof(uint64_t) * 4 * g.trace_cap * g.trace_ctas,
                               streams ? reinterpret_cast<cudaStream_t>(streams[g.lidx[0]]) : nullptr));
    }
    for (int r = 0; r < n; ++r) {
      p.flags[r] = reinterpret_cast<uint64_t*>(g.pool_view[r]);
      p.inbox[r] = g.pool_view[r] + kFlagBytes + comm->region_off[sl.proto];
    }
    for (size_t i = 0; i < g.lidx.size(); ++i) {
      const int l = g.lidx[i];
      p.rank[i] = comm->lranks[l];
      p.send[i] = static_cast<const char*>(sendbuffs[l]);
      p.recv[i] = static_cast<char*>(recvbuffs[l]);
      p.iter_state[i] = g.iter_state + i * kMaxChannels;
    }
  }
  Prepared local;
  Prepared& P = prep ? *prep : local;
  P.fused = fused;
  P.kind = kind;
  P.dtype = dtype;
  P.op = op;
  P.chunk_bytes = chunk_bytes;
  P.es = es;
  P.aligned16 = aligned16;
  P.plans = std::move(plans);
  if (prep) return patSuccess;
  if (!comm->host_profile) return submit_prepared(comm, P, nullptr, streams);
  const auto hp_t1 = std::chrono::steady_clock::now();
  const patResult_t rc = submit_prepared(comm, P, nullptr, streams);
  const auto hp_t2 = std::chrono::steady_clock::now();
  ++comm->hp_calls;
  comm->hp_plan_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(hp_t1 - hp_t0).count();
  comm->hp_submit_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(hp_t2 - hp_t1).count();
  return rc;
}

// Threads per CTA of a transport launch. The polling protocols give every thread whole lines, so
// a call whose step has few lines per channel runs smaller CTAs: their barriers are cheaper
// (tools/gpurun/r02bh.sh: 256- and 384-thread CTAs were 2-7% faster on calls <= 32 KiB).
// SIMPLE / PULL keep the configured size (warp-specialised roles, per-thread vector pipelines).
// PAT_POLL_THREADS=0 turns the sizing off.
int launch_threads(const patComm* comm, const KPlan& p) {
  static const bool on = [] {
    long long v = 1;
    return !env_int("PAT_POLL_THREADS", &v) || v != 0;
  }();
  const int cfg = comm->cfg.threads;
  if (!on || (p.proto != kProtoLL && p.proto != kProtoLL32)) return cfg;
  const int64_t lines = p.proto == kProtoLL ? (p.slice_bytes + 7) / 8
                                            : (p.slice_bytes + ll32_group(p.kind, p.esize) - 1) /
                                                  ll32_group(p.kind, p.esize) * 32;
  const int64_t want = std::max<int64_t>(64, (lines + 31) / 32 * 32);
  return static_cast<int>(std::min<int64_t>(cfg, want));
}

// Launch a prepared call — or a grouped pair (a = all-gather, b = reduce-scatter sum) as ONE
// launch per device — on the streams of the local ranks.
patResult_t submit_prepared(patComm* comm, const Prepared& a, const Prepared* b, const patStream_t* streams) {
  const int n = comm->n;
  // submission to one device: join the stream of every local rank of the device, one launch
  auto submit = [&](size_t gi) -> patResult_t {
    DevGroup& g = comm->groups[gi];
    const KPlan& p = a.plans[gi];
    CUDA_TRY(cudaSetDevice(g.device));
    const int threads = b ? std::max(launch_threads(comm, p), launch_threads(comm, b->plans[gi]))
                          : launch_threads(comm, p);
    cudaStream_t s0 = streams ? reinterpret_cast<cudaStream_t>(streams[g.lidx[0]]) : nullptr;
    // transport calls share the channels' flags, step counters and inboxes: each waits for the
    // previous one when it comes on another stream. The fused executor keeps no state between
    // calls, and a stream being captured into a graph is ordered by its user (the graph runs later)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    bool ordered = !a.fused && cudaStreamIsCapturing(s0, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
    if (!a.fused && !ordered) cudaGetLastError();  // the legacy stream under a global capture elsewhere
    if (ordered && g.has_last && g.last_stream != s0) CUDA_TRY(cudaStreamWaitEvent(s0, g.order_ev, 0));
    for (size_t i = 1; i < g.lidx.size(); ++i) {  // join the other local ranks' streams
      cudaStream_t si = streams ? reinterpret_cast<cudaStream_t>(streams[g.lidx[i]]) : nullptr;
      if (si == s0) continue;
      CUDA_TRY(cudaEventRecord(comm->events[g.lidx[i]], si));
      CUDA_TRY(cudaStreamWaitEvent(s0, comm->events[g.lidx[i]], 0));
    }
    if (a.fused) {  // every rank in this HBM: fused executor (local.cu), no transport
      const char* sb[kMaxRanks];
      char* rb[kMaxRanks];
      for (size_t i = 0; i < g.lidx.size(); ++i) {
        sb[p.rank[i]] = p.send[i];
        rb[p.rank[i]] = p.recv[i];
      }
      bool done = false;
      if (b) {
        const KPlan& q = b->plans[gi];
        const char* sb2[kMaxRanks];
        char* rb2[kMaxRanks];
        for (size_t i = 0; i < g.lidx.size(); ++i) {
          sb2[q.rank[i]] = q.send[i];
          rb2[q.rank[i]] = q.recv[i];
        }
        const cudaError_t e = launch_local_group(n, b->dtype, a.chunk_bytes, sb, rb, b->chunk_bytes, sb2, rb2,
                                                 g.sm_count, s0);
        if (e == cudaErrorNotSupported) {  // alignment: one after the other
          CUDA_TRY(launch_local(a.kind, n, a.dtype, a.op, a.aligned16 ? 16 : 0, static_cast<int>(a.es), a.chunk_bytes,
                                sb, rb, g.sm_count, s0));
          CUDA_TRY(launch_local(b->kind, n, b->dtype, b->op, b->aligned16 ? 16 : 0, static_cast<int>(b->es),
                                b->chunk_bytes, sb2, rb2, g.sm_count, s0));
        } else {
          CUDA_TRY(e);
        }
        done = true;
      }
      if (!done)
        CUDA_TRY(launch_local(a.kind, n, a.dtype, a.op, a.aligned16 ? 16 : 0, static_cast<int>(a.es), a.chunk_bytes,
                              sb, rb, g.sm_count, s0));
    } else if (b) {
      KPlan2 both;
      both.a = p;
      both.b = b->plans[gi];
      CUDA_TRY(launch_group(both, b->dtype, threads, s0));
    } else {
      CUDA_TRY(launch(p, a.dtype, a.op, threads, s0));
    }
    bool joined = false;
    for (size_t i = 1; i < g.lidx.size(); ++i) {
      cudaStream_t si = streams ? reinterpret_cast<cudaStream_t>(streams[g.lidx[i]]) : nullptr;
      if (si == s0) continue;
      if (!joined) CUDA_TRY(cudaEventRecord(comm->events[g.lidx[0]], s0));
      joined = true;
      CUDA_TRY(cudaStreamWaitEvent(si, comm->events[g.lidx[0]], 0));
    }
    if (ordered) {
      CUDA_TRY(cudaEventRecord(g.order_ev, s0));
      g.last_stream = s0;
      g.has_last = true;
    }
    return patSuccess;
  };
  // Several devices and an eager call: the launch workers submit to devices 1.. while this
  // thread submits to device 0. A stream being captured into a graph is submitted inline (the
  // launch cost is paid once at capture then).
  bool parallel = comm->workers.size() + 1 == comm->groups.size() && comm->groups.size() > 1;
  if (parallel) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaSetDevice(comm->groups[0].device));
    const cudaStream_t s0 = streams ? reinterpret_cast<cudaStream_t>(streams[comm->groups[0].lidx[0]]) : nullptr;
    if (cudaStreamIsCapturing(s0, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      parallel = false;
    }
  }
  if (!parallel) {
    for (size_t gi = 0; gi < comm->groups.size(); ++gi)
      if (patResult_t e = submit(gi)) return e;
    return patSuccess;
  }
  std::vector<std::function<int()>> jobs(comm->groups.size());
  for (size_t gi = 1; gi < comm->groups.size(); ++gi) {
    jobs[gi] = [&submit, gi] { return static_cast<int>(submit(gi)); };
    comm->workers[gi - 1]->post(&jobs[gi]);
  }
  patResult_t first = submit(0);
  for (size_t gi = 1; gi < comm->groups.size(); ++gi) {
    const auto e = static_cast<patResult_t>(comm->workers[gi - 1]->wait());
    if (first == patSuccess) first = e;
  }
  return first;
}

// ---------------------------------------------------------------------------- groups
// patGroupStart / patGroupEnd (NCCL's group semantics, per host thread): collectives issued in
// between are recorded and launched at the outermost patGroupEnd. An all-gather and a
// reduce-scatter (sum) of one communicator on the same streams become ONE launch — each on half
// of the channels, fused executor or transport — so their latencies overlap; anything else is
// launched call by call, in order. The calls of a group must be independent (as in NCCL).
struct PendingCall {
  patComm* comm = nullptr;
  int kind = 0, dtype = 0, op = 0;
  size_t count = 0;
  std::vector<const void*> send;
  std::vector<void*> recv;
  std::vector<patStream_t> streams;
  bool has_streams = false;
  bool has_sched = false;
  Schedule sched;
};
struct GroupState {
  int depth = 0;
  std::vector<PendingCall> calls;
};
thread_local GroupState t_group;

patResult_t record_call(patComm* comm, int kind, const void* const* sendbuffs, void* const* recvbuffs, size_t count,
                        int dtype, int op, const patStream_t* streams, const Schedule* sched) {
  if (!comm || !comm->finished) return patInvalidUsage;
  if (!sendbuffs || !recvbuffs) return patInvalidArgument;
  PendingCall c;
  c.comm = comm;
  c.kind = kind;
  c.dtype = dtype;
  c.op = op;
  c.count = count;
  const size_t L = comm->lranks.size();
  c.send.assign(sendbuffs, sendbuffs + L);
  c.recv.assign(recvbuffs, recvbuffs + L);
  if (streams) {
    c.streams.assign(streams, streams + L);
    c.has_streams = true;
  }
  if (sched) {
    c.sched = *sched;
    c.has_sched = true;
  }
  t_group.calls.push_back(std::move(c));
  return patSuccess;
}

patResult_t run_pending(PendingCall& c) {
  return run_collective(c.comm, c.kind, c.send.data(), c.recv.data(), c.count, c.dtype, c.op,
                        c.has_streams ? c.streams.data() : nullptr, c.has_sched ? &c.sched : nullptr);
}

bool groupable(const PendingCall& x, const PendingCall& y) {
  if (x.comm != y.comm || x.kind == y.kind || x.has_sched || y.has_sched || !x.count || !y.count) return false;
  if (x.has_streams != y.has_streams || x.streams != y.streams) return false;
  const PendingCall& rs = x.kind == kRS ? x : y;
  if (rs.op != patSum || !dtype_size(rs.dtype) || !dtype_size(x.kind == kAG ? x.dtype : y.dtype)) return false;
  static const bool off = [] {
    long long v = 0;
    return env_int("PAT_GROUP_FUSE", &v) && v == 0;
  }();
  return !off;
}

patResult_t run_group_pair(PendingCall& x, PendingCall& y) {
  PendingCall& ag = x.kind == kAG ? x : y;
  PendingCall& rs = x.kind == kAG ? y : x;
  patComm* comm = ag.comm;
  Prepared pa, pb;
  const patStream_t* st = ag.has_streams ? ag.streams.data() : nullptr;
  if (patResult_t e = run_collective(comm, kAG, ag.send.data(), ag.recv.data(), ag.count, ag.dtype, ag.op, st,
                                     nullptr, 1, &pa))
    return e;
  if (patResult_t e = run_collective(comm, kRS, rs.send.data(), rs.recv.data(), rs.count, rs.dtype, rs.op, st,
                                     nullptr, 2, &pb))
    return e;
  // zero-copy bulk calls (direct all-gather, PULL reduce-scatter) on half the channels each measured
  // slower than one after the other (ZeRO-3 shape with windows, n = 4: 0.787 vs 0.646 ms per step,
  // profiles/r02_zero3_grouped_n4.jsonl); staged and polling pairs gain (0.629 vs 0.670 ms)
  auto zero_copy_bulk = [](const Prepared& q) {
    return !q.fused && !q.plans.empty() && (q.plans[0].proto == kProtoPull || q.plans[0].direct);
  };
  // the halves index the per-channel flags and step counters by absolute channel: calls of two
  // protocols whose regions differ in size (an LL half is at most 16 channels, an LL32 or SIMPLE
  // half 74) can land on common channels, and must then run one after the other
  auto overlap = [](const Prepared& p, const Prepared& q) {
    const KPlan& x = p.plans[0];
    const KPlan& y = q.plans[0];
    return x.chan_base < y.chan_base + y.channels && y.chan_base < x.chan_base + x.channels;
  };
  if (pa.fused != pb.fused || (!pa.fused && (pa.plans.empty() || pb.plans.empty())) || zero_copy_bulk(pa) ||
      zero_copy_bulk(pb) || (!pa.fused && overlap(pa, pb))) {
    // not the same executor, or a pair that runs better apart: one after the other
    if (patResult_t e = run_pending(x)) return e;
    return run_pending(y);
  }
  std::lock_guard<std::mutex> lock(comm->mu);
  DeviceGuard guard;
  return submit_prepared(comm, pa, &pb, st);
}

}  // namespace

// =========================================================================== C ABI

#pragma GCC visibility push(default)
extern "C" {

const char* patGetErrorString(patResult_t r) {
  switch (r) {
    case patSuccess: return "success";
    case patUnhandledCudaError: return "unhandled CUDA error";
    case patSystemError: return "system error (peer access / IPC)";
    case patInternalError: return "internal error";
    case patInvalidArgument: return "invalid argument";
    case patInvalidUsage: return "invalid usage";
    case patRemoteError: return "remote error";
    case patScheduleError: return "ScheduleError";
    case patNonPowerOfTwo: return "NonPowerOfTwoError";
    case patInvalidTreeCount: return "InvalidTreeCountError";
    case patBufferTooSmall: return "BufferTooSmallError";
    case patRankOutOfRange: return "RankOutOfRangeError";
    case patSimulationError: return "SimulationError";
    case patPayloadShape: return "PayloadShapeError";
    case patUnsupportedOp: return "UnsupportedOpError";
    case patInvalidSchedule: return "InvalidScheduleError";
    case patTimeout: return "device wait timed out";
    case patCapacity: return "output buffer too small";
  }
  return "unknown error";
}

patResult_t patGetVersion(int* v) {
  if (!v) return patInvalidArgument;
  *v = PAT_B200_VERSION;
  return patSuccess;
}

patResult_t patConfigInit(patConfig_t* c) {
  if (!c) return patInvalidArgument;
  std::memset(c, 0, sizeof(*c));
  c->size = sizeof(*c);
  return patSuccess;
}

patResult_t patCommInitAll(patComm_t* out, int nranks, const int* devlist, const patConfig_t* config) {
  if (!out) return patInvalidArgument;
  *out = nullptr;
  auto comm = std::make_unique<patComm>();
  if (patResult_t e = common_init(comm.get(), nranks, config)) return e;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  DeviceGuard guard;
  for (int r = 0; r < nranks; ++r) {
    const int d = devlist ? devlist[r] : r;
    if (d < 0 || d >= ndev) return patInvalidArgument;
    comm->lranks.push_back(r);
    comm->ldevs.push_back(d);
  }
  // peer access between every pair of distinct devices
  std::vector<int> devs(comm->ldevs);
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) {
        std::fprintf(stderr, "pat_b200: device %d cannot access peer %d\n", a, b);
        return patSystemError;
      }
      CUDA_TRY(cudaSetDevice(a));
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return patSystemError;
    }
  if (patResult_t e = setup_groups(comm.get())) return e;
  // every rank on one device: calls run in the fused executor unless asked not to, so the
  // pools wait for the first transport launch (ensure_pools); otherwise allocate them now
  if (!(comm->groups.size() == 1 && comm->cfg.fused >= 0))
    if (patResult_t e = ensure_pools(comm.get())) return e;
  long long lt = 1;
  env_int("PAT_LAUNCH_THREADS", &lt);  // 0: one thread submits to every device in turn
  if (lt != 0)
    for (size_t gi = 1; gi < comm->groups.size(); ++gi) {
      auto w = std::make_unique<LaunchWorker>();
      long long spin = 0;
      if (env_int("PAT_WORKER_SPIN_US", &spin) && spin >= 0) w->spin_us = spin;
      const int dev = comm->groups[gi].device;
      LaunchWorker* wp = w.get();
      w->th = std::thread([wp, dev] {
        cudaSetDevice(dev);
        wp->run();
      });
      comm->workers.push_back(std::move(w));
    }
  comm->finished = true;
  *out = comm.release();
  return patSuccess;
}

patResult_t patCommInitRankPrepare(patComm_t* out, int nranks, int rank, int device, const patConfig_t* config,
                                   void* handle_out) {
  if (!out || !handle_out) return patInvalidArgument;
  *out = nullptr;
  if (rank < 0 || rank >= nranks) return patRankOutOfRange;
  auto comm = std::make_unique<patComm>();
  comm->multiprocess = true;
  if (patResult_t e = common_init(comm.get(), nranks, config)) return e;
  DeviceGuard guard;
  comm->lranks.push_back(rank);
  comm->ldevs.push_back(device);
  char* pool = nullptr;
  if (patResult_t e = alloc_pool(comm.get(), device, &pool)) return e;
  comm->owned_pool.push_back(pool);
  comm->pools_ready = true;  // mapped by the peers at patCommInitRankFinish
  Handle h{};
  h.magic = kMagic;
  h.version = PAT_B200_VERSION;
  h.nranks = nranks;
  h.rank = rank;
  h.device = device;
  h.channels = comm->channels;
  h.pool_bytes = comm->pool_bytes;
  h.slot_bytes = comm->slot_bytes;
  h.config_hash = comm->config_hash = config_fingerprint(comm.get());
  h.pid = static_cast<int32_t>(getpid());
  CUDA_TRY(cudaIpcGetMemHandle(&h.ipc, pool));
  std::memset(handle_out, 0, PAT_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  if (patResult_t e = setup_groups(comm.get())) return e;
  *out = comm.release();
  return patSuccess;
}

patResult_t patCommInitRankFinish(patComm_t comm, const void* all_handles) {
  if (!comm || !all_handles || !comm->multiprocess || comm->finished) return patInvalidUsage;
  DeviceGuard guard;
  DevGroup& g = comm->groups[0];
  CUDA_TRY(cudaSetDevice(g.device));
  for (int r = 0; r < comm->n; ++r) {
    Handle h;
    std::memcpy(&h, static_cast<const char*>(all_handles) + static_cast<size_t>(r) * PAT_HANDLE_BYTES, sizeof(h));
    if (h.magic != kMagic || h.version != PAT_B200_VERSION || h.nranks != comm->n || h.rank != r ||
        h.pool_bytes != comm->pool_bytes || h.slot_bytes != comm->slot_bytes || h.channels != comm->channels ||
        h.config_hash != comm->config_hash) {
      std::fprintf(stderr,
                   "pat_b200: handle %d inconsistent (rank %d, pool %llu vs %llu, config %016llx vs %016llx): every "
                   "process must resolve the same patConfig_t and PAT_* environment\n",
                   r, h.rank, (unsigned long long)h.pool_bytes, (unsigned long long)comm->pool_bytes,
                   (unsigned long long)h.config_hash, (unsigned long long)comm->config_hash);
      return patInvalidUsage;
    }
    if (r == comm->lranks[0]) {
      g.pool_view[r] = comm->owned_pool[0];
      continue;
    }
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h.ipc, cudaIpcMemLazyEnablePeerAccess));
    comm->ipc_opened.push_back(ptr);
    g.pool_view[r] = static_cast<char*>(ptr);
  }
  comm->finished = true;
  return patSuccess;
}

patResult_t patCommDestroy(patComm_t comm) {
  if (!comm) return patInvalidArgument;
  if (comm->host_profile && comm->hp_calls)
    std::fprintf(stderr, "pat_b200 host profile: %llu calls, plan %.2f us, submit %.2f us per call\n",
                 (unsigned long long)comm->hp_calls, 1e-3 * comm->hp_plan_ns / comm->hp_calls,
                 1e-3 * comm->hp_submit_ns / comm->hp_calls);
  for (auto& w : comm->workers) w->shutdown();
  comm->workers.clear();
  {
    DeviceGuard guard;
    for (size_t l = 0; l < comm->ldevs.size(); ++l) {
      cudaSetDevice(comm->ldevs[l]);
      cudaDeviceSynchronize();
    }
    for (DevGroup& g : comm->groups) {
      cudaSetDevice(g.device);
      for (void* p : comm->ipc_opened) cudaIpcCloseMemHandle(p);
      comm->ipc_opened.clear();
      for (auto& kv : comm->ipc_cache) cudaIpcCloseMemHandle(kv.second.first);
      comm->ipc_cache.clear();
      if (g.iter_state) cudaFree(g.iter_state);
      if (g.trace) cudaFree(g.trace);
      if (g.occ) cudaFree(g.occ);
    }
    for (size_t l = 0; l < comm->owned_pool.size(); ++l) {
      cudaSetDevice(comm->ldevs[l]);
      cudaFree(comm->owned_pool[l]);
    }
    for (size_t l = 0; l < comm->events.size(); ++l)
      if (comm->events[l]) cudaEventDestroy(comm->events[l]);
    for (DevGroup& g : comm->groups)
      if (g.order_ev) cudaEventDestroy(g.order_ev);
    if (comm->err_host) cudaFreeHost(comm->err_host);
  }
  delete comm;
  return patSuccess;
}

patResult_t patCommCount(patComm_t comm, int* n) {
  if (!comm || !n) return patInvalidArgument;
  *n = comm->n;
  return patSuccess;
}

patResult_t patCommLocalRanks(patComm_t comm, int* nlocal, int* ranks, int* devices) {
  if (!comm || !nlocal) return patInvalidArgument;
  *nlocal = static_cast<int>(comm->lranks.size());
  for (size_t l = 0; l < comm->lranks.size(); ++l) {
    if (ranks) ranks[l] = comm->lranks[l];
    if (devices) devices[l] = comm->ldevs[l];
  }
  return patSuccess;
}

patResult_t patCommTraceRead(patComm_t comm, int group, void* host, size_t cap, size_t* out_bytes, int* ctas,
                             int* entries) {
  if (!comm || group < 0 || group >= static_cast<int>(comm->groups.size())) return patInvalidArgument;
  DevGroup& g = comm->groups[group];
  if (!g.trace) return patInvalidUsage;  // set PAT_TRACE=<entries> before creating the communicator
  const size_t bytes = sizeof(uint64_t) * 4 * g.trace_cap * g.trace_ctas;
  if (out_bytes) *out_bytes = bytes;
  if (ctas) *ctas = g.trace_ctas;
  if (entries) *entries = g.trace_cap;
  if (!host || cap < bytes) return patCapacity;
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(g.device));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(host, g.trace, bytes, cudaMemcpyDeviceToHost));
  return patSuccess;
}

patResult_t patCommStatsRead(patComm_t comm, int32_t* occupancy, int* nlocal, int* nrounds) {
  if (!comm || !occupancy || !nlocal || !nrounds) return patInvalidArgument;
  std::lock_guard<std::mutex> lock(comm->mu);
  DeviceGuard guard;
  *nlocal = static_cast<int>(comm->lranks.size());
  *nrounds = -1;
  for (const DevGroup& g : comm->groups) {
    if (!g.occ) return patInvalidUsage;  // communicator created without PAT_STATS
    if (g.occ_rounds < 0) continue;
    std::vector<int> h(2 * kMaxRounds * g.lidx.size());
    CUDA_TRY(cudaSetDevice(g.device));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(h.data(), g.occ, sizeof(int) * h.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < g.lidx.size(); ++i) {
      int live = 0;
      for (int t = 0; t < kMaxRounds; ++t) {
        live += h[(i * 2 + 0) * kMaxRounds + t] - h[(i * 2 + 1) * kMaxRounds + t];
        occupancy[static_cast<size_t>(g.lidx[i]) * kMaxRounds + t] = t < g.occ_rounds ? live : 0;
      }
    }
    *nrounds = g.occ_rounds;
  }
  return patSuccess;
}

patResult_t patCommGetAsyncError(patComm_t comm, patResult_t* e) {
  if (!comm || !e) return patInvalidArgument;
  *e = check_async(comm);
  return patSuccess;
}

patResult_t patCommPlan(patComm_t comm, patCollKind_t kind, size_t count, patDataType_t dtype, patPlanInfo_t* info) {
  if (!comm || !info) return patInvalidArgument;
  const size_t es = dtype_size(dtype);
  if (!es) return patInvalidArgument;
  std::lock_guard<std::mutex> lock(comm->mu);
  const int trees = comm->cfg.trees ? comm->cfg.trees : max_trees(comm->n);
  Compiled* cp = nullptr;
  if (patResult_t e = compile(comm, kind, trees, &cp)) return e;
  const int64_t cb = static_cast<int64_t>(count * es);
  DeviceGuard guard;
  int cap = 0;
  if (patResult_t e = channel_cap(comm, kind, dtype, 0, &cap)) return e;
  // as run_collective decides, assuming cudaMalloc'd (peer-reachable) buffers
  const bool pull_ok = !comm->multiprocess && comm->cfg.protocol != patProtoSimple &&
                       (comm->cfg.protocol == patProtoPull || (static_cast<int>(kind) == kRS && cb > kPullMinRS));
  const bool direct_ok = static_cast<int>(kind) == kAG && !comm->multiprocess && comm->cfg.direct >= 0;
  const Slicing sl = choose_slicing(comm, kind, cb, cap, pull_ok, cp->proto.nrounds, static_cast<int64_t>(es),
                                    cp->proto.pull_nacc, direct_ok);
  std::memset(info, 0, sizeof(*info));
  info->trees = trees;
  info->rounds = cp->proto.nrounds;
  info->threads = comm->cfg.threads;
  info->launches = static_cast<int>(comm->groups.size());
  info->slots_per_step = cp->proto.nslots;
  info->pool_bytes = comm->pool_bytes;  // the whole per-rank pool: flags + every protocol region
  info->bytes_sent_per_rank = static_cast<int64_t>(comm->n - 1) * cb;
  info->peak_intermediate_slots = cp->peak_slots;
  if (fused_path(comm, cp)) {  // as run_collective: local.cu, one launch, no inbox
    info->protocol = patProtoFused;
    info->channels = 0;
    info->iterations = 1;
    info->threads = 0;
    info->predicted_us = 0;
    return patSuccess;
  }
  // direct all-gather as run_collective decides it for cudaMalloc'd buffers in one process
  const bool direct = direct_ok && sl.proto == kProtoSimple;
  const bool polling = sl.proto == kProtoLL || sl.proto == kProtoLL32;
  info->protocol = sl.proto;
  info->channels = sl.channels;
  info->iterations = sl.iters;
  info->slice_bytes = static_cast<size_t>(sl.slice);
  info->predicted_us = predict_us(sl.proto, comm->n, cp->proto.nrounds, cb, sl.iters);
  info->depth = polling ? comm->depth_poll : comm->cfg.depth;
  info->staged_slots_per_step = staged_slots(sl.proto, kind, direct, cp->proto);
  info->staging_bytes_used = static_cast<size_t>(sl.channels) * info->depth * info->staged_slots_per_step *
                             static_cast<size_t>(proto_slot_stride(comm, sl.proto, cp->proto.pull_nacc));
  return patSuccess;
}

patResult_t patCommMemInfo(patComm_t comm, patMemInfo_t* info) {
  if (!comm || !info) return patInvalidArgument;
  std::lock_guard<std::mutex> lock(comm->mu);
  std::memset(info, 0, sizeof(*info));
  info->pool_bytes_per_rank = comm->pool_bytes;
  info->allocated_bytes = comm->pools_allocated;
  info->pools_allocated = comm->pools_ready ? 1 : 0;
  info->depth = comm->cfg.depth;
  info->depth_poll = comm->depth_poll;
  const int order[3] = {kProtoSimple, kProtoLL, kProtoLL32};
  const size_t slot[3] = {comm->slot_bytes, comm->ll_slot_bytes, comm->ll32_slot_bytes};
  for (int i = 0; i < 3; ++i) {
    info->region_channels[i] = comm->region_channels[order[i]];
    info->region_bytes[i] = comm->region_bytes[order[i]];
    info->slot_bytes[i] = slot[i];
  }
  return patSuccess;
}

patResult_t patCommRegisterPrepare(patComm_t comm, void* buf, size_t bytes, void* handle_out) {
  if (!comm || !buf || !bytes || !handle_out) return patInvalidArgument;
  if (!comm->multiprocess || !comm->finished) return patInvalidUsage;
  std::lock_guard<std::mutex> lock(comm->mu);
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(comm->ldevs[0]));
  char* base = nullptr;
  size_t size = 0;
  if (!allocation_base(buf, &base, &size) || static_cast<char*>(buf) + bytes > base + size) return patInvalidArgument;
  if (!legacy_ipc_capable(buf)) {
    std::fprintf(stderr, "pat_b200: patCommRegisterPrepare needs cudaMalloc memory (CUDA IPC)\n");
    return patInvalidUsage;
  }
  RegHandle h{};
  h.magic = kMagic;
  h.version = PAT_B200_VERSION;
  h.nranks = comm->n;
  h.rank = comm->lranks[0];
  h.bytes = bytes;
  h.offset = static_cast<uint64_t>(static_cast<char*>(buf) - base);
  h.config_hash = comm->config_hash;
  CUDA_TRY(cudaIpcGetMemHandle(&h.ipc, base));
  std::memset(handle_out, 0, PAT_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  return patSuccess;
}

patResult_t patCommRegisterFinish(patComm_t comm, void* buf, const void* all_handles) {
  if (!comm || !buf || !all_handles) return patInvalidArgument;
  if (!comm->multiprocess || !comm->finished) return patInvalidUsage;
  std::lock_guard<std::mutex> lock(comm->mu);
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(comm->ldevs[0]));
  const int me = comm->lranks[0];
  std::vector<RegHandle> hs(comm->n);
  for (int r = 0; r < comm->n; ++r) {
    std::memcpy(&hs[r], static_cast<const char*>(all_handles) + static_cast<size_t>(r) * PAT_HANDLE_BYTES,
                sizeof(RegHandle));
    const RegHandle& h = hs[r];
    if (h.magic != kMagic || h.version != PAT_B200_VERSION || h.nranks != comm->n || h.rank != r ||
        h.bytes != hs[0].bytes || h.config_hash != comm->config_hash)
      return patInvalidUsage;  // every rank registers a window of the same size, in the same order
  }
  patComm::Window w;
  w.local = static_cast<char*>(buf);
  w.bytes = hs[me].bytes;
  w.id = comm->next_window++;
  for (int r = 0; r < comm->n; ++r) {
    if (r == me) {
      w.peer[r] = w.local;
      continue;
    }
    std::string key(reinterpret_cast<const char*>(&hs[r].ipc), sizeof(cudaIpcMemHandle_t));
    auto it = comm->ipc_cache.find(key);
    if (it == comm->ipc_cache.end()) {  // an allocation is opened once per process, refcounted
      void* ptr = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, hs[r].ipc, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (int q = 0; q < r; ++q)  // undo this window's references
          if (q != me) {
            auto& ent = comm->ipc_cache[w.key[q]];
            if (--ent.second == 0) {
              cudaIpcCloseMemHandle(ent.first);
              comm->ipc_cache.erase(w.key[q]);
            }
          }
        std::fprintf(stderr, "pat_b200: cudaIpcOpenMemHandle (window of rank %d): %s\n", r, cudaGetErrorString(e));
        return patUnhandledCudaError;
      }
      it = comm->ipc_cache.emplace(key, std::make_pair(static_cast<char*>(ptr), 0)).first;
    }
    ++it->second.second;
    w.key[r] = key;
    w.peer[r] = it->second.first + hs[r].offset;
  }
  comm->windows.push_back(w);
  return patSuccess;
}

patResult_t patCommDeregister(patComm_t comm, void* buf) {
  if (!comm || !buf) return patInvalidArgument;
  std::lock_guard<std::mutex> lock(comm->mu);
  DeviceGuard guard;
  for (size_t i = 0; i < comm->windows.size(); ++i) {
    if (comm->windows[i].local != buf) continue;
    CUDA_TRY(cudaSetDevice(comm->ldevs[0]));
    for (int r = 0; r < comm->n; ++r) {
      auto it = comm->ipc_cache.find(comm->windows[i].key[r]);
      if (r == comm->lranks[0] || it == comm->ipc_cache.end()) continue;
      if (--it->second.second == 0) {
        cudaIpcCloseMemHandle(it->second.first);
        comm->ipc_cache.erase(it);
      }
    }
    comm->windows.erase(comm->windows.begin() + static_cast<std::ptrdiff_t>(i));
    return patSuccess;
  }
  return patInvalidArgument;
}

patResult_t patCommBarrier(patComm_t comm, const patStream_t* streams) {
  if (!comm || !comm->finished) return patInvalidUsage;
  if (patResult_t e = check_async(comm)) return e;
  std::lock_guard<std::mutex> lock(comm->mu);
  DeviceGuard guard;
  ++comm->barrier_seq;
  if (comm->groups.size() == 1 && !comm->multiprocess) return patSuccess;  // one device: stream order
  if (patResult_t e = ensure_pools(comm)) return e;
  for (const DevGroup& g : comm->groups) {
    BPlan b{};
    for (int r = 0; r < comm->n; ++r) b.bar[r] = reinterpret_cast<uint64_t*>(g.pool_view[r] + kBarrierOff);
    b.nlocal = static_cast<int>(g.lidx.size());
    for (size_t i = 0; i < g.lidx.size(); ++i) b.rank[i] = comm->lranks[g.lidx[i]];
    b.n = comm->n;
    b.gpu = 0;
    b.seq = comm->barrier_seq;
    b.timeout_ns = static_cast<uint64_t>(comm->cfg.timeout_ms) * 1000000ull;
    b.err = comm->err_dev;
    CUDA_TRY(cudaSetDevice(g.device));
    CUDA_TRY(launch_barrier(b, streams ? reinterpret_cast<cudaStream_t>(streams[g.lidx[0]]) : nullptr));
  }
  return patSuccess;
}

patResult_t patAllGather(patComm_t comm, const void* const* sendbuffs, void* const* recvbuffs, size_t sendcount,
                         patDataType_t datatype, const patStream_t* streams) {
  if (t_group.depth > 0) return record_call(comm, kAG, sendbuffs, recvbuffs, sendcount, datatype, patSum, streams, nullptr);
  return run_collective(comm, kAG, sendbuffs, recvbuffs, sendcount, datatype, patSum, streams);
}

patResult_t patReduceScatter(patComm_t comm, const void* const* sendbuffs, void* const* recvbuffs,
                             size_t recvcount, patDataType_t datatype, patRedOp_t op, const patStream_t* streams) {
  if (t_group.depth > 0) return record_call(comm, kRS, sendbuffs, recvbuffs, recvcount, datatype, op, streams, nullptr);
  return run_collective(comm, kRS, sendbuffs, recvbuffs, recvcount, datatype, op, streams);
}

patResult_t patAllGatherSchedule(patComm_t comm, const int32_t* sched, size_t len, const void* const* sendbuffs,
                                 void* const* recvbuffs, size_t sendcount, patDataType_t datatype,
                                 const patStream_t* streams) {
  Schedule s;
  if (Err e = decode(sched, len, &s)) return to_result(e);
  if (t_group.depth > 0) return record_call(comm, kAG, sendbuffs, recvbuffs, sendcount, datatype, patSum, streams, &s);
  return run_collective(comm, kAG, sendbuffs, recvbuffs, sendcount, datatype, patSum, streams, &s);
}

patResult_t patReduceScatterSchedule(patComm_t comm, const int32_t* sched, size_t len, const void* const* sendbuffs,
                                     void* const* recvbuffs, size_t recvcount, patDataType_t datatype,
                                     patRedOp_t op, const patStream_t* streams) {
  Schedule s;
  if (Err e = decode(sched, len, &s)) return to_result(e);
  if (t_group.depth > 0) return record_call(comm, kRS, sendbuffs, recvbuffs, recvcount, datatype, op, streams, &s);
  return run_collective(comm, kRS, sendbuffs, recvbuffs, recvcount, datatype, op, streams, &s);
}

patResult_t patGroupStart(void) {
  ++t_group.depth;
  return patSuccess;
}

patResult_t patGroupEnd(void) {
  if (t_group.depth <= 0) return patInvalidUsage;
  if (--t_group.depth > 0) return patSuccess;
  std::vector<PendingCall> calls;
  calls.swap(t_group.calls);
  patResult_t first = patSuccess;
  for (size_t i = 0; i < calls.size(); ++i) {
    patResult_t e;
    if (i + 1 < calls.size() && groupable(calls[i], calls[i + 1])) {
      e = run_group_pair(calls[i], calls[i + 1]);
      ++i;
    } else {
      e = run_pending(calls[i]);
    }
    if (first == patSuccess) first = e;
  }
  return first;
}

// ---------------------------------------------------------------- schedules (host only)

static patResult_t put(const std::vector<int32_t>& v, int32_t* buf, size_t cap, size_t* len) {
  if (len) *len = v.size();
  if (!buf || cap < v.size()) return patCapacity;
  std::memcpy(buf, v.data(), v.size() * sizeof(int32_t));
  return patSuccess;
}

patResult_t patScheduleBuild(int kind, int algorithm, int nranks, int trees, int32_t* buf, size_t cap, size_t* len) {
  if (kind < 0 || kind > 1 || algorithm < 0 || algorithm > 4) return patInvalidArgument;
  Schedule s;
  if (Err e = build(static_cast<Kind>(kind), static_cast<Algo>(algorithm), nranks, trees, &s)) return to_result(e);
  return put(encode(s), buf, cap, len);
}

patResult_t patScheduleMirror(const int32_t* in, size_t len, int32_t* out, size_t cap, size_t* out_len) {
  Schedule s;
  if (Err e = decode(in, len, &s)) return to_result(e);
  return put(encode(mirror(s)), out, cap, out_len);
}

patResult_t patScheduleValidate(const int32_t* sched, size_t len, int* nviolations, char* first, size_t cap) {
  if (!nviolations) return patInvalidArgument;
  Schedule s;
  if (Err e = decode(sched, len, &s)) return to_result(e);
  std::string msg;
  *nviolations = validate(s, &msg);
  if (first && cap) {
    std::strncpy(first, msg.c_str(), cap - 1);
    first[cap - 1] = 0;
  }
  return patSuccess;
}

patResult_t patScheduleStats(const int32_t* sched, size_t len, int64_t chunk_bytes, patExecStats_t* st) {
  if (!st) return patInvalidArgument;
  Schedule s;
  if (Err e = decode(sched, len, &s)) return to_result(e);
  const Stats x = schedule_stats(s, chunk_bytes);
  std::memset(st, 0, sizeof(*st));
  st->rounds = x.rounds;
  st->max_chunks_per_message = x.max_chunks;
  st->messages = x.messages;
  st->bytes_sent_per_rank = x.bytes_sent_per_rank;
  st->peak_intermediate_slots = x.peak;
  st->n_occupancy = static_cast<int32_t>(x.occupancy.size());
  for (size_t i = 0; i < x.occupancy.size() && i < 512; ++i) st->occupancy_per_round[i] = x.occupancy[i];
  return patSuccess;
}

patResult_t patScheduleTraceCsv(const int32_t* sched, size_t len, int64_t chunk_bytes, char* buf, size_t cap,
                                size_t* out_len) {
  Schedule s;
  if (Err e = decode(sched, len, &s)) return to_result(e);
  std::string out = "round,dim,split,sender,receiver,chunks,bytes\n";
  char line[160];
  for (const Round& r : s.rounds)
    for (int snd = 0; snd < s.n; ++snd) {
      const int recv = r.exchange ? (snd ^ std::abs(r.peer)) : mod_ranks(int64_t{snd} + r.peer, s.n);
      std::snprintf(line, sizeof line, "%d,%d,%d,%d,%d,%zu,%lld\n", r.index, r.dim, r.split, snd, recv,
                    r.chunks.size(), static_cast<long long>(chunk_bytes * static_cast<int64_t>(r.chunks.size())));
      out += line;
    }
  if (out_len) *out_len = out.size();
  if (!buf || cap <= out.size()) return patCapacity;
  std::memcpy(buf, out.c_str(), out.size() + 1);
  return patSuccess;
}

patResult_t patMaxTrees(int n, int* t) {
  if (!t || n < 1) return patScheduleError;
  *t = max_trees(n);
  return patSuccess;
}

patResult_t patTreesFromBuffer(int64_t b, int64_t c, int n, int* t) {
  if (!t) return patInvalidArgument;
  return to_result(trees_from_buffer(b, c, n, t));
}

patResult_t patPatBufferSlots(int n, int trees, int* slots) {
  if (!slots) return patInvalidArgument;
  *slots = pat_buffer_slots(n, trees);
  return patSuccess;
}

patResult_t patRoundCountFormula(int n, int trees, int* rounds) {
  if (!rounds) return patInvalidArgument;
  return to_result(round_count_formula(n, trees, rounds));
}

}  // extern "C"
#pragma GCC visibility pop
