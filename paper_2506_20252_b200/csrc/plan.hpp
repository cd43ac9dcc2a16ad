// plan.hpp — the launch plan shared by the host runtime (comm.cpp) and the sm_100a kernels
// (kernels.cu). One KPlan is passed by value (__grid_constant__) per kernel launch; it holds
// the compiled PAT schedule, the slicing, and the pointer table of every rank's inbox pool as
// seen from the launching device.
#pragma once

#include <cstdint>

namespace pat {

constexpr int kMaxRanks = 8;    // one NVSwitch box
constexpr int kMaxRounds = 8;   // >= n-1 (single-tree PAT / ring at n = 8)
constexpr int kMaxChunks = 8;   // chunk offsets per round
constexpr int kMaxSlots = 8;    // inbox slots per pipeline step (= n-1 arrivals)
constexpr int kMaxArr = 8;      // arrivals folded into one forwarded offset
constexpr int kMaxLocal = 8;    // ranks driven by one kernel (local mode)
constexpr int kMaxChannels = 160;  // >= the 148 SMs of a B200 (channels are clamped to co-residency)
constexpr int kMaxThreads = 512;  // per CTA: 128 registers per thread for the unrolled SIMPLE loops
constexpr int kFlagWords = 32;  // per channel: data flag per round [0,8), done-from per rank [8,16),
                                // ready-from per rank [16,24) (direct mode entry handshake),
                                // window tag from each rank [24,32) (symmetric windows)

// (4 is retired: LL128, 128-byte lines with one flag word, was measured to tear over NVLink —
// a line's flag sector can land before its data sectors — and was removed. LL32's lines are
// written by ONE 32-byte store each, which lands whole: tools/atomicity_probe.cu.)
enum Proto : int { kProtoLL = 1, kProtoSimple = 2, kProtoPull = 3, kProtoLL32 = 5 };
constexpr int kNumProtoSlots = 6;

// PULL reduce-scatter: what a rank does with the arrival it pulled into slot j.
enum PullAct : int8_t {
  kOutFirst = 0,  // out = own[R] (+) m        (simulate.cpp:239, 278-279)
  kOutNext = 1,   // out = out (+) m
  kAccOnly = 2,   // stage[dst] = m (+) own     (single arrival; own folded last, :260-266)
  kAccFirst = 3,  // stage[dst] = m             (accumulator opened by the first arrival, :282-283)
  kAccMid = 4,    // stage[dst] = stage (+) m   (later arrivals in round order, :285)
  kAccLast = 5    // stage[dst] = (stage (+) m) (+) own
};
enum KindK : int { kAG = 0, kRS = 1 };

// One PAT round compiled for the kernel.
struct KRound {
  int8_t peer;        // send peer delta, (r + peer) mod n, already in [1, n)
  int8_t nchunks;
  int8_t slot_base;   // first inbox slot this round fills at the receiver
  int8_t pad;
  int8_t chunk[kMaxChunks];   // offsets k, send order
  int8_t narr[kMaxChunks];    // AG: 0 = own chunk, 1 = forward of slot arr[pos][0]
                              // RS: arrivals folded (in round order) before the own contribution
  int8_t arr[kMaxChunks][kMaxArr];
};

struct KPlan {
  int n, nrounds, nslots, nlocal;
  int kind, proto, vec, esize;
  int channels, iters;
  int chan_base;    // first channel (flags, counters, inbox) of this call: grouped calls share a launch
                    // on disjoint channel ranges [chan_base, chan_base + channels)
  int depth;        // inbox buffers per channel (pipeline depth); buffer of step g = g % depth
  int send_warps;   // SIMPLE: warps [0, send_warps) push, the rest deliver / fold
  int gpu_scope;    // all ranks on this device: flags and fences at .gpu scope instead of .sys
  int direct;       // AG: push straight into the peers' recvbufs (peer_recv), no inbox
  int skew;         // SIMPLE sender runs round t of step k - t in iteration k (needs depth >= nrounds)
  int leaves_first; // SIMPLE: a step's first task pushes the leaf chunks (no arrivals) of every round
  int64_t chunk_bytes;   // bytes of one rank chunk (AG sendcount*esize, RS recvcount*esize)
  int64_t slice_bytes;   // payload bytes per slot per pipeline step
  int64_t slot_stride;   // inbox bytes per slot
  int64_t chan_stride;   // inbox bytes per channel (depth buffers x slots per buffer x slot_stride)
  uint64_t timeout_ns;
  KRound rounds[kMaxRounds];
  int8_t slot_round[kMaxSlots];    // round whose arrival fills slot j
  int8_t slot_offset[kMaxSlots];   // received offset k' held in slot j
  int8_t nfin;                     // RS: slots holding offset-0 arrivals, round order
  int8_t fin[kMaxSlots];
  int8_t npeers;                   // distinct send peers (credit waits)
  int8_t peers[kMaxRounds];
  // PULL protocol (receiver reads the upstream's buffers): per arrival slot j
  int8_t pull_act[kMaxSlots];      // RS: PullAct
  int8_t pull_dst[kMaxSlots];      // RS: accumulator (staging slot) id folding the arrival of slot j
  int8_t pull_nacc;                // RS: accumulators per step (staging slots per buffer)
  int8_t round_dep[kMaxRounds];    // upstream round whose arrivals round t reads; -1 = own data only
  uint8_t sig_after[kMaxRounds];   // reader rounds (bitmask) that become ready when round t completes
  uint8_t stage_rounds;            // RS: bitmask of rounds that write the local staging (need credits)
  // ranks driven by this launch
  int rank[kMaxLocal];
  const char* send[kMaxLocal];
  char* recv[kMaxLocal];
  uint64_t* iter_state[kMaxLocal];  // [kMaxChannels] pipeline-step counters per rank
  // every rank's pool, mapped into this device's address space
  char* inbox[kMaxRanks];
  char* peer_recv[kMaxRanks];       // direct mode: every rank's recvbuf as seen from this device
  const char* peer_send[kMaxRanks]; // PULL: every rank's sendbuf as seen from this device
  uint64_t* flags[kMaxRanks];       // [kMaxChannels][kFlagWords]
  int* err;                         // mapped pinned host word (first async error)
  // optional device trace (PAT_TRACE=1): per (CTA, role) ring of {globaltimer ns, event code}
  uint64_t* trace;
  int trace_cap;                    // entries per (CTA, role)
  // 32-bit line flags (LL, LL32) repeat every 2^32 steps: every kernel's receiver re-stamps its
  // own polling buffers once per epoch (epoch_clean), so no line can hold a flag 2^32 steps old
  uint64_t epoch_mask;              // (1 << 31) - 1; PAT_EPOCH_SHIFT overrides (tests)
  int depth_poll;                   // LL / LL32 inbox buffers per channel
  int poll_channels[2];             // channels of the LL / LL32 regions
  int64_t poll_off[2];              // LL / LL32 region offsets from a pool's base (= flags[rank])
  int64_t poll_slot[2];             // LL / LL32 slot bytes
  // symmetric windows (multi-process zero copy): the tag (window id, offsets) of the user
  // buffers this call reads or writes at its peers; 0 = not windowed. Published to the peers
  // with the entry handshake and compared there (kernels: sym_check)
  uint64_t sym_tag;
  // PAT_STATS: live intermediate-slot counts of the call's first SIMPLE step on channel 0,
  // [nlocal][2][kMaxRounds]: slots that became held in round t / were released by round t
  // (the reference's StatsBuilder occupancy, simulate.cpp:109-129, brute_force.hpp:25-54)
  int* occ;
  int64_t region_bytes;  // bytes of the inbox region this launch uses (bounds checks, PAT_BOUNDS_CHECK builds)
};

// Two independent collectives of one communicator in one launch (patGroupStart/End): CTAs
// [0, a.nlocal * a.channels) run `a` (all-gather), the rest `b` (reduce-scatter).
struct KPlan2 {
  KPlan a, b;
};

// Device barrier (patCommBarrier): every rank's barrier words, as seen from the launching device.
struct BPlan {
  uint64_t* bar[kMaxRanks];  // [kMaxRanks] words of each rank's pool, word q = last seq from rank q
  int rank[kMaxLocal];
  int nlocal, n, gpu;
  uint64_t seq, timeout_ns;
  int* err;
};

}  // namespace pat
