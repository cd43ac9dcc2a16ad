// ce.hpp — copy-engine executor of PAT all-gather / reduce-scatter (ce.cpp, ce_fold.cu).
//
// For the largest messages of a single-process communicator the chunk slices travel on the
// GPUs' copy engines (cudaMemcpyAsync between peer-mapped HBM) instead of SM stores: measured
// on this pool, SM-issued NVLink stores saturate at ~704 GB/s per direction when every GPU
// sends and receives at once, the copy engines at ~774 GB/s (profiles/r01_bidir_probe_g*.txt).
// The PAT schedule, its per-round peers and chunk offsets, and the reference's fold order are
// unchanged; the per-(slice, round) release/acquire flags become CUDA events between the
// ranks' streams, and reduce-scatter folds run as small SM kernels between the copies.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace pat {

struct CeFold {
  struct One {
    char* dst;
    const char* src[kMaxArr + 1];
    int m;
  };
  One op[kMaxChunks];
  int nop;
  int vec, esize;
  int64_t len;
};

cudaError_t launch_ce_fold(const CeFold& f, int dtype, int op, int sm_count, cudaStream_t stream);

// Per-communicator state of the executor: events, one internal fold stream per rank, and
// the reduce-scatter inbox/staging buffers (allocated on first use, bounded by slice size).
struct CeState {
  int n = 0, E = 0;
  std::vector<int> dev;                  // device of rank r
  std::vector<int> sms;                  // SM count of rank r's device
  std::vector<cudaStream_t> fold_stream; // per rank
  std::vector<cudaEvent_t> copy_ev;      // [r][E][kMaxRounds]: rank r's round-t copies of a slice
  std::vector<cudaEvent_t> fold_ev;      // [r][E][kMaxRounds]: rank r's round-t folds of a slice
  std::vector<cudaEvent_t> fin_ev;       // [r][E]: rank r consumed a slice (final fold)
  std::vector<cudaEvent_t> entry_ev;     // [r]: rank r's stream reached the call
  std::vector<cudaEvent_t> done_ev;      // [r]: rank r's fold stream finished the previous call
  std::vector<char*> buf;                // [r]: inbox (E x nslots) + staging (E x nslots) slices
  int64_t buf_slice = 0;
  int buf_slots = 0, buf_depth = 0;
};

struct CeCall {
  int kind, dtype, op, vec, esize;
  int64_t chunk_bytes, slice;
  const KPlan* sched;                    // compiled schedule (rounds, slots, arrivals)
  const char* const* send;               // by rank
  char* const* recv;                     // by rank
  const cudaStream_t* stream;            // by rank (the caller's streams)
};

// 0 on success, else a cudaError_t value.
int ce_init(CeState& st, int n, const int* devices, int max_rounds);
int ce_run(CeState& st, const CeCall& call);
void ce_destroy(CeState& st);

}  // namespace pat
