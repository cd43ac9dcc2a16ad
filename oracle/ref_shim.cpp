// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile together with the reference sources where they lie
// (/root/reference/proj/src/{schedule,algorithms,simulate,oracle,costmodel}.cpp) into
// oracle/_ref/libpatsim_ref.so. Used only to (1) generate the golden fixtures in
// tests/golden/ (tests/golden/make_golden.py) and (2) time the reference's own CPU
// path in bench.py (--impl reference, cpu_baseline). Nothing here is product code.
//
// Schedules cross this boundary in the flat int32 encoding of oracle/pat_oracle.h.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "patsim/algorithms.hpp"
#include "patsim/oracle.hpp"
#include "patsim/schedule.hpp"
#include "patsim/serialize.hpp"
#include "patsim/simulate.hpp"

using namespace patsim;

namespace {

thread_local std::string g_last_error;

int code_of(const std::exception& e) {
  if (dynamic_cast<const ParseError*>(&e)) return 30;
  if (dynamic_cast<const NonPowerOfTwoError*>(&e)) return 2;
  if (dynamic_cast<const InvalidTreeCountError*>(&e)) return 3;
  if (dynamic_cast<const BufferTooSmallError*>(&e)) return 4;
  if (dynamic_cast<const RankOutOfRangeError*>(&e)) return 5;
  if (dynamic_cast<const ScheduleError*>(&e)) return 1;
  if (dynamic_cast<const PayloadShapeError*>(&e)) return 11;
  if (dynamic_cast<const UnsupportedOpError*>(&e)) return 12;
  if (dynamic_cast<const InvalidScheduleError*>(&e)) return 13;
  if (dynamic_cast<const SimulationError*>(&e)) return 10;
  return 99;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return code_of(e);
  }
}

int encode(const RelativeSchedule& s, int32_t* buf, int64_t cap, int64_t* len) {
  std::vector<int32_t> v;
  v.push_back(s.kind == CollectiveKind::AllGather ? 0 : 1);
  v.push_back(static_cast<int32_t>(s.algorithm));
  v.push_back(s.n_ranks);
  v.push_back(s.params ? 1 : 0);
  v.push_back(s.params ? s.params->trees : 0);
  v.push_back(s.params ? s.params->buffer_slots : 0);
  v.push_back(static_cast<int32_t>(s.rounds.size()));
  for (const RelativeRound& r : s.rounds) {
    v.push_back(r.round_index);
    v.push_back(r.dimension);
    v.push_back(r.split_index);
    v.push_back(r.peer_send_offset);
    v.push_back(r.exchange ? 1 : 0);
    v.push_back(static_cast<int32_t>(r.chunk_offsets.size()));
    for (int k : r.chunk_offsets) v.push_back(k);
  }
  *len = static_cast<int64_t>(v.size());
  if (*len > cap) return 20;
  std::memcpy(buf, v.data(), v.size() * sizeof(int32_t));
  return 0;
}

RelativeSchedule decode(const int32_t* s, int64_t len) {
  if (len < 7) throw ScheduleError("short schedule encoding");
  RelativeSchedule out;
  out.kind = s[0] == 0 ? CollectiveKind::AllGather : CollectiveKind::ReduceScatter;
  out.algorithm = static_cast<Algorithm>(s[1]);
  out.n_ranks = s[2];
  if (s[3]) out.params = PatParams{s[4], s[5]};
  int64_t p = 7;
  for (int t = 0; t < s[6]; t++) {
    if (p + 6 > len) throw ScheduleError("truncated schedule encoding");
    RelativeRound r;
    r.round_index = s[p];
    r.dimension = s[p + 1];
    r.split_index = s[p + 2];
    r.peer_send_offset = s[p + 3];
    r.exchange = s[p + 4] != 0;
    const int nk = s[p + 5];
    p += 6;
    if (p + nk > len) throw ScheduleError("truncated schedule encoding");
    for (int i = 0; i < nk; i++) r.chunk_offsets.push_back(s[p + i]);
    p += nk;
    out.rounds.push_back(std::move(r));
  }
  return out;
}

void fill_stats(const ExecStats& st, int64_t* out) {
  // [rounds, messages, max_chunks, bytes_per_rank, peak, n_occ, occ...]
  out[0] = st.rounds;
  out[1] = st.messages;
  out[2] = st.max_chunks_per_message;
  out[3] = st.bytes_sent_per_rank;
  out[4] = st.peak_intermediate_slots;
  out[5] = static_cast<int64_t>(st.occupancy_per_round.size());
  for (size_t i = 0; i < st.occupancy_per_round.size() && i < 512; i++)
    out[6 + i] = st.occupancy_per_round[i];
}

RunOptions options_of(int mode, int threads) {
  RunOptions o;
  o.mode = mode ? ExecMode::Parallel : ExecMode::Lockstep;
  o.threads = threads;
  return o;
}

template <class T>
Payload<T> payload_of(int n, int64_t elems, int64_t nchunks, const T* in) {
  Payload<T> p;
  p.n_ranks = n;
  p.elements_per_chunk = static_cast<int>(elems);
  p.chunks.resize(nchunks);
  for (int64_t c = 0; c < nchunks; c++) p.chunks[c].assign(in + c * elems, in + (c + 1) * elems);
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_schedule(int kind, int algo, int n, int trees, int32_t* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    RelativeSchedule s;
    switch (algo) {
      case 0: s = ring_allgather(n); break;
      case 1: s = bruck_nearest(n); break;
      case 2: s = bruck_farthest(n); break;
      case 3: s = recursive_doubling(n); break;
      default: s = pat_allgather(n, trees); break;
    }
    if (kind == 1) s = mirror_schedule(s);
    return encode(s, buf, cap, len);
  });
}

// schedule_to_json / schedule_from_json (serialize.cpp:49-101): the schedule file format
int64_t ref_schedule_to_json(const int32_t* in, int64_t in_len, int indent, char* out, int64_t cap) {
  int64_t n = -1;
  guarded([&] {
    const std::string t = schedule_to_json(decode(in, in_len), indent);
    n = static_cast<int64_t>(t.size());
    if (out && cap > n) std::memcpy(out, t.c_str(), t.size() + 1);
    return 0;
  });
  return n;
}

int ref_schedule_from_json(const char* text, int32_t* out, int64_t cap, int64_t* len) {
  return guarded([&] { return encode(schedule_from_json(text), out, cap, len); });
}

int ref_mirror(const int32_t* in, int64_t in_len, int32_t* out, int64_t cap, int64_t* len) {
  return guarded([&] { return encode(mirror_schedule(decode(in, in_len)), out, cap, len); });
}

int ref_validate(const int32_t* s, int64_t len, char* msg, int cap) {
  return guarded([&] {
    auto v = validate(decode(s, len));
    if (cap > 0) {
      std::string m = v.empty() ? std::string() : v.front().message;
      std::strncpy(msg, m.c_str(), cap - 1);
      msg[cap - 1] = 0;
    }
    return -static_cast<int>(v.size());  // <= 0: negated violation count
  });
}

int ref_max_trees(int n) { return max_trees(n); }
int ref_pat_buffer_slots(int n, int t) { return pat_buffer_slots(n, t); }
int ref_trees_from_buffer(int64_t b, int64_t c, int n, int* out) {
  return guarded([&] { *out = trees_from_buffer(b, c, n); return 0; });
}
int ref_round_count_formula(int n, int t, int* out) {
  return guarded([&] { *out = round_count_formula(n, t); return 0; });
}

// dtype 4 = int64, 8 = float64 (NCCL numbering, as in oracle/pat_oracle.h)
int ref_run_allgather(const int32_t* s, int64_t len, int dtype, int64_t elems, const void* in,
                      void* out, int64_t* stats, int mode, int threads) {
  return guarded([&] {
    RelativeSchedule sched = decode(s, len);
    const int n = sched.n_ranks;
    if (dtype == 4) {
      auto r = run_allgather(sched, payload_of(n, elems, n, static_cast<const int64_t*>(in)),
                             options_of(mode, threads));
      for (int i = 0; i < n; i++)
        std::memcpy(static_cast<int64_t*>(out) + i * n * elems, r.outputs[i].data(), n * elems * 8);
      if (stats) fill_stats(r.stats, stats);
    } else {
      auto r = run_allgather(sched, payload_of(n, elems, n, static_cast<const double*>(in)),
                             options_of(mode, threads));
      for (int i = 0; i < n; i++)
        std::memcpy(static_cast<double*>(out) + i * n * elems, r.outputs[i].data(), n * elems * 8);
      if (stats) fill_stats(r.stats, stats);
    }
    return 0;
  });
}

int ref_run_reduce_scatter(const int32_t* s, int64_t len, int dtype, int64_t elems,
                           const void* in, void* out, int64_t* stats, int mode, int threads) {
  return guarded([&] {
    RelativeSchedule sched = decode(s, len);
    const int n = sched.n_ranks;
    if (dtype == 4) {
      auto r = run_reduce_scatter(
          sched, payload_of(n, elems, (int64_t)n * n, static_cast<const int64_t*>(in)),
          ReduceOp::WrappingIntSum, options_of(mode, threads));
      for (int i = 0; i < n; i++)
        std::memcpy(static_cast<int64_t*>(out) + i * elems, r.outputs[i].data(), elems * 8);
      if (stats) fill_stats(r.stats, stats);
    } else {
      auto r = run_reduce_scatter(
          sched, payload_of(n, elems, (int64_t)n * n, static_cast<const double*>(in)),
          ReduceOp::FloatSum, options_of(mode, threads));
      for (int i = 0; i < n; i++)
        std::memcpy(static_cast<double*>(out) + i * elems, r.outputs[i].data(), elems * 8);
      if (stats) fill_stats(r.stats, stats);
    }
    return 0;
  });
}

// Seeded payloads straight from the reference (oracle.cpp:92-112).
int ref_random_payload(int rs, int dtype, int n, int64_t elems, uint64_t seed, void* out) {
  return guarded([&] {
    if (dtype == 4) {
      auto p = rs ? random_reduce_scatter_payload(n, (int)elems, seed)
                  : random_allgather_payload(n, (int)elems, seed);
      for (size_t c = 0; c < p.chunks.size(); c++)
        std::memcpy(static_cast<int64_t*>(out) + c * elems, p.chunks[c].data(), elems * 8);
    } else {
      auto p = rs ? random_reduce_scatter_payload_f64(n, (int)elems, seed)
                  : random_allgather_payload_f64(n, (int)elems, seed);
      for (size_t c = 0; c < p.chunks.size(); c++)
        std::memcpy(static_cast<double*>(out) + c * elems, p.chunks[c].data(), elems * 8);
    }
    return 0;
  });
}

int ref_oracle_reduce_scatter(int dtype, int n, int64_t elems, const void* in, void* out) {
  return guarded([&] {
    if (dtype == 4) {
      auto o = oracle_reduce_scatter(payload_of(n, elems, (int64_t)n * n, static_cast<const int64_t*>(in)),
                                     ReduceOp::WrappingIntSum);
      for (int i = 0; i < n; i++) std::memcpy(static_cast<int64_t*>(out) + i * elems, o[i].data(), elems * 8);
    } else {
      auto o = oracle_reduce_scatter(payload_of(n, elems, (int64_t)n * n, static_cast<const double*>(in)),
                                     ReduceOp::FloatSum);
      for (int i = 0; i < n; i++) std::memcpy(static_cast<double*>(out) + i * elems, o[i].data(), elems * 8);
    }
    return 0;
  });
}

int64_t ref_trace_csv(const int32_t* s, int64_t len, int64_t chunk_bytes, char* buf, int64_t cap) {
  try {
    std::ostringstream os;
    write_trace_csv(os, decode(s, len), chunk_bytes);
    std::string str = os.str();
    if ((int64_t)str.size() < cap) std::memcpy(buf, str.c_str(), str.size() + 1);
    return static_cast<int64_t>(str.size());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -1;
  }
}

// Prepared workload for timing the reference's own CPU path (bench.py --impl reference and
// cpu_baseline): the schedules and the seeded Payload<T>s (oracle.cpp:92-112) are built ONCE
// here, so a timed step is exactly the reference's run_allgather(int64) +
// run_reduce_scatter(double, FloatSum) — no marshalling from flat arrays, no copy-out (the
// returned CollectiveResult is the reference's own allocation and is dropped).
struct RefWorkload {
  RelativeSchedule ag, rs;
  Payload<std::int64_t> ag_in;
  Payload<double> rs_in;
  RunOptions opt;
};

void* ref_prepare(int n, int trees, int64_t elems, int mode, int threads) {
  RefWorkload* w = nullptr;
  guarded([&] {
    auto p = std::make_unique<RefWorkload>();
    p->ag = pat_allgather(n, trees);
    p->rs = pat_reduce_scatter(n, trees);
    p->ag_in = random_allgather_payload(n, static_cast<int>(elems), 0);
    p->rs_in = random_reduce_scatter_payload_f64(n, static_cast<int>(elems), 1);
    p->opt = options_of(mode, threads);
    w = p.release();
    return 0;
  });
  return w;
}

// which: bit 0 = all-gather, bit 1 = reduce-scatter
int ref_run_prepared(void* h, int which) {
  return guarded([&] {
    auto* w = static_cast<RefWorkload*>(h);
    if (which & 1) (void)run_allgather(w->ag, w->ag_in, w->opt);
    if (which & 2) (void)run_reduce_scatter(w->rs, w->rs_in, ReduceOp::FloatSum, w->opt);
    return 0;
  });
}

void ref_free_prepared(void* h) { delete static_cast<RefWorkload*>(h); }

// Acceptance-style sweep straight from the reference (oracle.cpp:237-282), for the record.
int ref_oracle_sweep(int n_min, int n_max, int elems, int64_t* mismatches) {
  return guarded([&] {
    SweepOptions o;
    o.n_min = n_min;
    o.n_max = n_max;
    o.elements_per_chunk = elems;
    *mismatches = static_cast<int64_t>(oracle_sweep(o).size());
    return 0;
  });
}

}  // extern "C"
