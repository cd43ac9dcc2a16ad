// schedule.hpp — host-side PAT step rule for the B200 runtime.
//
// Rank-relative schedules in the reference's vocabulary (schedule.hpp:56-86 of
// /root/reference/proj/include/patsim): a round is (dimension d, split, signed peer
// offset, ordered chunk offsets K); offset k at rank r names the chunk of origin
// (all-gather) / destination (reduce-scatter) rank (r - k) mod n.
//
// This is the product's own generator (the oracle in oracle/ is a separate C
// restatement used only by the tests). It is written as an explicit-stack walk over
// dimension groups rather than the reference's recursive emitter; the golden fixtures
// in tests/golden/ pin both to the reference output.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace pat {

enum class Kind : int { AllGather = 0, ReduceScatter = 1 };
enum class Algo : int { Ring = 0, BruckNearest = 1, BruckFarthest = 2, RecursiveDoubling = 3, Pat = 4 };

// Error codes mirror patResult_t (include/pat_b200.h).
enum Err : int {
  kOk = 0,
  kInvalidArgument = 4,
  kScheduleError = 20,
  kNonPowerOfTwo = 21,
  kInvalidTreeCount = 22,
  kBufferTooSmall = 23,
  kRankOutOfRange = 24,
  kSimulationError = 30,
  kPayloadShape = 31,
  kUnsupportedOp = 32,
  kInvalidSchedule = 33,
  kCapacity = 41,
};

struct Round {
  int index = 0;
  int dim = 0;
  int split = 0;
  int peer = 0;  // signed send offset, |peer| = 2^dim
  bool exchange = false;
  std::vector<int> chunks;
  bool operator==(const Round&) const = default;
};

struct Schedule {
  Kind kind = Kind::AllGather;
  Algo algo = Algo::Pat;
  int n = 1;
  bool has_params = false;
  int trees = 0;
  int buffer_slots = 0;
  std::vector<Round> rounds;
  bool operator==(const Schedule&) const = default;
};

int ceil_log2(int64_t v);
int mod_ranks(int64_t v, int n);
bool is_pow2(int64_t v);

int max_trees(int n);                                               // algorithms.cpp:49-53
int pat_buffer_slots(int n, int trees);                             // algorithms.cpp:76-81
Err trees_from_buffer(int64_t buffer, int64_t chunk, int n, int* trees);  // algorithms.cpp:61-74
Err round_count_formula(int n, int trees, int* rounds);             // algorithms.cpp:83-93
std::vector<int> sendable_offsets(int n, int dim);                  // algorithms.cpp:95-103

Err build(Kind kind, Algo algo, int n, int trees, Schedule* out);   // algorithms.cpp:105-249
Schedule mirror(const Schedule& s);                                  // algorithms.cpp:218-245
int received_offset(const Round& r, int k, int n);                   // schedule.cpp:24-32

// validate (schedule.cpp:194-212). Returns the violation count; first message stored.
int validate(const Schedule& s, std::string* first);

// ExecStats occupancy (simulate.cpp:109-129 accounting), independent of data.
struct Stats {
  int rounds = 0;
  int max_chunks = 0;
  int64_t messages = 0;
  int64_t bytes_sent_per_rank = 0;
  int peak = 0;
  std::vector<int> occupancy;
};
Stats schedule_stats(const Schedule& s, int64_t chunk_bytes);

std::vector<int32_t> encode(const Schedule& s);
Err decode(const int32_t* buf, size_t len, Schedule* out);

}  // namespace pat
