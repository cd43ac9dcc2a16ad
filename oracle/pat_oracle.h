/*
 * pat_oracle.h — CPU restatement of the reference's PAT path (TEST INFRASTRUCTURE ONLY).
 *
 * This header and pat_oracle.c are the parity checker for the B200 product in
 * paper_2506_20252_b200/. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product never links it.
 *
 * Reference: /root/reference/proj (patsim, C++20). Each function cites the
 * reference file:line it restates. Parity of this restatement is pinned by
 * tests/test_oracle_golden.py against fixtures produced by the reference
 * itself (oracle/_ref, built from the reference sources by oracle/Makefile;
 * generator script tests/golden/make_golden.py).
 *
 * Schedules use the flat int32 encoding shared with the product C-ABI
 * (include/pat_b200.h, PAT_SCHED_* layout):
 *   [kind, algorithm, n_ranks, has_params, trees, buffer_slots, nrounds,
 *    then per round: round_index, dimension, split_index, peer, exchange,
 *    nchunks, offsets[nchunks]...]
 */
#ifndef PAT_ORACLE_H
#define PAT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CollectiveKind (schedule.hpp:11) */
enum { PO_ALLGATHER = 0, PO_REDUCESCATTER = 1 };
/* Algorithm (schedule.hpp:13) */
enum { PO_RING = 0, PO_BRUCK_NEAREST = 1, PO_BRUCK_FARTHEST = 2, PO_RECURSIVE_DOUBLING = 3, PO_PAT = 4 };

/* Error codes: the reference's exception hierarchy (schedule.hpp:18-32, simulate.hpp:18-31). */
enum {
  PO_OK = 0,
  PO_SCHEDULE_ERROR = 1,
  PO_NON_POWER_OF_TWO = 2,
  PO_INVALID_TREE_COUNT = 3,
  PO_BUFFER_TOO_SMALL = 4,
  PO_RANK_OUT_OF_RANGE = 5,
  PO_SIMULATION_ERROR = 10,
  PO_PAYLOAD_SHAPE = 11,
  PO_UNSUPPORTED_OP = 12,
  PO_INVALID_SCHEDULE = 13,
  PO_CAPACITY = 20
};

/* Data types: numbering follows NCCL's ncclDataType_t, as does the product. */
enum {
  PO_INT8 = 0, PO_UINT8 = 1, PO_INT32 = 2, PO_UINT32 = 3, PO_INT64 = 4, PO_UINT64 = 5,
  PO_FLOAT16 = 6, PO_FLOAT32 = 7, PO_FLOAT64 = 8, PO_BFLOAT16 = 9
};
/* Reduction ops: numbering follows ncclRedOp_t. */
enum { PO_SUM = 0, PO_PROD = 1, PO_MAX = 2, PO_MIN = 3 };

/* ExecStats (simulate.hpp:43-53); fixed layout for the C boundary. */
typedef struct {
  int32_t rounds;
  int32_t max_chunks_per_message;
  int64_t messages;
  int64_t bytes_sent_per_rank;
  int32_t peak_intermediate_slots;
  int32_t n_occupancy;
  int32_t occupancy_per_round[512];
} po_stats;

size_t po_dtype_size(int dtype);

/* schedule.hpp:37-47, algorithms.cpp:49-103 */
int po_ceil_log2(int64_t v);
int po_mod_ranks(int64_t value, int n);
int po_max_trees(int n);
int po_trees_from_buffer(int64_t buffer_bytes, int64_t chunk_bytes, int n, int* trees_out);
int po_pat_buffer_slots(int n, int trees);
int po_round_count_formula(int n, int trees, int* out);
int po_sendable_offsets(int n, int dim, int32_t* out, int cap);

/* Generators (algorithms.cpp:105-249). Return PO_* code; *len = int32 words written. */
int po_schedule(int kind, int algorithm, int n, int trees, int32_t* buf, int64_t cap, int64_t* len);
int po_mirror(const int32_t* in, int64_t in_len, int32_t* out, int64_t cap, int64_t* len);

/* validate (schedule.cpp:194-212): returns number of violations; first message copied. */
int po_validate(const int32_t* sched, int64_t len, char* first_msg, int msg_cap);

/* Executors (simulate.cpp:151-300).
 * allgather: in = n chunks of elems (rank r at r*elems), out = n * (n*elems).
 * reduce_scatter: in = n*n chunks (chunks[s*n+d] at (s*n+d)*elems), out = n * elems. */
int po_run_allgather(const int32_t* sched, int64_t len, int dtype, int64_t elems,
                     const void* in, void* out, po_stats* stats);
int po_run_reduce_scatter(const int32_t* sched, int64_t len, int dtype, int op, int64_t elems,
                          const void* in, void* out, po_stats* stats);

/* Definitional references (oracle.cpp:15-40): concatenation; rank-order fold. */
int po_oracle_allgather(int n, int dtype, int64_t elems, const void* in, void* out);
int po_oracle_reduce_scatter(int n, int dtype, int op, int64_t elems, const void* in, void* out);

/* Closed-form PAT reduction tree for one element column, used as a
 * second, schedule-free statement of the floating-point order. x[j] = contribution of
 * rank (r+j) mod n to r. */
int po_tree_fold(int n, int dtype, int op, const void* x, void* result);

/* Seeded payloads (oracle.cpp:42-62 for int64/f64; SURVEY §8d for the rest). */
void po_random_payload(int dtype, int64_t nchunks, int64_t elems, uint64_t seed, void* out);

/* mt19937_64 raw draws (for tests of the generator itself). */
void po_mt19937_64(uint64_t seed, int64_t count, uint64_t* out);

/* Element-wise fold a = a (op) b with per-hop rounding in the wire dtype. */
int po_fold(int dtype, int op, void* a, const void* b, int64_t elems);

/* write_trace_csv (simulate.cpp:334-346) into buf; returns bytes (excl NUL) or -1. */
int64_t po_trace_csv(const int32_t* sched, int64_t len, int64_t chunk_bytes, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
