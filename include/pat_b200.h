/*
 * pat_b200.h — C ABI of the B200-native PAT all-gather / reduce-scatter.
 *
 * This is the drop-in boundary for the reference's hot path (patsim, /root/reference/proj).
 * The reference exposes a C++ template API; every entry point below names the reference
 * interface it replaces (file:line, relative to /root/reference/proj). Plain pointers and
 * sizes only — no C++ or torch types. Errors are return codes (never exceptions); the
 * reference's exception classes map onto patResult_t values (see below).
 *
 *   reference (C++)                                          this ABI
 *   ---------------------------------------------------------------------------------------
 *   run_allgather(sched, Payload<T>, RunOptions)             patAllGather
 *       include/patsim/simulate.hpp:78-84, src/simulate.cpp:151-222,304-314
 *   run_reduce_scatter(sched, Payload<T>, ReduceOp, ...)     patReduceScatter
 *       include/patsim/simulate.hpp:93-96, src/simulate.cpp:224-300,316-332
 *   pat_allgather / mirror_schedule / pat_reduce_scatter      patScheduleBuild / patScheduleMirror
 *       include/patsim/algorithms.hpp:54-62, src/algorithms.cpp:191-249
 *   ring / bruck_nearest / bruck_farthest / rec. doubling    patScheduleBuild (algorithm arg)
 *       include/patsim/algorithms.hpp:33-47, src/algorithms.cpp:105-155
 *   validate(sched)                                          patScheduleValidate
 *       include/patsim/schedule.hpp:108-115, src/schedule.cpp:194-212
 *   max_trees / trees_from_buffer / pat_buffer_slots /       patMaxTrees / patTreesFromBuffer /
 *   round_count_formula                                      patPatBufferSlots / patRoundCountFormula
 *       include/patsim/algorithms.hpp:12-27, src/algorithms.cpp:49-93
 *   ExecStats (slot occupancy, bytes, messages)              patScheduleStats
 *       include/patsim/simulate.hpp:43-53, src/simulate.cpp:109-129
 *   write_trace_csv                                          patScheduleTraceCsv
 *       include/patsim/simulate.hpp:98-100, src/simulate.cpp:334-346
 *   RunOptions{mode,threads} / in-process ranks              patCommInitAll (one process, many GPUs,
 *       include/patsim/simulate.hpp:63-67                      several logical ranks per GPU allowed)
 *
 * Payload layouts are the reference's (simulate.hpp:33-41, 55-59) and NCCL's:
 *   all-gather:     sendbuff[r] = count elements; recvbuff[r] = n*count, block o = rank o's data
 *   reduce-scatter: sendbuff[s] = n*count, block d destined to rank d; recvbuff[d] = count
 *
 * Results are bit-identical to the reference executor: all-gather is a copy; reduce-scatter
 * folds in the PAT tree order of simulate.cpp (first arrival opens an accumulator, later
 * arrivals fold in round order, own contribution folded last at send, offset-0 arrivals
 * folded into the output after the own contribution), with every fold rounded to the
 * wire dtype (fp16/bf16 computed in fp32, round-to-nearest-even).
 */
#ifndef PAT_B200_H
#define PAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAT_B200_VERSION 10000 /* 1.0.0 */
#define PAT_MAX_RANKS 8        /* one 8xB200 NVSwitch box */
#define PAT_HANDLE_BYTES 128   /* per-rank exchange blob for multi-process init */

struct CUstream_st; /* cudaStream_t without pulling in the CUDA headers */
typedef struct CUstream_st* patStream_t;

typedef struct patComm* patComm_t;

typedef enum {
  /* NCCL-compatible codes */
  patSuccess = 0,
  patUnhandledCudaError = 1,
  patSystemError = 2,
  patInternalError = 3,
  patInvalidArgument = 4,
  patInvalidUsage = 5,
  patRemoteError = 6,
  /* the reference's typed exceptions (schedule.hpp:18-32, simulate.hpp:18-31) */
  patScheduleError = 20,       /* ScheduleError */
  patNonPowerOfTwo = 21,       /* NonPowerOfTwoError */
  patInvalidTreeCount = 22,    /* InvalidTreeCountError */
  patBufferTooSmall = 23,      /* BufferTooSmallError */
  patRankOutOfRange = 24,      /* RankOutOfRangeError */
  patSimulationError = 30,     /* SimulationError (wrong schedule kind, ...) */
  patPayloadShape = 31,        /* PayloadShapeError */
  patUnsupportedOp = 32,       /* UnsupportedOpError */
  patInvalidSchedule = 33,     /* InvalidScheduleError */
  patTimeout = 40,             /* device-side wait exceeded config.timeout_ms */
  patCapacity = 41             /* caller buffer too small */
} patResult_t;

/* numbering follows ncclDataType_t */
typedef enum {
  patInt8 = 0, patUint8 = 1, patInt32 = 2, patUint32 = 3, patInt64 = 4, patUint64 = 5,
  patFloat16 = 6, patFloat32 = 7, patFloat64 = 8, patBfloat16 = 9, patNumTypes = 10
} patDataType_t;

/* numbering follows ncclRedOp_t (avg not provided) */
typedef enum { patSum = 0, patProd = 1, patMax = 2, patMin = 3, patNumOps = 4 } patRedOp_t;

typedef enum { patAllGatherKind = 0, patReduceScatterKind = 1 } patCollKind_t;
typedef enum { patAlgoRing = 0, patAlgoBruckNearest = 1, patAlgoBruckFarthest = 2,
               patAlgoRecursiveDoubling = 3, patAlgoPat = 4 } patAlgorithm_t;
/* LL32: 32-byte lines {28 payload bytes, flag} written by one 32-byte store each, polled by the
   receiver: small and mid-size chunks. LL: 16-byte lines {4 B, flag, 4 B, flag} (8-byte store
   atomicity only; selectable, no longer chosen by auto).
   SIMPLE: pushed slices through the peers' inbox pools.
   PULL: receivers read the upstream's buffers (user sendbuf / recvbuf, staged RS partials);
   needs every rank's user buffers mapped in this process (patCommInitAll, cudaMalloc memory).
   Auto: LL32 while the calibrated cost model predicts it faster (or up to ll_threshold when that
   is set), then SIMPLE — except reduce-scatter
   below 128 MiB, which PULLs where possible (measured, profiles/r01_sp_simple_vs_pull.jsonl). */
typedef enum { patProtoAuto = 0, patProtoLL = 1, patProtoSimple = 2, patProtoPull = 3,
               patProtoLL32 = 5,
               patProtoFused = 6  /* reported by patCommPlan only: every rank on one device, the
                                     fused single-device executor runs the call (no transport) */
} patProtocol_t;

typedef struct {
  size_t size;              /* sizeof(patConfig_t) */
  size_t staging_bytes;     /* cap on the per-rank inbox pool (all protocol regions, flags aside);
                               0 = default (512 MiB of SIMPLE slots + the LL region) */
  size_t slice_bytes;       /* SIMPLE bytes per slot per pipeline step; 0 = 64-256 KiB from the pool budget */
  size_t ll_threshold;      /* per-rank chunk bytes up to which LL32 is used; 0 = cost model */
  int trees;                /* PAT tree count T; 0 = max_trees(n) (full aggregation) */
  int max_channels;         /* CTAs per rank; 0 = default */
  int protocol;             /* patProtocol_t */
  int timeout_ms;           /* device-side spin timeout; 0 = default 20000 */
  int threads;              /* threads per CTA, <= 512; 0 = 512 */
  int depth;                /* inbox buffers per channel (pipeline depth, >= 2); 0 = ceil(log2 n) + 1 */
  int direct;               /* all-gather zero-copy push into peers' recvbufs: -1 off, 0 auto, 1 on.
                               auto = single-process communicator whose recvbufs are reachable
                               (same device, or cudaMalloc memory with peer access) */
  int send_warps;           /* SIMPLE: warps per CTA that push (rest deliver); 0 = half */
  int fused;                /* all ranks on one device: -1 = run the transport kernel anyway,
                               0 = fused single-device executor (one read of every input, one
                               write of every output, same fold tree as the schedule) */
} patConfig_t;

/* Plan the library would launch for one call (introspection / benchmarks). */
typedef struct {
  int protocol;             /* patProtocol_t actually chosen (patProtoFused: no transport) */
  int trees;
  int rounds;               /* PAT rounds (= sync steps) */
  int channels;             /* CTAs per rank */
  int iterations;           /* pipeline steps per channel */
  int threads;              /* per CTA */
  int launches;             /* kernel launches (one per device) */
  int slots_per_step;       /* inbox slots per pipeline step (n-1) */
  size_t slice_bytes;       /* payload bytes per slot per step */
  size_t pool_bytes;        /* the whole per-rank inbox pool (flags + every protocol region) */
  int64_t bytes_sent_per_rank;   /* (n-1) * chunk bytes */
  int peak_intermediate_slots;   /* reference accounting (simulate.hpp:50) */
  double predicted_us;           /* the calibrated alpha-beta model's time for this call (comm.cpp) */
  int staged_slots_per_step;     /* inbox slots a pipeline step occupies at the receiver: n-1 landing
                                    slots (LL, LL32, SIMPLE), the schedule's accumulators (PULL
                                    reduce-scatter), 0 (direct / PULL all-gather, fused) */
  int depth;                     /* inbox buffers per channel for this protocol */
  size_t staging_bytes_used;     /* bytes of the inbox this call touches per rank:
                                    channels x depth x staged_slots_per_step x slot stride */
} patPlanInfo_t;

/* Memory the communicator holds (this process). */
typedef struct {
  size_t pool_bytes_per_rank;    /* flags + every protocol region of one rank's inbox pool */
  size_t allocated_bytes;        /* inbox pool bytes allocated by this process (all its ranks);
                                    0 while a one-device communicator only ran fused calls */
  int pools_allocated;           /* 1 once this process's pools exist */
  int depth;                     /* SIMPLE / PULL inbox buffers per channel */
  int depth_poll;                /* LL / LL32 inbox buffers per channel */
  int region_channels[4];        /* SIMPLE(+PULL), LL, LL32, (unused) */
  size_t region_bytes[4];
  size_t slot_bytes[4];          /* slot size per region (SIMPLE slice, LL slot, LL32 slot) */
} patMemInfo_t;

/* ExecStats (simulate.hpp:43-53) computed from a schedule; chunk_bytes as given. */
typedef struct {
  int32_t rounds;
  int32_t max_chunks_per_message;
  int64_t messages;
  int64_t bytes_sent_per_rank;
  int32_t peak_intermediate_slots;
  int32_t n_occupancy;
  int32_t occupancy_per_round[512];
} patExecStats_t;

const char* patGetErrorString(patResult_t result);
patResult_t patGetVersion(int* version);
patResult_t patConfigInit(patConfig_t* config);

/* ---- communicators ---------------------------------------------------------------- */

/* One process drives every rank (ncclCommInitAll analogue; the reference's in-process
 * ranks). devlist[r] is the CUDA device of rank r; a device may repeat, in which case its
 * ranks run inside ONE cooperative kernel per call ("local mode", e.g. 8 logical ranks on
 * one GPU). Peer access is enabled between distinct devices. NULL devlist = 0..n-1. */
patResult_t patCommInitAll(patComm_t* comm, int nranks, const int* devlist, const patConfig_t* config);

/* One process per rank (torchrun). Step 1 allocates this rank's inbox pool on `device`
 * and writes a PAT_HANDLE_BYTES blob; the caller all-gathers the blobs (any transport) and
 * passes all nranks blobs, rank-ordered, to step 2, which maps the peers' pools (CUDA IPC). */
patResult_t patCommInitRankPrepare(patComm_t* comm, int nranks, int rank, int device,
                                   const patConfig_t* config, void* handle_out);
patResult_t patCommInitRankFinish(patComm_t comm, const void* all_handles);

patResult_t patCommDestroy(patComm_t comm);
patResult_t patCommCount(patComm_t comm, int* nranks);
/* Ranks driven by this communicator, in the order the array arguments use. */
patResult_t patCommLocalRanks(patComm_t comm, int* nlocal, int* ranks, int* devices);
/* Device event trace of the last transport launch on device group `group` (communicators
 * created with PAT_TRACE=<entries per CTA role> in the environment). Layout: ctas x 2 roles
 * (push, deliver) x entries x {globaltimer ns, code}; code bits 56..63 event, 40..55 step,
 * 32..39 round. Synchronises the device. */
patResult_t patCommTraceRead(patComm_t comm, int group, void* host, size_t cap, size_t* out_bytes, int* ctas,
                             int* entries);
/* Intermediate-slot occupancy after every round, counted by the device during the last SIMPLE
 * launch (first pipeline step, channel 0) of a communicator created with PAT_STATS=1 in the
 * environment: occupancy[l * 8 + t] for local rank l, round t < *nrounds — the reference's
 * ExecStats.occupancy_per_round (simulate.hpp:43-53), measured instead of replayed. Synchronises. */
patResult_t patCommStatsRead(patComm_t comm, int32_t* occupancy, int* nlocal, int* nrounds);
/* Device-reported asynchronous error (timeouts); readable without synchronising. */
patResult_t patCommGetAsyncError(patComm_t comm, patResult_t* async_error);
patResult_t patCommPlan(patComm_t comm, patCollKind_t kind, size_t count, patDataType_t dtype,
                        patPlanInfo_t* info);
patResult_t patCommMemInfo(patComm_t comm, patMemInfo_t* info);

/* Device-side barrier on the given streams (one entry per local rank; the first stream of each
 * device is used): returns once enqueued; the kernels complete when every rank reached its
 * barrier. Every rank calls it the same number of times. A no-op with one device. */
patResult_t patCommBarrier(patComm_t comm, const patStream_t* streams);

/* ---- symmetric user-buffer windows (one process per rank; zero copy) -------------------
 * The paper's way around staging is to register the user buffers (NCCL's
 * ncclCommRegister / symmetric windows). Collective over a multi-process communicator: every
 * rank calls Prepare with a window of the same byte size (cudaMalloc memory, e.g. PyTorch's
 * caching allocator), all-gathers the PAT_HANDLE_BYTES blobs (like init) and calls Finish with
 * them, rank-ordered; windows are matched by registration order. Afterwards, a call whose
 * all-gather recvbuf (direct push) or reduce-scatter sendbuf (PULL) lies inside a window runs
 * zero copy, provided every rank passes its buffer at the SAME offset of its window — the
 * kernels check that at entry (a mismatch is the asynchronous error patInvalidUsage).
 * Deregister is local and must follow the completion of every call that used the window. */
patResult_t patCommRegisterPrepare(patComm_t comm, void* buf, size_t bytes, void* handle_out);
patResult_t patCommRegisterFinish(patComm_t comm, void* buf, const void* all_handles);
patResult_t patCommDeregister(patComm_t comm, void* buf);

/* ---- collectives (asynchronous on the given streams) ----------------------------------
 * Array arguments are indexed by local rank (patCommLocalRanks order): one entry per rank
 * this communicator drives. Ranks sharing a device are launched as one kernel on the stream
 * of the first of them (the others' streams are joined with events). In-place all-gather
 * (sendbuff == recvbuff + rank*count) is allowed. count == 0 is a no-op. */
patResult_t patAllGather(patComm_t comm, const void* const* sendbuffs, void* const* recvbuffs,
                         size_t sendcount, patDataType_t datatype, const patStream_t* streams);
patResult_t patReduceScatter(patComm_t comm, const void* const* sendbuffs, void* const* recvbuffs,
                             size_t recvcount, patDataType_t datatype, patRedOp_t op,
                             const patStream_t* streams);

/* Groups (NCCL's ncclGroupStart / ncclGroupEnd, per host thread): the collectives issued between
 * the outermost patGroupStart and patGroupEnd are launched at patGroupEnd. An all-gather followed
 * by a reduce-scatter (sum) of the same communicator on the same streams becomes ONE launch per
 * device — each call on half of the channels — so the two calls run at the same time; other calls
 * are launched one by one, in order. Calls in a group must not depend on each other; their
 * buffers must stay valid until patGroupEnd. Errors of recorded calls are returned by patGroupEnd. */
patResult_t patGroupStart(void);
patResult_t patGroupEnd(void);

/* Same collectives over an explicit, caller-supplied rank-relative schedule (any validated
 * non-exchange schedule of the communicator's rank count: PAT with any T, ring, Bruck), the
 * generic executor of the reference (run_allgather/run_reduce_scatter take a schedule,
 * simulate.hpp:78-96). Errors as the reference: patSimulationError for a schedule of the
 * wrong kind, patInvalidSchedule when validate() reports violations (simulate.cpp:72-85). */
patResult_t patAllGatherSchedule(patComm_t comm, const int32_t* sched, size_t len, const void* const* sendbuffs,
                                 void* const* recvbuffs, size_t sendcount, patDataType_t datatype,
                                 const patStream_t* streams);
patResult_t patReduceScatterSchedule(patComm_t comm, const int32_t* sched, size_t len,
                                     const void* const* sendbuffs, void* const* recvbuffs, size_t recvcount,
                                     patDataType_t datatype, patRedOp_t op, const patStream_t* streams);

/* ---- schedules (host only; no GPU needed) ---------------------------------------------
 * Flat int32 encoding: [kind, algorithm, n_ranks, has_params, trees, buffer_slots, nrounds,
 * then per round: round_index, dimension, split_index, peer, exchange, nchunks, offsets...] */
patResult_t patScheduleBuild(int kind, int algorithm, int nranks, int trees,
                             int32_t* buf, size_t cap, size_t* len);
patResult_t patScheduleMirror(const int32_t* sched, size_t len, int32_t* out, size_t cap, size_t* out_len);
patResult_t patScheduleValidate(const int32_t* sched, size_t len, int* nviolations,
                                char* first_message, size_t message_cap);
patResult_t patScheduleStats(const int32_t* sched, size_t len, int64_t chunk_bytes, patExecStats_t* stats);
patResult_t patScheduleTraceCsv(const int32_t* sched, size_t len, int64_t chunk_bytes,
                                char* buf, size_t cap, size_t* out_len);
patResult_t patMaxTrees(int nranks, int* trees);
patResult_t patTreesFromBuffer(int64_t buffer_bytes, int64_t chunk_bytes, int nranks, int* trees);
patResult_t patPatBufferSlots(int nranks, int trees, int* slots);
patResult_t patRoundCountFormula(int nranks, int trees, int* rounds);

#ifdef __cplusplus
}
#endif
#endif /* PAT_B200_H */
