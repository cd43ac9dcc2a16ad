// ce.cpp — copy-engine executor of PAT all-gather / reduce-scatter (see ce.hpp).
//
// A call is cut into S slices of every chunk; slice s runs through the PAT rounds like the
// transport kernel's pipeline step (kernels: transport.cuh), enqueued skewed (host iteration k
// issues round t of slice k - t) so each stream always has independent work queued ahead of
// work that waits. Per rank r, on the caller's stream:
//   all-gather     round t copies the |K_t| chunk slices straight into the peer's recvbuf at
//                  their origin block (simulate.cpp:186-212); a forwarded chunk is read from
//                  r's own recvbuf, where its upstream delivered it. No staging at all.
//   reduce-scatter round t copies each message into the peer's inbox slot: a leaf straight from
//                  r's sendbuf, a forwarded offset from r's staging, where a fold kernel (on
//                  r's fold stream) computed fold(arrivals in round order) (+) own
//                  (simulate.cpp:257-266, 281-285). The output is own (+) offset-0 arrivals in
//                  round order (simulate.cpp:239, 278-279), folded once they are in.
// Event edges replace the kernels' flags: copy_ev (data of (slice, round) landed), fold_ev
// (message staged), fin_ev (a slice's inbox may be reused), entry_ev / done_ev (call bounds).
#include "ce.hpp"

#include <algorithm>
#include <cstdio>

namespace pat {

namespace {

#define CE_TRY(x)                                 \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return static_cast<int>(e_); \
  } while (0)

constexpr int kE = kMaxRounds + 1;  // event ring per rank; > any (round - dependency round) distance

cudaEvent_t& ev2(std::vector<cudaEvent_t>& v, int r, int s, int t) { return v[(r * kE + s % kE) * kMaxRounds + t]; }
cudaEvent_t& ev1(std::vector<cudaEvent_t>& v, int r, int s) { return v[r * kE + s % kE]; }

}  // namespace

int ce_init(CeState& st, int n, const int* devices, int /*max_rounds*/) {
  st.n = n;
  st.E = kE;
  st.dev.assign(devices, devices + n);
  st.sms.assign(n, 0);
  st.fold_stream.assign(n, nullptr);
  st.buf.assign(n, nullptr);
  int prev = 0;
  cudaGetDevice(&prev);
  int rc = 0;
  for (int r = 0; r < n && !rc; ++r) {
    if ((rc = cudaSetDevice(st.dev[r]))) break;
    if ((rc = cudaDeviceGetAttribute(&st.sms[r], cudaDevAttrMultiProcessorCount, st.dev[r]))) break;
    if ((rc = cudaStreamCreateWithFlags(&st.fold_stream[r], cudaStreamNonBlocking))) break;
  }
  // events live on the device that records them: create each rank's on its device
  st.copy_ev.assign(static_cast<size_t>(n) * kE * kMaxRounds, nullptr);
  st.fold_ev.assign(static_cast<size_t>(n) * kE * kMaxRounds, nullptr);
  st.fin_ev.assign(static_cast<size_t>(n) * kE, nullptr);
  st.entry_ev.assign(n, nullptr);
  st.done_ev.assign(n, nullptr);
  for (int r = 0; r < n && !rc; ++r) {
    if ((rc = cudaSetDevice(st.dev[r]))) break;
    auto mk = [&](cudaEvent_t& e) { if (!rc) rc = cudaEventCreateWithFlags(&e, cudaEventDisableTiming); };
    for (int i = 0; i < kE * kMaxRounds; ++i) {
      mk(st.copy_ev[static_cast<size_t>(r) * kE * kMaxRounds + i]);
      mk(st.fold_ev[static_cast<size_t>(r) * kE * kMaxRounds + i]);
    }
    for (int i = 0; i < kE; ++i) mk(st.fin_ev[static_cast<size_t>(r) * kE + i]);
    mk(st.entry_ev[r]);
    mk(st.done_ev[r]);
  }
  cudaSetDevice(prev);
  return rc;
}

void ce_destroy(CeState& st) {
  for (int r = 0; r < st.n; ++r) {
    cudaSetDevice(st.dev[r]);
    cudaStreamSynchronize(st.fold_stream[r]);
    if (st.buf[r]) cudaFree(st.buf[r]);
    if (st.fold_stream[r]) cudaStreamDestroy(st.fold_stream[r]);
  }
  for (auto* v : {&st.copy_ev, &st.fold_ev, &st.fin_ev, &st.entry_ev, &st.done_ev})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  st = CeState{};
}

namespace {

// Reduce-scatter inbox + staging: per rank, D buffers x nslots slots of one slice each, twice.
int ensure_buffers(CeState& st, int64_t slice, int slots, int D) {
  if (st.buf_slice >= slice && st.buf_slots >= slots && st.buf_depth >= D && st.buf[0]) return 0;
  for (int r = 0; r < st.n; ++r) {
    CE_TRY(cudaSetDevice(st.dev[r]));
    CE_TRY(cudaDeviceSynchronize());
    if (st.buf[r]) CE_TRY(cudaFree(st.buf[r]));
    st.buf[r] = nullptr;
  }
  st.buf_slice = slice;
  st.buf_slots = slots;
  st.buf_depth = D;
  const size_t bytes = 2ull * D * slots * static_cast<size_t>(slice);
  for (int r = 0; r < st.n; ++r) {
    CE_TRY(cudaSetDevice(st.dev[r]));
    CE_TRY(cudaMalloc(&st.buf[r], bytes));
  }
  return 0;
}

}  // namespace

int ce_run(CeState& st, const CeCall& c) {
  const KPlan& p = *c.sched;
  const int n = st.n, NR = p.nrounds;
  const int64_t Cb = c.chunk_bytes, slice = c.slice;
  const int S = static_cast<int>((Cb + slice - 1) / slice);
  const int D = std::min(NR + 1, kMaxRounds);  // reduce-scatter inbox/staging buffers (> rounds)
  if (c.kind == kRS && NR >= kMaxRounds) return static_cast<int>(cudaErrorInvalidValue);
  if (c.kind == kRS) {
    if (int e = ensure_buffers(st, slice, std::max(p.nslots, 1), D)) return e;
  }
  auto dev = [&](int r) { return cudaSetDevice(st.dev[r]); };
  auto inbox = [&](int r, int s, int j) {
    return st.buf[r] + (static_cast<int64_t>(s % D) * st.buf_slots + j) * st.buf_slice;
  };
  auto stage = [&](int r, int s, int j) {
    return st.buf[r] + (static_cast<int64_t>(st.buf_depth + s % D) * st.buf_slots + j) * st.buf_slice;
  };
  auto up = [&](int r, int t) { return (r - p.rounds[t].peer + n) % n; };  // who sends to r in round t

  // ---- entry: every stream reached the call; downstream buffers are free
  for (int r = 0; r < n; ++r) {
    CE_TRY(dev(r));
    CE_TRY(cudaEventRecord(st.entry_ev[r], c.stream[r]));
  }
  for (int r = 0; r < n; ++r) {
    CE_TRY(dev(r));
    bool seen[kMaxRanks] = {};
    for (int t = 0; t < NR; ++t) {
      const int P = (r + p.rounds[t].peer) % n;
      if (seen[P]) continue;
      seen[P] = true;
      CE_TRY(cudaStreamWaitEvent(c.stream[r], st.entry_ev[P], 0));  // P's recvbuf / inbox
      if (c.kind == kRS) CE_TRY(cudaStreamWaitEvent(c.stream[r], st.done_ev[P], 0));
    }
    CE_TRY(cudaStreamWaitEvent(st.fold_stream[r], st.entry_ev[r], 0));
  }
  // ---- all-gather own block (simulate.cpp:160-165) on the fold stream's SMs, beside the copies
  if (c.kind == kAG)
    for (int r = 0; r < n; ++r) {
      if (c.recv[r] + r * Cb == c.send[r]) continue;  // in place
      CE_TRY(dev(r));
      CeFold f{};
      f.nop = 1;
      f.vec = c.vec;
      f.esize = c.esize;
      f.len = Cb;
      f.op[0].dst = c.recv[r] + r * Cb;
      f.op[0].src[0] = c.send[r];
      f.op[0].m = 1;
      CE_TRY(launch_ce_fold(f, /*uint8*/ 1, /*sum*/ 0, st.sms[r], st.fold_stream[r]));  // m = 1: a copy
    }

  // ---- rounds, skewed: iteration k issues round t of slice k - t (and, for RS, the output fold
  // of slice k - NR)
  for (int k = 0; k < S + NR; ++k) {
    for (int t = 0; t <= NR; ++t) {
      const int s = k - t;
      if (s < 0 || s >= S) continue;
      const int64_t off = static_cast<int64_t>(s) * slice;
      const int64_t len = std::min(slice, Cb - off);
      for (int r = 0; r < n; ++r) {
        CE_TRY(dev(r));
        cudaStream_t sr = c.stream[r], fr = st.fold_stream[r];
        if (t == NR) {  // RS output: own (+) offset-0 arrivals in round order
          if (c.kind != kRS) continue;
          CeFold f{};
          f.nop = 1;
          f.vec = c.vec;
          f.esize = c.esize;
          f.len = len;
          f.op[0].dst = c.recv[r] + off;
          f.op[0].src[f.op[0].m++] = c.send[r] + r * Cb + off;
          for (int q = 0; q < p.nfin; ++q) {
            const int j = p.fin[q], tr = p.slot_round[j];
            CE_TRY(cudaStreamWaitEvent(fr, ev2(st.copy_ev, up(r, tr), s, tr), 0));
            f.op[0].src[f.op[0].m++] = inbox(r, s, j);
          }
          CE_TRY(launch_ce_fold(f, c.dtype, c.op, st.sms[r], fr));
          CE_TRY(cudaEventRecord(ev1(st.fin_ev, r, s), fr));
          continue;
        }
        const KRound& rd = p.rounds[t];
        const int P = (r + rd.peer) % n;
        if (c.kind == kAG) {
          // forwarded chunks arrived in earlier rounds from their upstreams
          uint32_t waited = 0;
          for (int pos = 0; pos < rd.nchunks; ++pos) {
            if (!rd.narr[pos]) continue;
            const int tr = p.slot_round[rd.arr[pos][0]];
            if ((waited >> tr) & 1u) continue;
            waited |= 1u << tr;
            CE_TRY(cudaStreamWaitEvent(sr, ev2(st.copy_ev, up(r, tr), s, tr), 0));
          }
          for (int pos = 0; pos < rd.nchunks; ++pos) {
            const int origin = (r - rd.chunk[pos] + n) % n;
            const char* src = rd.narr[pos] ? c.recv[r] + origin * Cb + off : c.send[r] + off;
            CE_TRY(cudaMemcpyAsync(c.recv[P] + origin * Cb + off, src, len, cudaMemcpyDefault, sr));
          }
          CE_TRY(cudaEventRecord(ev2(st.copy_ev, r, s, t), sr));
          continue;
        }
        // reduce-scatter: stage the forwarded messages of this round
        CeFold f{};
        f.vec = c.vec;
        f.esize = c.esize;
        f.len = len;
        uint32_t waited = 0;
        for (int pos = 0; pos < rd.nchunks; ++pos) {
          const int na = rd.narr[pos];
          if (!na) continue;
          CeFold::One& o = f.op[f.nop++];
          o.dst = stage(r, s, rd.slot_base + pos);
          for (int a = 0; a < na; ++a) {
            const int j = rd.arr[pos][a], tr = p.slot_round[j];
            if (!((waited >> tr) & 1u)) {
              waited |= 1u << tr;
              CE_TRY(cudaStreamWaitEvent(fr, ev2(st.copy_ev, up(r, tr), s, tr), 0));
            }
            o.src[o.m++] = inbox(r, s, j);
          }
          o.src[o.m++] = c.send[r] + ((r - rd.chunk[pos] + n) % n) * Cb + off;  // own folded last
        }
        if (f.nop) {
          if (s >= D) CE_TRY(cudaStreamWaitEvent(fr, ev2(st.copy_ev, r, s - D, t), 0));  // staging free
          CE_TRY(launch_ce_fold(f, c.dtype, c.op, st.sms[r], fr));
          CE_TRY(cudaEventRecord(ev2(st.fold_ev, r, s, t), fr));
          CE_TRY(cudaStreamWaitEvent(sr, ev2(st.fold_ev, r, s, t), 0));
        }
        if (s >= D) CE_TRY(cudaStreamWaitEvent(sr, ev1(st.fin_ev, P, s - D), 0));  // P's inbox free
        for (int pos = 0; pos < rd.nchunks; ++pos) {
          const char* src = rd.narr[pos] ? stage(r, s, rd.slot_base + pos)
                                         : c.send[r] + ((r - rd.chunk[pos] + n) % n) * Cb + off;
          CE_TRY(cudaMemcpyAsync(inbox(P, s, rd.slot_base + pos), src, len, cudaMemcpyDefault, sr));
        }
        CE_TRY(cudaEventRecord(ev2(st.copy_ev, r, s, t), sr));
      }
    }
  }

  // ---- exit: everything written into r (all upstreams' last copies) and r's folds are done
  for (int r = 0; r < n; ++r) {
    CE_TRY(dev(r));
    if (c.kind == kAG)
      for (int t = 0; t < NR; ++t) CE_TRY(cudaStreamWaitEvent(c.stream[r], ev2(st.copy_ev, up(r, t), S - 1, t), 0));
    CE_TRY(cudaEventRecord(st.done_ev[r], st.fold_stream[r]));
    CE_TRY(cudaStreamWaitEvent(c.stream[r], st.done_ev[r], 0));
  }
  return 0;
}

}  // namespace pat
