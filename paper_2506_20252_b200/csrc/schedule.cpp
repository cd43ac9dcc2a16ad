// schedule.cpp — PAT step rule, mirror, validation and slot accounting (host side).
// Reference semantics: /root/reference/proj/src/algorithms.cpp, schedule.cpp,
// simulate.cpp (stats). See schedule.hpp.
#include "schedule.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>

namespace pat {

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int ceil_log2(int64_t v) {
  int d = 0;
  while ((int64_t{1} << d) < v) ++d;
  return d;
}

int mod_ranks(int64_t v, int n) {
  const int64_t m = v % n;
  return static_cast<int>(m < 0 ? m + n : m);
}

int max_trees(int n) { return n <= 2 ? 1 : 1 << (ceil_log2(n) - 1); }

int pat_buffer_slots(int n, int trees) {
  int m = 0;
  while ((int64_t{trees} << m) < n) ++m;
  return trees + m;
}

static Err check_trees(int n, int trees) {
  if (!is_pow2(trees) || trees > max_trees(n)) return kInvalidTreeCount;
  return kOk;
}

Err trees_from_buffer(int64_t buffer, int64_t chunk, int n, int* trees) {
  if (chunk < 1 || n < 2) return kScheduleError;
  if (buffer < chunk) return kBufferTooSmall;
  const int64_t fit = buffer / chunk;
  int t = 1;
  while (int64_t{t} * 2 <= fit && t * 2 <= max_trees(n)) t *= 2;
  *trees = t;
  return kOk;
}

Err round_count_formula(int n, int trees, int* rounds) {
  if (!is_pow2(n) || !is_pow2(trees)) return kNonPowerOfTwo;
  if (Err e = check_trees(n, trees)) return e;
  *rounds = n == 1 ? 0 : ceil_log2(trees) + n / trees - 1;
  return kOk;
}

std::vector<int> sendable_offsets(int n, int dim) {
  // k with k = 0 mod 2^(d+1) and k + 2^d < n, farthest first.
  std::vector<int> out;
  const int64_t stride = int64_t{1} << (dim + 1);
  const int64_t reach = int64_t{1} << dim;
  for (int64_t k = ((n - 1) / stride) * stride; k >= 0; k -= stride)
    if (k + reach < n) out.push_back(static_cast<int>(k));
  return out;
}

int received_offset(const Round& r, int k, int n) {
  return r.exchange ? (k ^ std::abs(r.peer)) : mod_ranks(int64_t{k} + r.peer, n);
}

namespace {

Schedule header(Algo algo, int n) {
  Schedule s;
  s.kind = Kind::AllGather;
  s.algo = algo;
  s.n = n;
  return s;
}

void push_round(Schedule& s, int dim, int split, int peer, bool exchange, std::vector<int> chunks) {
  Round r;
  r.index = static_cast<int>(s.rounds.size());
  r.dim = dim;
  r.split = split;
  r.peer = peer;
  r.exchange = exchange;
  r.chunks = std::move(chunks);
  s.rounds.push_back(std::move(r));
}

// PAT all-gather (algorithms.cpp:159-216): per dimension, the sendable offsets split into
// groups of <= T, far groups first. A group may fire once all its offsets are held; after a
// group fires, the next lower dimension is drained before the same dimension fires again
// (depth-first). Walked here with an explicit stack of dimensions.
Schedule pat_allgather(int n, int trees) {
  Schedule s = header(Algo::Pat, n);
  s.has_params = true;
  s.trees = trees;
  s.buffer_slots = pat_buffer_slots(n, trees);
  if (n == 1) return s;
  const int dims = ceil_log2(n);
  std::vector<std::vector<std::vector<int>>> groups(dims);
  for (int d = 0; d < dims; ++d) {
    const std::vector<int> k = sendable_offsets(n, d);
    for (size_t i = 0; i < k.size(); i += trees)
      groups[d].emplace_back(k.begin() + i, k.begin() + std::min(k.size(), i + trees));
  }
  std::vector<size_t> cursor(dims, 0);
  std::vector<char> held(n, 0);
  held[0] = 1;
  std::vector<int> stack = {dims - 1};
  while (!stack.empty()) {
    const int d = stack.back();
    bool fired = false;
    if (cursor[d] < groups[d].size()) {
      const std::vector<int>& g = groups[d][cursor[d]];
      if (std::all_of(g.begin(), g.end(), [&](int k) { return held[k] != 0; })) {
        push_round(s, d, static_cast<int>(cursor[d]), 1 << d, false, g);
        ++cursor[d];
        for (int k : g) held[k + (1 << d)] = 1;
        fired = true;
      }
    }
    if (!fired) {
      stack.pop_back();
    } else if (d > 0) {
      stack.push_back(d - 1);
    }
  }
  return s;
}

}  // namespace

Schedule mirror(const Schedule& s) {
  Schedule m;
  m.kind = s.kind == Kind::AllGather ? Kind::ReduceScatter : Kind::AllGather;
  m.algo = s.algo;
  m.n = s.n;
  m.has_params = s.has_params;
  m.trees = s.trees;
  m.buffer_slots = s.buffer_slots;
  std::map<int, int> groups_per_dim;
  for (const Round& r : s.rounds) groups_per_dim[r.dim] = std::max(groups_per_dim[r.dim], r.split + 1);
  for (auto it = s.rounds.rbegin(); it != s.rounds.rend(); ++it) {
    std::vector<int> chunks;
    for (int k : it->chunks) chunks.push_back(received_offset(*it, k, s.n));
    push_round(m, it->dim, groups_per_dim[it->dim] - 1 - it->split, -it->peer, it->exchange, std::move(chunks));
  }
  return m;
}

Err build(Kind kind, Algo algo, int n, int trees, Schedule* out) {
  if (n < 1) return kScheduleError;
  Schedule s;
  switch (algo) {
    case Algo::Pat:
      if (Err e = check_trees(n, trees)) return e;
      s = pat_allgather(n, trees);
      break;
    case Algo::Ring:
      s = header(algo, n);
      for (int i = 0; i + 1 < n; ++i) push_round(s, 0, 0, 1, false, {i});
      break;
    case Algo::BruckNearest: {
      s = header(algo, n);
      for (int d = 0; d < ceil_log2(n); ++d) {
        const int64_t cnt = std::min<int64_t>(int64_t{1} << d, n - (int64_t{1} << d));
        std::vector<int> k(cnt);
        for (int i = 0; i < cnt; ++i) k[i] = i;
        push_round(s, d, 0, 1 << d, false, std::move(k));
      }
      break;
    }
    case Algo::BruckFarthest:
      s = header(algo, n);
      for (int d = ceil_log2(n) - 1; d >= 0; --d) push_round(s, d, 0, 1 << d, false, sendable_offsets(n, d));
      break;
    case Algo::RecursiveDoubling: {
      if (!is_pow2(n)) return kNonPowerOfTwo;
      s = header(algo, n);
      for (int d = 0; (1 << d) < n; ++d) {
        std::vector<int> k(1 << d);
        for (int i = 0; i < (1 << d); ++i) k[i] = i;
        push_round(s, d, 0, 1 << d, true, std::move(k));
      }
      break;
    }
    default:
      return kInvalidArgument;
  }
  *out = kind == Kind::ReduceScatter ? mirror(s) : std::move(s);
  return kOk;
}

// ---------------------------------------------------------------- validation

namespace {

struct Log {
  int count = 0;
  std::string first;
  void add(const std::string& m) {
    if (count++ == 0) first = m;
  }
};

std::string fmt(const char* f, long long a = 0, long long b = 0, long long c = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b, c);
  return buf;
}

std::string set_str(const std::set<int>& s) {
  std::string out = "{";
  bool first = true;
  for (int k : s) {
    if (!first) out += ",";
    out += std::to_string(k);
    first = false;
  }
  return out + "}";
}

}  // namespace

int validate(const Schedule& s, std::string* first) {
  Log log;
  const int n = s.n;
  if (n < 1) {
    log.add("n_ranks must be >= 1");
  } else if (n == 1) {
    if (!s.rounds.empty()) log.add("single-rank schedule must be empty");
  } else {
    // structure (schedule.cpp:74-124)
    for (size_t i = 0; i < s.rounds.size(); ++i) {
      const Round& r = s.rounds[i];
      const int t = static_cast<int>(i);
      if (r.index != t) {
        log.add(fmt("round_index %lld at position %lld (must increase from 0)", r.index, t));
        continue;
      }
      if (r.dim < 0 || r.dim > 30) {
        log.add("dimension out of range [0, 30]");
        continue;
      }
      if (r.split < 0) log.add("negative split_index");
      const int64_t expect = int64_t{1} << r.dim;
      if (r.peer == 0 || std::llabs(r.peer) != expect) {
        log.add(fmt("peer offset %lld does not match dimension %lld (|peer| must be %lld)", r.peer, r.dim, expect));
      } else if (!r.exchange && expect % n == 0) {
        log.add(fmt("peer offset %lld is a self-loop for %lld ranks", r.peer, n));
      }
      if (r.chunks.empty()) {
        log.add("empty chunk set");
        continue;
      }
      std::set<int> seen;
      for (int k : r.chunks) {
        if (k < 0 || k >= n) log.add(fmt("offset %lld out of range [0, %lld)", k, n));
        else if (!seen.insert(k).second) log.add(fmt("duplicate offset %lld", k));
      }
      for (int k : r.chunks) {
        const int rk = received_offset(r, k, n);
        if (rk < 0 || rk >= n) log.add(fmt("received offset %lld out of range [0, %lld)", rk, n));
      }
    }
    if (log.count == 0 && s.kind == Kind::AllGather) {
      // hold-before-send + coverage (schedule.cpp:126-149)
      std::set<int> held = {0};
      for (const Round& r : s.rounds) {
        for (int k : r.chunks)
          if (!held.count(k)) log.add(fmt("offset %lld not held at round %lld", k, r.index));
        for (int k : r.chunks) held.insert(received_offset(r, k, n));
      }
      if (static_cast<int>(held.size()) != n) {
        std::set<int> missing;
        for (int k = 0; k < n; ++k)
          if (!held.count(k)) missing.insert(k);
        log.add("coverage gap " + set_str(missing));
      }
    } else if (log.count == 0) {
      // pending-accumulator flow (schedule.cpp:151-190)
      std::set<int> pending;
      for (int k = 0; k < n; ++k) pending.insert(k);
      for (const Round& r : s.rounds) {
        std::set<int> sent;
        for (int k : r.chunks) {
          if (!pending.count(k)) log.add(fmt("offset %lld already forwarded before round %lld", k, r.index));
          if (k == 0) log.add(fmt("offset 0 (own destination) forwarded at round %lld", r.index));
          sent.insert(k);
        }
        for (int k : r.chunks) {
          const int rk = received_offset(r, k, n);
          if (sent.count(rk))
            log.add(fmt("contribution for offset %lld arrives in round %lld which also forwards it", rk, r.index));
          else if (!pending.count(rk))
            log.add(fmt("contribution for offset %lld arrives at round %lld after its accumulator was forwarded", rk, r.index));
        }
        for (int k : sent) pending.erase(k);
      }
      pending.erase(0);
      if (!pending.empty()) log.add("offsets never forwarded " + set_str(pending));
    }
  }
  if (first) *first = log.first;
  return log.count;
}

// ---------------------------------------------------------------- stats

Stats schedule_stats(const Schedule& s, int64_t chunk_bytes) {
  // Slot accounting of run_allgather_impl / run_reduce_scatter_impl (simulate.cpp:167-214,
  // 241-292): AG arrivals stay staged while a later round still forwards them; RS
  // accumulators open at the first arrival and close when forwarded.
  Stats st;
  const int n = s.n;
  std::vector<int> last_send(n, -1);
  for (const Round& r : s.rounds)
    for (int k : r.chunks)
      if (k != 0) last_send[k] = r.index;
  std::set<int> slots;
  for (const Round& r : s.rounds) {
    if (s.kind == Kind::AllGather) {
      for (int k : r.chunks) {
        const int rk = received_offset(r, k, n);
        if (last_send[rk] > r.index) slots.insert(rk);
      }
      for (int k : r.chunks)
        if (k != 0 && last_send[k] == r.index) slots.erase(k);
    } else {
      for (int k : r.chunks) {
        const int rk = received_offset(r, k, n);
        if (rk != 0) slots.insert(rk);
      }
      for (int k : r.chunks) slots.erase(k);
    }
    const int occ = static_cast<int>(slots.size());
    st.rounds++;
    st.messages += n;
    st.max_chunks = std::max(st.max_chunks, static_cast<int>(r.chunks.size()));
    st.bytes_sent_per_rank += chunk_bytes * static_cast<int64_t>(r.chunks.size());
    st.occupancy.push_back(occ);
    st.peak = std::max(st.peak, occ);
  }
  return st;
}

// ---------------------------------------------------------------- encoding

std::vector<int32_t> encode(const Schedule& s) {
  std::vector<int32_t> v = {static_cast<int32_t>(s.kind), static_cast<int32_t>(s.algo), s.n,
                            s.has_params ? 1 : 0, s.has_params ? s.trees : 0,
                            s.has_params ? s.buffer_slots : 0, static_cast<int32_t>(s.rounds.size())};
  for (const Round& r : s.rounds) {
    v.insert(v.end(), {r.index, r.dim, r.split, r.peer, r.exchange ? 1 : 0, static_cast<int32_t>(r.chunks.size())});
    v.insert(v.end(), r.chunks.begin(), r.chunks.end());
  }
  return v;
}

Err decode(const int32_t* b, size_t len, Schedule* out) {
  if (!b || len < 7 || b[6] < 0) return kScheduleError;
  Schedule s;
  s.kind = b[0] == 0 ? Kind::AllGather : Kind::ReduceScatter;
  s.algo = static_cast<Algo>(b[1]);
  s.n = b[2];
  s.has_params = b[3] != 0;
  s.trees = b[4];
  s.buffer_slots = b[5];
  size_t p = 7;
  for (int t = 0; t < b[6]; ++t) {
    if (p + 6 > len) return kScheduleError;
    Round r;
    r.index = b[p];
    r.dim = b[p + 1];
    r.split = b[p + 2];
    r.peer = b[p + 3];
    r.exchange = b[p + 4] != 0;
    const int nk = b[p + 5];
    p += 6;
    if (nk < 0 || p + static_cast<size_t>(nk) > len) return kScheduleError;
    r.chunks.assign(b + p, b + p + nk);
    p += nk;
    s.rounds.push_back(std::move(r));
  }
  *out = std::move(s);
  return kOk;
}

}  // namespace pat
