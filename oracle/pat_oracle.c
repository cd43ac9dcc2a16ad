/*
 * pat_oracle.c — CPU restatement of the reference PAT path. TEST INFRASTRUCTURE ONLY:
 * loaded by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg) as the
 * checker; never linked into or called by the product (paper_2506_20252_b200/).
 *
 * Parity: pinned against the reference itself (oracle/_ref, built from
 * /root/reference/proj/src by oracle/Makefile) through the committed fixtures in
 * tests/golden/ (generator: tests/golden/make_golden.py). See DESIGN.md §Oracle.
 *
 * Restated reference code (all paths relative to /root/reference/proj):
 *   schedule.hpp:34-47            ceil_log2 / mod_ranks / is_power_of_two
 *   algorithms.cpp:49-103         max_trees, trees_from_buffer, pat_buffer_slots,
 *                                 round_count_formula, sendable_offsets
 *   algorithms.cpp:105-155        ring / bruck_nearest / bruck_farthest / recursive_doubling
 *   algorithms.cpp:159-216        PatEmitter depth-first far-first emission, pat_allgather
 *   algorithms.cpp:218-249        mirror_schedule / pat_reduce_scatter
 *   schedule.cpp:24-32, 74-212    received_offsets, validate
 *   simulate.cpp:151-300          run_allgather_impl / run_reduce_scatter_impl
 *   simulate.cpp:31-44            fold_one / fold_into (generalised to the NCCL dtypes/ops,
 *                                 each fold rounded to the wire dtype, RNE)
 *   oracle.cpp:15-62              definitional oracles, mt19937_64 payloads
 *   simulate.cpp:334-346          write_trace_csv
 */
#include "pat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ math (schedule.hpp:34-47) */

static int is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int po_ceil_log2(int64_t v) {
  int d = 0;
  while (((int64_t)1 << d) < v) d++;
  return d;
}

int po_mod_ranks(int64_t value, int n) {
  int64_t m = value % n;
  return (int)(m < 0 ? m + n : m);
}

size_t po_dtype_size(int dtype) {
  switch (dtype) {
    case PO_INT8: case PO_UINT8: return 1;
    case PO_FLOAT16: case PO_BFLOAT16: return 2;
    case PO_INT32: case PO_UINT32: case PO_FLOAT32: return 4;
    case PO_INT64: case PO_UINT64: case PO_FLOAT64: return 8;
    default: return 0;
  }
}

/* ------------------------------------------------------------------ parameters (algorithms.cpp:49-103) */

int po_max_trees(int n) {
  if (n <= 2) return 1;
  return 1 << (po_ceil_log2(n) - 1);
}

static int check_trees(int n, int trees) {
  if (!is_pow2(trees)) return PO_INVALID_TREE_COUNT;
  if (trees > po_max_trees(n)) return PO_INVALID_TREE_COUNT;
  return PO_OK;
}

int po_trees_from_buffer(int64_t buffer_bytes, int64_t chunk_bytes, int n, int* trees_out) {
  if (chunk_bytes < 1) return PO_SCHEDULE_ERROR;
  if (n < 2) return PO_SCHEDULE_ERROR;
  if (buffer_bytes < chunk_bytes) return PO_BUFFER_TOO_SMALL;
  int64_t fit = buffer_bytes / chunk_bytes;
  int t = 1;
  while ((int64_t)t * 2 <= fit && t * 2 <= po_max_trees(n)) t *= 2;
  *trees_out = t;
  return PO_OK;
}

int po_pat_buffer_slots(int n, int trees) {
  int m = 0;
  while (((int64_t)trees << m) < n) m++;
  return trees + m;
}

int po_round_count_formula(int n, int trees, int* out) {
  if (!is_pow2(n) || !is_pow2(trees)) return PO_NON_POWER_OF_TWO;
  int rc = check_trees(n, trees);
  if (rc) return rc;
  *out = n == 1 ? 0 : po_ceil_log2(trees) + n / trees - 1;
  return PO_OK;
}

int po_sendable_offsets(int n, int dim, int32_t* out, int cap) {
  int64_t stride = (int64_t)1 << (dim + 1), reach = (int64_t)1 << dim;
  int cnt = 0;
  for (int64_t k = ((n - 1) / stride) * stride; k >= 0; k -= stride) {
    if (k + reach < n) {
      if (cnt < cap) out[cnt] = (int32_t)k;
      cnt++;
    }
  }
  return cnt;
}

/* ------------------------------------------------------------------ schedule builder */

typedef struct {
  int32_t* buf;
  int64_t cap, len;
  int overflow;
  int nrounds;
} sbuild;

static void sb_put(sbuild* b, int32_t v) {
  if (b->len < b->cap) b->buf[b->len] = v; else b->overflow = 1;
  b->len++;
}

static void sb_header(sbuild* b, int kind, int algo, int n, int has_params, int trees, int slots) {
  b->len = 0; b->overflow = 0; b->nrounds = 0;
  sb_put(b, kind); sb_put(b, algo); sb_put(b, n); sb_put(b, has_params);
  sb_put(b, trees); sb_put(b, slots); sb_put(b, 0);
}

static void sb_round(sbuild* b, int dim, int split, int peer, int exchange, const int32_t* k, int nk) {
  sb_put(b, b->nrounds); sb_put(b, dim); sb_put(b, split); sb_put(b, peer); sb_put(b, exchange);
  sb_put(b, nk);
  for (int i = 0; i < nk; i++) sb_put(b, k[i]);
  b->nrounds++;
  if (b->cap > 6) b->buf[6] = b->nrounds;
}

/* Decoded view of a flat schedule. */
typedef struct {
  int round_index, dim, split, peer, exchange, nchunks;
  const int32_t* chunks;
} oround;
typedef struct {
  int kind, algo, n, has_params, trees, slots, nrounds;
  oround* rounds;
} osched;

static int decode(const int32_t* s, int64_t len, osched* o) {
  memset(o, 0, sizeof(*o));
  if (len < 7) return PO_SCHEDULE_ERROR;
  o->kind = s[0]; o->algo = s[1]; o->n = s[2]; o->has_params = s[3]; o->trees = s[4];
  o->slots = s[5]; o->nrounds = s[6];
  if (o->nrounds < 0 || o->nrounds > 100000) return PO_SCHEDULE_ERROR;
  o->rounds = (oround*)calloc((size_t)(o->nrounds ? o->nrounds : 1), sizeof(oround));
  int64_t p = 7;
  for (int t = 0; t < o->nrounds; t++) {
    if (p + 6 > len) { free(o->rounds); o->rounds = NULL; return PO_SCHEDULE_ERROR; }
    oround* r = &o->rounds[t];
    r->round_index = s[p]; r->dim = s[p + 1]; r->split = s[p + 2]; r->peer = s[p + 3];
    r->exchange = s[p + 4]; r->nchunks = s[p + 5];
    p += 6;
    if (r->nchunks < 0 || p + r->nchunks > len) { free(o->rounds); o->rounds = NULL; return PO_SCHEDULE_ERROR; }
    r->chunks = s + p;
    p += r->nchunks;
  }
  return PO_OK;
}

static void release(osched* o) { free(o->rounds); o->rounds = NULL; }

/* received_offsets (schedule.cpp:24-32) */
static int recv_offset(const oround* r, int k, int n) {
  return r->exchange ? (k ^ abs(r->peer)) : po_mod_ranks((int64_t)k + r->peer, n);
}

/* ------------------------------------------------------------------ generators (algorithms.cpp:105-216) */

typedef struct {
  int n, dims;
  int32_t** groups;    /* groups[d] flat offsets */
  int* gstart;         /* per dim: group boundaries packed: group g of dim d = [gbeg[d][g], gbeg[d][g+1]) */
  int** gbeg;
  int* ngroups;
  int* next_group;
  char* held;
  sbuild* out;
} emitter;

/* PatEmitter::fire (algorithms.cpp:176-186): depth-first, far group first, stop at the
 * first group that is not fully held. */
static void fire(emitter* e, int dim) {
  while (e->next_group[dim] < e->ngroups[dim]) {
    int g = e->next_group[dim];
    int b = e->gbeg[dim][g], en = e->gbeg[dim][g + 1];
    for (int i = b; i < en; i++)
      if (!e->held[e->groups[dim][i]]) return;
    sb_round(e->out, dim, g, 1 << dim, 0, e->groups[dim] + b, en - b);
    e->next_group[dim]++;
    for (int i = b; i < en; i++) e->held[e->groups[dim][i] + (1 << dim)] = 1;
    if (dim > 0) fire(e, dim - 1);
  }
}

static int gen_pat(sbuild* b, int n, int trees) {
  if (n < 1) return PO_SCHEDULE_ERROR;
  int rc = check_trees(n, trees);
  if (rc) return rc;
  sb_header(b, PO_ALLGATHER, PO_PAT, n, 1, trees, po_pat_buffer_slots(n, trees));
  if (n == 1) return PO_OK;
  int dims = po_ceil_log2(n);
  emitter e;
  memset(&e, 0, sizeof(e));
  e.n = n; e.dims = dims; e.out = b;
  e.groups = (int32_t**)calloc(dims, sizeof(int32_t*));
  e.gbeg = (int**)calloc(dims, sizeof(int*));
  e.ngroups = (int*)calloc(dims, sizeof(int));
  e.next_group = (int*)calloc(dims, sizeof(int));
  e.held = (char*)calloc(n, 1);
  e.held[0] = 1;
  for (int d = 0; d < dims; d++) {
    int cnt = po_sendable_offsets(n, d, NULL, 0);
    e.groups[d] = (int32_t*)calloc(cnt ? cnt : 1, sizeof(int32_t));
    po_sendable_offsets(n, d, e.groups[d], cnt);
    int ng = (cnt + trees - 1) / trees;
    e.ngroups[d] = ng;
    e.gbeg[d] = (int*)calloc(ng + 1, sizeof(int));
    for (int g = 0; g <= ng; g++) e.gbeg[d][g] = g * trees < cnt ? g * trees : cnt;
  }
  fire(&e, dims - 1);
  for (int d = 0; d < dims; d++) { free(e.groups[d]); free(e.gbeg[d]); }
  free(e.groups); free(e.gbeg); free(e.ngroups); free(e.next_group); free(e.held);
  return PO_OK;
}

static int gen_ring(sbuild* b, int n) {
  if (n < 1) return PO_SCHEDULE_ERROR;
  sb_header(b, PO_ALLGATHER, PO_RING, n, 0, 0, 0);
  for (int i = 0; i + 1 < n; i++) {
    int32_t k = i;
    sb_round(b, 0, 0, 1, 0, &k, 1);
  }
  return PO_OK;
}

static int gen_bruck_nearest(sbuild* b, int n) {
  if (n < 1) return PO_SCHEDULE_ERROR;
  sb_header(b, PO_ALLGATHER, PO_BRUCK_NEAREST, n, 0, 0, 0);
  int dims = po_ceil_log2(n);
  int32_t* k = (int32_t*)calloc(n, sizeof(int32_t));
  for (int d = 0; d < dims; d++) {
    int64_t cnt = ((int64_t)1 << d) < (n - ((int64_t)1 << d)) ? ((int64_t)1 << d) : (n - ((int64_t)1 << d));
    for (int i = 0; i < cnt; i++) k[i] = i;
    sb_round(b, d, 0, 1 << d, 0, k, (int)cnt);
  }
  free(k);
  return PO_OK;
}

static int gen_bruck_farthest(sbuild* b, int n) {
  if (n < 1) return PO_SCHEDULE_ERROR;
  sb_header(b, PO_ALLGATHER, PO_BRUCK_FARTHEST, n, 0, 0, 0);
  int dims = po_ceil_log2(n);
  int32_t* k = (int32_t*)calloc(n, sizeof(int32_t));
  for (int d = dims - 1; d >= 0; d--) {
    int cnt = po_sendable_offsets(n, d, k, n);
    sb_round(b, d, 0, 1 << d, 0, k, cnt);
  }
  free(k);
  return PO_OK;
}

static int gen_recursive_doubling(sbuild* b, int n) {
  if (n < 1) return PO_SCHEDULE_ERROR;
  if (!is_pow2(n)) return PO_NON_POWER_OF_TWO;
  sb_header(b, PO_ALLGATHER, PO_RECURSIVE_DOUBLING, n, 0, 0, 0);
  int32_t* k = (int32_t*)calloc(n, sizeof(int32_t));
  for (int d = 0; (1 << d) < n; d++) {
    for (int i = 0; i < (1 << d); i++) k[i] = i;
    sb_round(b, d, 0, 1 << d, 1, k, 1 << d);
  }
  free(k);
  return PO_OK;
}

/* mirror_schedule (algorithms.cpp:218-245) */
int po_mirror(const int32_t* in, int64_t in_len, int32_t* out, int64_t cap, int64_t* len) {
  osched s;
  int rc = decode(in, in_len, &s);
  if (rc) return rc;
  int maxdim = 0;
  for (int t = 0; t < s.nrounds; t++) if (s.rounds[t].dim > maxdim) maxdim = s.rounds[t].dim;
  int* gcount = (int*)calloc(maxdim + 2, sizeof(int));
  for (int t = 0; t < s.nrounds; t++) {
    int d = s.rounds[t].dim;
    if (d >= 0 && d <= maxdim && s.rounds[t].split + 1 > gcount[d]) gcount[d] = s.rounds[t].split + 1;
  }
  sbuild b = {out, cap, 0, 0, 0};
  sb_header(&b, s.kind == PO_ALLGATHER ? PO_REDUCESCATTER : PO_ALLGATHER, s.algo, s.n,
            s.has_params, s.trees, s.slots);
  int32_t* k = (int32_t*)calloc(s.n + 1, sizeof(int32_t));
  for (int t = s.nrounds - 1; t >= 0; t--) {
    const oround* r = &s.rounds[t];
    for (int i = 0; i < r->nchunks; i++) k[i] = recv_offset(r, r->chunks[i], s.n);
    int d = r->dim;
    int split = (d >= 0 && d <= maxdim ? gcount[d] : 0) - 1 - r->split;
    sb_round(&b, d, split, -r->peer, r->exchange, k, r->nchunks);
  }
  free(k); free(gcount); release(&s);
  *len = b.len;
  return b.overflow ? PO_CAPACITY : PO_OK;
}

int po_schedule(int kind, int algorithm, int n, int trees, int32_t* buf, int64_t cap, int64_t* len) {
  sbuild b = {buf, cap, 0, 0, 0};
  int rc;
  switch (algorithm) {
    case PO_PAT: rc = gen_pat(&b, n, trees); break;
    case PO_RING: rc = gen_ring(&b, n); break;
    case PO_BRUCK_NEAREST: rc = gen_bruck_nearest(&b, n); break;
    case PO_BRUCK_FARTHEST: rc = gen_bruck_farthest(&b, n); break;
    case PO_RECURSIVE_DOUBLING: rc = gen_recursive_doubling(&b, n); break;
    default: return PO_SCHEDULE_ERROR;
  }
  if (rc) return rc;
  if (b.overflow) { *len = b.len; return PO_CAPACITY; }
  if (kind == PO_REDUCESCATTER) {
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)b.len);
    memcpy(tmp, buf, sizeof(int32_t) * (size_t)b.len);
    rc = po_mirror(tmp, b.len, buf, cap, len);
    free(tmp);
    return rc;
  }
  *len = b.len;
  return PO_OK;
}

/* ------------------------------------------------------------------ validate (schedule.cpp:74-212) */

typedef struct {
  int count;
  char* first;
  int cap;
} vlog;

static void violation(vlog* v, const char* msg) {
  if (v->count == 0 && v->first && v->cap > 0) {
    strncpy(v->first, msg, (size_t)v->cap - 1);
    v->first[v->cap - 1] = 0;
  }
  v->count++;
}

static void set_string(char* dst, size_t cap, const char* prefix, const char* set, int n) {
  size_t p = (size_t)snprintf(dst, cap, "%s{", prefix);
  int first = 1;
  for (int k = 0; k < n && p < cap; k++) {
    if (!set[k]) continue;
    p += (size_t)snprintf(dst + p, cap - p, first ? "%d" : ",%d", k);
    first = 0;
  }
  if (p < cap) snprintf(dst + p, cap - p, "}");
}

int po_validate(const int32_t* sched, int64_t len, char* first_msg, int msg_cap) {
  vlog v = {0, first_msg, msg_cap};
  char m[512];
  if (first_msg && msg_cap > 0) first_msg[0] = 0;
  osched s;
  if (decode(sched, len, &s)) { violation(&v, "malformed schedule encoding"); return v.count; }
  const int n = s.n;
  if (n < 1) { violation(&v, "n_ranks must be >= 1"); release(&s); return v.count; }
  if (n == 1) {
    if (s.nrounds) violation(&v, "single-rank schedule must be empty");
    release(&s);
    return v.count;
  }
  /* check_structure (schedule.cpp:74-124) */
  for (int t = 0; t < s.nrounds; t++) {
    const oround* r = &s.rounds[t];
    if (r->round_index != t) {
      snprintf(m, sizeof m, "round_index %d at position %d (must increase from 0)", r->round_index, t);
      violation(&v, m);
      continue;
    }
    if (r->dim < 0 || r->dim > 30) { violation(&v, "dimension out of range [0, 30]"); continue; }
    if (r->split < 0) violation(&v, "negative split_index");
    int64_t expected = (int64_t)1 << r->dim;
    if (r->peer == 0 || llabs((long long)r->peer) != expected) {
      snprintf(m, sizeof m, "peer offset %d does not match dimension %d (|peer| must be %lld)",
               r->peer, r->dim, (long long)expected);
      violation(&v, m);
    } else if (!r->exchange && expected % n == 0) {
      snprintf(m, sizeof m, "peer offset %d is a self-loop for %d ranks", r->peer, n);
      violation(&v, m);
    }
    if (r->nchunks == 0) { violation(&v, "empty chunk set"); continue; }
    char* seen = (char*)calloc(n, 1);
    for (int i = 0; i < r->nchunks; i++) {
      int k = r->chunks[i];
      if (k < 0 || k >= n) {
        snprintf(m, sizeof m, "offset %d out of range [0, %d)", k, n);
        violation(&v, m);
      } else if (seen[k]) {
        snprintf(m, sizeof m, "duplicate offset %d", k);
        violation(&v, m);
      } else {
        seen[k] = 1;
      }
    }
    free(seen);
    for (int i = 0; i < r->nchunks; i++) {
      int k = recv_offset(r, r->chunks[i], n);
      if (k < 0 || k >= n) {
        snprintf(m, sizeof m, "received offset %d out of range [0, %d)", k, n);
        violation(&v, m);
      }
    }
  }
  if (v.count) { release(&s); return v.count; }
  if (s.kind == PO_ALLGATHER) {
    /* check_allgather_flow (schedule.cpp:126-149) */
    char* held = (char*)calloc(n, 1);
    held[0] = 1;
    for (int t = 0; t < s.nrounds; t++) {
      const oround* r = &s.rounds[t];
      for (int i = 0; i < r->nchunks; i++) {
        if (!held[r->chunks[i]]) {
          snprintf(m, sizeof m, "offset %d not held at round %d", r->chunks[i], t);
          violation(&v, m);
        }
      }
      for (int i = 0; i < r->nchunks; i++) {
        int k = recv_offset(r, r->chunks[i], n);
        if (k >= 0 && k < n) held[k] = 1;
      }
    }
    int cnt = 0;
    for (int k = 0; k < n; k++) cnt += held[k];
    if (cnt != n) {
      char* missing = (char*)calloc(n, 1);
      for (int k = 0; k < n; k++) missing[k] = !held[k];
      char big[4096];
      set_string(big, sizeof big, "coverage gap ", missing, n);
      violation(&v, big);
      free(missing);
    }
    free(held);
  } else {
    /* check_reduce_scatter_flow (schedule.cpp:151-190) */
    char* pending = (char*)malloc(n);
    memset(pending, 1, n);
    char* sent = (char*)calloc(n, 1);
    for (int t = 0; t < s.nrounds; t++) {
      const oround* r = &s.rounds[t];
      memset(sent, 0, n);
      for (int i = 0; i < r->nchunks; i++) {
        int k = r->chunks[i];
        if (!pending[k]) {
          snprintf(m, sizeof m, "offset %d already forwarded before round %d", k, t);
          violation(&v, m);
        }
        if (k == 0) {
          snprintf(m, sizeof m, "offset 0 (own destination) forwarded at round %d", t);
          violation(&v, m);
        }
        sent[k] = 1;
      }
      for (int i = 0; i < r->nchunks; i++) {
        int k = recv_offset(r, r->chunks[i], n);
        if (k < 0 || k >= n) continue;
        if (sent[k]) {
          snprintf(m, sizeof m, "contribution for offset %d arrives in round %d which also forwards it", k, t);
          violation(&v, m);
        } else if (!pending[k]) {
          snprintf(m, sizeof m, "contribution for offset %d arrives at round %d after its accumulator was forwarded", k, t);
          violation(&v, m);
        }
      }
      for (int k = 0; k < n; k++) if (sent[k]) pending[k] = 0;
    }
    pending[0] = 0;
    int any = 0;
    for (int k = 0; k < n; k++) any |= pending[k];
    if (any) {
      char big[4096];
      set_string(big, sizeof big, "offsets never forwarded ", pending, n);
      violation(&v, big);
    }
    free(pending); free(sent);
  }
  release(&s);
  return v.count;
}

/* ------------------------------------------------------------------ element arithmetic */

static float bf16_to_f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* float -> bf16, round to nearest even (NaN kept quiet). */
static uint16_t f_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

static float f16_to_f(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1fu, man = h & 0x3ffu;
  uint32_t u;
  if (exp == 0) {
    if (man == 0) {
      u = sign;
    } else { /* subnormal: value = man * 2^-24 */
      float f = (float)man * 5.9604644775390625e-8f;
      memcpy(&u, &f, 4);
      u |= sign;
    }
  } else if (exp == 31) {
    u = sign | 0x7f800000u | (man << 13);
  } else {
    u = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* float -> fp16, round to nearest even, with subnormals and overflow to inf. */
static uint16_t f_to_f16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
  uint32_t a = u & 0x7fffffffu;
  if (a > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);
  if (a >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* >= 65520 rounds to inf */
  if (a < 0x38800000u) {                                   /* below 2^-14: subnormal or zero */
    /* value / 2^-24 rounded to nearest even integer */
    float af;
    memcpy(&af, &a, 4);
    double q = (double)af * 16777216.0; /* exact in double */
    double r = nearbyint(q);            /* default rounding mode: nearest even */
    return (uint16_t)(sign | (uint16_t)r);
  }
  uint32_t exp = ((a >> 23) - 112u);
  uint32_t man = a & 0x7fffffu;
  uint32_t h = (exp << 10) | (man >> 13);
  uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  return (uint16_t)(sign | h);
}

#define FOLD_INT(T)                                                            \
  do {                                                                         \
    T* x = (T*)a;                                                              \
    const T* y = (const T*)b;                                                  \
    for (int64_t i = 0; i < elems; i++) {                                      \
      switch (op) {                                                            \
        case PO_SUM: x[i] = (T)((U)x[i] + (U)y[i]); break;                     \
        case PO_PROD: x[i] = (T)((U)x[i] * (U)y[i]); break;                    \
        case PO_MAX: x[i] = y[i] > x[i] ? y[i] : x[i]; break;                  \
        case PO_MIN: x[i] = y[i] < x[i] ? y[i] : x[i]; break;                  \
      }                                                                        \
    }                                                                          \
  } while (0)

#define FOLD_FLT(T)                                                            \
  do {                                                                         \
    T* x = (T*)a;                                                              \
    const T* y = (const T*)b;                                                  \
    for (int64_t i = 0; i < elems; i++) {                                      \
      switch (op) {                                                            \
        case PO_SUM: x[i] = x[i] + y[i]; break;                                \
        case PO_PROD: x[i] = x[i] * y[i]; break;                               \
        case PO_MAX: x[i] = y[i] > x[i] ? y[i] : x[i]; break;                  \
        case PO_MIN: x[i] = y[i] < x[i] ? y[i] : x[i]; break;                  \
      }                                                                        \
    }                                                                          \
  } while (0)

static float fop(int op, float x, float y) {
  switch (op) {
    case PO_SUM: return x + y;
    case PO_PROD: return x * y;
    case PO_MAX: return y > x ? y : x;
    default: return y < x ? y : x;
  }
}

/* fold_one / fold_into (simulate.cpp:31-44): a = a (op) b, left operand = accumulator.
 * Integers wrap (two's complement); fp16/bf16 compute in fp32 and round RNE per hop. */
int po_fold(int dtype, int op, void* a, const void* b, int64_t elems) {
  if (op < PO_SUM || op > PO_MIN) return PO_UNSUPPORTED_OP;
  switch (dtype) {
    case PO_INT8: { typedef uint8_t U; FOLD_INT(int8_t); break; }
    case PO_UINT8: { typedef uint8_t U; FOLD_INT(uint8_t); break; }
    case PO_INT32: { typedef uint32_t U; FOLD_INT(int32_t); break; }
    case PO_UINT32: { typedef uint32_t U; FOLD_INT(uint32_t); break; }
    case PO_INT64: { typedef uint64_t U; FOLD_INT(int64_t); break; }
    case PO_UINT64: { typedef uint64_t U; FOLD_INT(uint64_t); break; }
    case PO_FLOAT32: FOLD_FLT(float); break;
    case PO_FLOAT64: FOLD_FLT(double); break;
    case PO_FLOAT16: {
      uint16_t* x = (uint16_t*)a;
      const uint16_t* y = (const uint16_t*)b;
      for (int64_t i = 0; i < elems; i++) x[i] = f_to_f16(fop(op, f16_to_f(x[i]), f16_to_f(y[i])));
      break;
    }
    case PO_BFLOAT16: {
      uint16_t* x = (uint16_t*)a;
      const uint16_t* y = (const uint16_t*)b;
      for (int64_t i = 0; i < elems; i++) x[i] = f_to_bf16(fop(op, bf16_to_f(x[i]), bf16_to_f(y[i])));
      break;
    }
    default: return PO_UNSUPPORTED_OP;
  }
  return PO_OK;
}

/* ------------------------------------------------------------------ executors (simulate.cpp:151-300) */

static void stats_round(po_stats* st, const oround* r, int n, int64_t chunk_bytes, int slots) {
  if (!st) return;
  st->rounds++;
  st->messages += n;
  if (r->nchunks > st->max_chunks_per_message) st->max_chunks_per_message = r->nchunks;
  st->bytes_sent_per_rank += chunk_bytes * r->nchunks;
  if (st->n_occupancy < 512) st->occupancy_per_round[st->n_occupancy] = slots;
  st->n_occupancy++;
  if (slots > st->peak_intermediate_slots) st->peak_intermediate_slots = slots;
}

static int ensure_schedule(const int32_t* sched, int64_t len, int kind, osched* s) {
  int rc = decode(sched, len, s);
  if (rc) return PO_SIMULATION_ERROR;
  if (s->kind != kind) { release(s); return PO_SIMULATION_ERROR; }
  if (po_validate(sched, len, NULL, 0)) { release(s); return PO_INVALID_SCHEDULE; }
  return PO_OK;
}

static int peer_of(int rank, const oround* r, int n) {
  return r->exchange ? (rank ^ abs(r->peer)) : po_mod_ranks((int64_t)rank + r->peer, n);
}
static int source_of(int rank, const oround* r, int n) {
  return r->exchange ? (rank ^ abs(r->peer)) : po_mod_ranks((int64_t)rank - r->peer, n);
}
static int origin_of(int rank, int k, const oround* r, int n) {
  return r->exchange ? (rank ^ k) : po_mod_ranks((int64_t)rank - k, n);
}

/* run_allgather_impl (simulate.cpp:151-222). Stats count 8-byte elements as the
 * reference does (kElementBytes, simulate.cpp:17) so they compare 1:1. */
int po_run_allgather(const int32_t* sched, int64_t len, int dtype, int64_t elems,
                     const void* in, void* out, po_stats* st) {
  size_t es = po_dtype_size(dtype);
  if (!es) return PO_UNSUPPORTED_OP;
  osched s;
  int rc = ensure_schedule(sched, len, PO_ALLGATHER, &s);
  if (rc) return rc;
  if (elems < 1) { release(&s); return PO_PAYLOAD_SHAPE; }
  const int n = s.n;
  const size_t cb = (size_t)elems * es;
  const char* inb = (const char*)in;
  char* outb = (char*)out;
  if (st) memset(st, 0, sizeof(*st));
  /* own chunk first (simulate.cpp:160-165) */
  for (int r = 0; r < n; r++) memcpy(outb + ((size_t)r * n + r) * cb, inb + (size_t)r * cb, cb);
  int* last_send = (int*)malloc(sizeof(int) * n);
  for (int k = 0; k < n; k++) last_send[k] = -1;
  for (int t = 0; t < s.nrounds; t++)
    for (int i = 0; i < s.rounds[t].nchunks; i++)
      if (s.rounds[t].chunks[i] != 0) last_send[s.rounds[t].chunks[i]] = t;
  /* staged[r][k] + presence; mailbox[sender][i] */
  char* staged = (char*)malloc((size_t)n * n * cb);
  char* present = (char*)calloc((size_t)n * n, 1);
  char* mail = (char*)malloc((size_t)n * n * cb);
  for (int t = 0; t < s.nrounds; t++) {
    const oround* r = &s.rounds[t];
    /* send phase (simulate.cpp:186-194) */
    for (int rank = 0; rank < n; rank++) {
      for (int i = 0; i < r->nchunks; i++) {
        int k = r->chunks[i];
        const char* src = k == 0 ? inb + (size_t)rank * cb : staged + ((size_t)rank * n + k) * cb;
        memcpy(mail + ((size_t)rank * n + i) * cb, src, cb);
      }
    }
    /* deliver phase (simulate.cpp:199-212) */
    for (int rank = 0; rank < n; rank++) {
      int source = source_of(rank, r, n);
      for (int i = 0; i < r->nchunks; i++) {
        int k = recv_offset(r, r->chunks[i], n);
        int origin = origin_of(rank, k, r, n);
        const char* msg = mail + ((size_t)source * n + i) * cb;
        memcpy(outb + ((size_t)rank * n + origin) * cb, msg, cb);
        if (last_send[k] > t) {
          memcpy(staged + ((size_t)rank * n + k) * cb, msg, cb);
          present[(size_t)rank * n + k] = 1;
        }
      }
      for (int i = 0; i < r->nchunks; i++) {
        int k = r->chunks[i];
        if (k != 0 && last_send[k] == t) present[(size_t)rank * n + k] = 0;
      }
    }
    int slots = 0;
    for (int k = 0; k < n; k++) slots += present[k];
    stats_round(st, r, n, elems * 8, slots);
  }
  free(last_send); free(staged); free(present); free(mail);
  release(&s);
  return PO_OK;
}

/* run_reduce_scatter_impl (simulate.cpp:224-300) */
int po_run_reduce_scatter(const int32_t* sched, int64_t len, int dtype, int op, int64_t elems,
                          const void* in, void* out, po_stats* st) {
  size_t es = po_dtype_size(dtype);
  if (!es) return PO_UNSUPPORTED_OP;
  if (op < PO_SUM || op > PO_MIN) return PO_UNSUPPORTED_OP;
  osched s;
  int rc = ensure_schedule(sched, len, PO_REDUCESCATTER, &s);
  if (rc) return rc;
  if (elems < 1) { release(&s); return PO_PAYLOAD_SHAPE; }
  const int n = s.n;
  const size_t cb = (size_t)elems * es;
  const char* inb = (const char*)in;
  char* outb = (char*)out;
#define CONTRIB(rank, dest) (inb + ((size_t)(rank) * n + (dest)) * cb)
  if (st) memset(st, 0, sizeof(*st));
  for (int r = 0; r < n; r++) memcpy(outb + (size_t)r * cb, CONTRIB(r, r), cb); /* :237-239 */
  char* acc = (char*)malloc((size_t)n * n * cb);
  char* present = (char*)calloc((size_t)n * n, 1);
  char* mail = (char*)malloc((size_t)n * n * cb);
  for (int t = 0; t < s.nrounds; t++) {
    const oround* r = &s.rounds[t];
    /* send phase: value = acc (if any) folded with own contribution (:252-268) */
    for (int rank = 0; rank < n; rank++) {
      for (int i = 0; i < r->nchunks; i++) {
        int k = r->chunks[i];
        int dest = origin_of(rank, k, r, n);
        char* m = mail + ((size_t)rank * n + i) * cb;
        if (!present[(size_t)rank * n + k]) {
          memcpy(m, CONTRIB(rank, dest), cb);
        } else {
          memcpy(m, acc + ((size_t)rank * n + k) * cb, cb);
          po_fold(dtype, op, m, CONTRIB(rank, dest), elems);
        }
      }
    }
    /* deliver phase (:273-290) */
    for (int rank = 0; rank < n; rank++) {
      int source = source_of(rank, r, n);
      for (int i = 0; i < r->nchunks; i++) {
        int k = recv_offset(r, r->chunks[i], n);
        const char* m = mail + ((size_t)source * n + i) * cb;
        if (k == 0) {
          po_fold(dtype, op, outb + (size_t)rank * cb, m, elems);
        } else if (!present[(size_t)rank * n + k]) {
          memcpy(acc + ((size_t)rank * n + k) * cb, m, cb);
          present[(size_t)rank * n + k] = 1;
        } else {
          po_fold(dtype, op, acc + ((size_t)rank * n + k) * cb, m, elems);
        }
      }
      for (int i = 0; i < r->nchunks; i++) present[(size_t)rank * n + r->chunks[i]] = 0;
    }
    int slots = 0;
    for (int k = 0; k < n; k++) slots += present[k];
    stats_round(st, r, n, elems * 8, slots);
  }
#undef CONTRIB
  free(acc); free(present); free(mail);
  release(&s);
  return PO_OK;
}

/* ------------------------------------------------------------------ definitional oracles (oracle.cpp:15-40) */

int po_oracle_allgather(int n, int dtype, int64_t elems, const void* in, void* out) {
  size_t es = po_dtype_size(dtype);
  if (!es || n < 1) return PO_PAYLOAD_SHAPE;
  size_t cb = (size_t)elems * es;
  for (int r = 0; r < n; r++) memcpy((char*)out + (size_t)r * n * cb, in, (size_t)n * cb);
  return PO_OK;
}

int po_oracle_reduce_scatter(int n, int dtype, int op, int64_t elems, const void* in, void* out) {
  size_t es = po_dtype_size(dtype);
  if (!es || n < 1) return PO_PAYLOAD_SHAPE;
  size_t cb = (size_t)elems * es;
  for (int d = 0; d < n; d++) {
    char* o = (char*)out + (size_t)d * cb;
    memcpy(o, (const char*)in + (size_t)d * cb, cb);
    for (int s = 1; s < n; s++) {
      int rc = po_fold(dtype, op, o, (const char*)in + ((size_t)s * n + d) * cb, elems);
      if (rc) return rc;
    }
  }
  return PO_OK;
}

/* Closed-form tree (derived from simulate.cpp:239, 263-265, 278-285):
 *   V(k) = fold over c = k + 2^j (j < ctz(k), c < n, ascending j) of V(c), then (+) x_k
 *   out  = ((x_0 (+) V(1)) (+) V(2)) (+) V(4) ...           (k = 2^j < n, ascending j)
 * Valid for the full-aggregation (bruck-farthest) tree, which every valid T shares. */
static void tree_value(int n, int dtype, int op, const char* x, size_t es, int k, char* res) {
  int tz = 0;
  while (!((k >> tz) & 1)) tz++;
  int have = 0;
  char* tmp = (char*)malloc(es);
  for (int j = 0; j < tz; j++) {
    int c = k + (1 << j);
    if (c >= n) break;
    tree_value(n, dtype, op, x, es, c, tmp);
    if (!have) { memcpy(res, tmp, es); have = 1; } else po_fold(dtype, op, res, tmp, 1);
  }
  if (!have) memcpy(res, x + (size_t)k * es, es); else po_fold(dtype, op, res, x + (size_t)k * es, 1);
  free(tmp);
}

int po_tree_fold(int n, int dtype, int op, const void* x, void* result) {
  size_t es = po_dtype_size(dtype);
  if (!es || n < 1) return PO_PAYLOAD_SHAPE;
  char* res = (char*)result;
  char* tmp = (char*)malloc(es);
  memcpy(res, x, es);
  for (int k = 1; k < n; k <<= 1) {
    tree_value(n, dtype, op, (const char*)x, es, k, tmp);
    po_fold(dtype, op, res, tmp, 1);
  }
  free(tmp);
  return PO_OK;
}

/* ------------------------------------------------------------------ mt19937_64 (oracle.cpp:42-62) */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; i++)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = 312;
}

static uint64_t mt_next(mt64* m) {
  if (m->idx >= 312) {
    for (int i = 0; i < 312; i++) {
      uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t y = m->mt[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void po_mt19937_64(uint64_t seed, int64_t count, uint64_t* out) {
  mt64 m;
  mt_seed(&m, seed);
  for (int64_t i = 0; i < count; i++) out[i] = mt_next(&m);
}

/* random_payload (oracle.cpp:48-62): chunk-major, one generator per payload.
 * int64: raw draw (oracle.cpp:42); f64: (g>>11)*2^-53 (oracle.cpp:44-46);
 * f32: (g>>40)*2^-24; fp16/bf16: (g>>56)*2^-8; 32/8-bit ints: low bits. */
void po_random_payload(int dtype, int64_t nchunks, int64_t elems, uint64_t seed, void* out) {
  mt64 m;
  mt_seed(&m, seed);
  int64_t total = nchunks * elems;
  for (int64_t i = 0; i < total; i++) {
    uint64_t g = mt_next(&m);
    switch (dtype) {
      case PO_INT8: case PO_UINT8: ((uint8_t*)out)[i] = (uint8_t)g; break;
      case PO_INT32: case PO_UINT32: ((uint32_t*)out)[i] = (uint32_t)g; break;
      case PO_INT64: case PO_UINT64: ((uint64_t*)out)[i] = g; break;
      case PO_FLOAT64: ((double*)out)[i] = (double)(g >> 11) * 0x1.0p-53; break;
      case PO_FLOAT32: ((float*)out)[i] = (float)(g >> 40) * 0x1.0p-24f; break;
      case PO_BFLOAT16: ((uint16_t*)out)[i] = f_to_bf16((float)(g >> 56) * 0x1.0p-8f); break;
      case PO_FLOAT16: ((uint16_t*)out)[i] = f_to_f16((float)(g >> 56) * 0x1.0p-8f); break;
    }
  }
}

/* ------------------------------------------------------------------ trace (simulate.cpp:334-346) */

int64_t po_trace_csv(const int32_t* sched, int64_t len, int64_t chunk_bytes, char* buf, int64_t cap) {
  osched s;
  if (decode(sched, len, &s)) return -1;
  int64_t p = 0;
  char line[160];
#define EMIT(str)                                          \
  do {                                                     \
    int64_t l_ = (int64_t)strlen(str);                     \
    if (p + l_ < cap) memcpy(buf + p, str, (size_t)l_);    \
    p += l_;                                               \
  } while (0)
  EMIT("round,dim,split,sender,receiver,chunks,bytes\n");
  for (int t = 0; t < s.nrounds; t++) {
    const oround* r = &s.rounds[t];
    for (int snd = 0; snd < s.n; snd++) {
      snprintf(line, sizeof line, "%d,%d,%d,%d,%d,%d,%lld\n", r->round_index, r->dim, r->split, snd,
               peer_of(snd, r, s.n), r->nchunks, (long long)(chunk_bytes * r->nchunks));
      EMIT(line);
    }
  }
#undef EMIT
  if (p < cap) buf[p] = 0;
  release(&s);
  return p;
}
