/*
 * hanf_oracle.c -- CPU restatement of the reference HyperANF hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hanf_oracle.h): the parity checker, never
 * the product.  Each block cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/hyperanf/).
 */
#include "hanf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================== */
/* hash.hpp                                                              */
/* ===================================================================== */

/* hash.hpp:8-15 -- murmur3 fmix64 */
uint64_t or_mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}

/* hash.hpp:20-22 */
uint64_t or_item_hash(uint64_t item, uint64_t seed) {
  return or_mix64(item ^ or_mix64(seed ^ 0x9e3779b97f4a7c15ULL));
}

/* hash.hpp:31-40 */
uint64_t or_sm_next(or_splitmix* s) {
  s->state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s->state;
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}

/* hash.hpp:43-46 -- multiply-shift reduction */
uint64_t or_sm_next_below(or_splitmix* s, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)or_sm_next(s) * bound) >> 64);
}

/* ===================================================================== */
/* hll.hpp                                                               */
/* ===================================================================== */

/* hll.hpp:27-34 */
double or_alpha_for_registers(unsigned m) {
  switch (m) {
    case 16: return 0.673;
    case 32: return 0.697;
    case 64: return 0.709;
    default: return 0.7213 / (1.0 + 1.079 / (double)m);
  }
}

/* hll.hpp:43-60 */
int or_params_make(unsigned b, uint64_t seed, unsigned r, or_params* out) {
  if (b < 4 || b > 20) return -1;
  if (r < 5 || r > 8) return -1;
  out->bucket_bits = b;
  out->registers = 1u << b;
  out->register_bits = r;
  out->alpha = or_alpha_for_registers(out->registers);
  out->seed = seed;
  out->words = (out->registers * r + 63) / 64;
  return 0;
}

/* hll.hpp:75-83 */
unsigned or_read_register(const uint64_t* c, const or_params* p, unsigned j) {
  const uint64_t bit = (uint64_t)j * p->register_bits;
  const uint64_t word = bit >> 6;
  const unsigned off = (unsigned)(bit & 63);
  uint64_t v = c[word] >> off;
  if (off + p->register_bits > 64) v |= c[word + 1] << (64 - off);
  return (unsigned)v & ((1u << p->register_bits) - 1);
}

/* hll.hpp:85-99 */
void or_write_register(uint64_t* c, const or_params* p, unsigned j, unsigned value) {
  const uint64_t mask = (1u << p->register_bits) - 1;
  const uint64_t bit = (uint64_t)j * p->register_bits;
  const uint64_t word = bit >> 6;
  const unsigned off = (unsigned)(bit & 63);
  c[word] = (c[word] & ~(mask << off)) | ((uint64_t)(value & mask) << off);
  if (off + p->register_bits > 64) {
    const unsigned spill = off + p->register_bits - 64;
    const uint64_t hi_mask = (1ULL << spill) - 1;
    c[word + 1] = (c[word + 1] & ~hi_mask) | ((uint64_t)(value & mask) >> (64 - off));
  }
}

/* hll.hpp:104-117 -- bucket from the top b bits, rho+ of the rest */
int or_counter_add(uint64_t* c, const or_params* p, uint64_t item) {
  const uint64_t h = or_item_hash(item, p->seed);
  const unsigned bucket = (unsigned)(h >> (64 - p->bucket_bits));
  const uint64_t rest = h << p->bucket_bits;
  unsigned v = rest == 0 ? (64 - p->bucket_bits) + 1
                         : (unsigned)__builtin_clzll(rest) + 1;
  const unsigned maxv = (1u << p->register_bits) - 1;
  if (v > maxv) v = maxv;
  const unsigned cur = or_read_register(c, p, bucket);
  if (v <= cur) return 0;
  or_write_register(c, p, bucket, v);
  return 1;
}

/* hll.hpp:122-141 -- alpha m^2 / sum 2^-M, linear counting below 2.5m */
double or_counter_estimate(const uint64_t* c, const or_params* p) {
  double harmonic = 0.0;
  unsigned zeros = 0;
  for (unsigned j = 0; j < p->registers; ++j) {
    const unsigned reg = or_read_register(c, p, j);
    harmonic += ldexp(1.0, -(int)reg);
    zeros += reg == 0;
  }
  const double m = (double)p->registers;
  const double raw = p->alpha * m * m / harmonic;
  if (raw <= 2.5 * m && zeros > 0) return m * log(m / (double)zeros);
  return raw;
}

/* hll.hpp:144-156 */
int or_naive_union(uint64_t* dst, const uint64_t* src, const or_params* p) {
  int changed = 0;
  for (unsigned j = 0; j < p->registers; ++j) {
    const unsigned a = or_read_register(dst, p, j);
    const unsigned b = or_read_register(src, p, j);
    if (b > a) {
      or_write_register(dst, p, j, b);
      changed = 1;
    }
  }
  return changed;
}

/* ===================================================================== */
/* broadword.hpp:71-130 -- PackedMax: two-pass multi-precision SWAR max   */
/* ===================================================================== */

static void packed_masks(const or_params* p, uint64_t* low, uint64_t* high) {
  const unsigned k = p->register_bits;
  memset(low, 0, sizeof(uint64_t) * p->words);
  memset(high, 0, sizeof(uint64_t) * p->words);
  for (uint64_t j = 0; j < p->registers; ++j) {  /* broadword.hpp:81-86 */
    const uint64_t lo = j * k;
    const uint64_t hi = lo + k - 1;
    low[lo >> 6] |= 1ULL << (lo & 63);
    high[hi >> 6] |= 1ULL << (hi & 63);
  }
}

/* max_into with caller-provided masks and scratch (the engine builds the
 * masks once, as PackedMax's constructor does) */
static int packed_max_with(const or_params* p, const uint64_t* low, const uint64_t* high,
                           uint64_t* scratch, uint64_t* dst, const uint64_t* src) {
  const unsigned w = p->words;
  uint64_t borrow = 0;
  for (unsigned i = 0; i < w; ++i) { /* pass 1: broadword.hpp:98-110 */
    const uint64_t x = dst[i], y = src[i], h = high[i];
    const uint64_t a = x | h;
    const uint64_t b = y & ~h;
    const uint64_t t = a - b;
    uint64_t borrow_out = a < b ? 1u : 0u;
    const uint64_t d = t - borrow;
    borrow_out |= d > t ? 1u : 0u;
    borrow = borrow_out;
    scratch[i] = ((d | (x ^ y)) ^ (x | ~y)) & h;
  }
  const unsigned s = p->register_bits - 1;
  int changed = 0;
  borrow = 0;
  for (unsigned i = 0; i < w; ++i) { /* pass 2: broadword.hpp:114-128 */
    const uint64_t lt = scratch[i];
    const uint64_t lt_up = i + 1 < w ? scratch[i + 1] : 0;
    const uint64_t shifted = (lt >> s) | (lt_up << (64 - s));
    const uint64_t a = shifted | high[i];
    const uint64_t t = a - low[i];
    uint64_t borrow_out = a < low[i] ? 1u : 0u;
    const uint64_t d = t - borrow;
    borrow_out |= d > t ? 1u : 0u;
    borrow = borrow_out;
    const uint64_t mask = (d | high[i]) ^ lt;
    const uint64_t res = (dst[i] & mask) | (src[i] & ~mask);
    changed |= res != dst[i];
    dst[i] = res;
  }
  return changed;
}

int or_packed_max_into(const or_params* p, uint64_t* dst, const uint64_t* src) {
  const unsigned w = p->words;
  uint64_t* low = (uint64_t*)malloc(sizeof(uint64_t) * w * 3);
  packed_masks(p, low, low + w);
  const int changed = packed_max_with(p, low, low + w, low + 2 * w, dst, src);
  free(low);
  return changed;
}

/* broadword == naive over every value pair of two straddling registers
 * (test_hll.cpp:145-169, registers 12/13 of m=16, r=5): mismatch count */
uint64_t or_selftest_straddle(void) {
  or_params p;
  or_params_make(4, 0, 5, &p);
  uint64_t a[2], b[2], n[2], mism = 0;
  for (unsigned x12 = 0; x12 < 32; ++x12)
    for (unsigned x13 = 0; x13 < 32; ++x13)
      for (unsigned y12 = 0; y12 < 32; ++y12)
        for (unsigned y13 = 0; y13 < 32; ++y13) {
          a[0] = a[1] = b[0] = b[1] = 0;
          or_write_register(a, &p, 12, x12);
          or_write_register(a, &p, 13, x13);
          or_write_register(b, &p, 12, y12);
          or_write_register(b, &p, 13, y13);
          n[0] = a[0];
          n[1] = a[1];
          const int cb = or_packed_max_into(&p, a, b);
          const int cn = or_naive_union(n, b, &p);
          mism += (a[0] != n[0] || a[1] != n[1] || cb != cn);
        }
  return mism;
}

/* ===================================================================== */
/* graph.hpp                                                             */
/* ===================================================================== */

static int cmp_pair(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

void or_graph_free(or_graph* g) {
  free(g->offsets);
  free(g->succ);
  g->offsets = NULL;
  g->succ = NULL;
  g->n = g->arcs = 0;
}

/* graph.hpp:29-44: validate ids, sort pairs, collapse duplicates, CSR */
int or_graph_from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst,
                        uint64_t count, or_graph* out) {
  for (uint64_t i = 0; i < count; ++i)
    if (src[i] >= n || dst[i] >= n) return -1;
  uint64_t* pairs = (uint64_t*)malloc(sizeof(uint64_t) * (count ? count : 1));
  for (uint64_t i = 0; i < count; ++i) pairs[i] = ((uint64_t)src[i] << 32) | dst[i];
  qsort(pairs, count, sizeof(uint64_t), cmp_pair);
  uint64_t u = 0;
  for (uint64_t i = 0; i < count; ++i)
    if (i == 0 || pairs[i] != pairs[u - 1]) pairs[u++] = pairs[i];
  out->n = n;
  out->arcs = u;
  out->offsets = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  out->succ = (uint32_t*)malloc(sizeof(uint32_t) * (u ? u : 1));
  for (uint64_t i = 0; i < u; ++i) ++out->offsets[(pairs[i] >> 32) + 1];
  for (uint64_t v = 0; v < n; ++v) out->offsets[v + 1] += out->offsets[v];
  for (uint64_t i = 0; i < u; ++i) out->succ[i] = (uint32_t)pairs[i];
  free(pairs);
  return 0;
}

/* graph.hpp:72-84 */
int or_graph_transpose(const or_graph* g, or_graph* t) {
  t->n = g->n;
  t->arcs = g->arcs;
  t->offsets = (uint64_t*)calloc(g->n + 1, sizeof(uint64_t));
  t->succ = (uint32_t*)malloc(sizeof(uint32_t) * (g->arcs ? g->arcs : 1));
  for (uint64_t i = 0; i < g->arcs; ++i) ++t->offsets[g->succ[i] + 1];
  for (uint64_t v = 0; v < g->n; ++v) t->offsets[v + 1] += t->offsets[v];
  uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * (g->n ? g->n : 1));
  memcpy(cursor, t->offsets, sizeof(uint64_t) * g->n);
  for (uint64_t v = 0; v < g->n; ++v)
    for (uint64_t i = g->offsets[v]; i < g->offsets[v + 1]; ++i)
      t->succ[cursor[g->succ[i]]++] = (uint32_t)v;
  free(cursor);
  return 0;
}

/* graph.hpp:262-285: round(d) distinct uniform successors per node */
int or_gen_uniform_random(uint64_t n, double d, uint64_t seed, or_graph* out) {
  if (n < 1 || n > 0xffffffffULL) return -1;
  const uint64_t deg = (uint64_t)llround(d);
  if (d < 0 || deg >= n) return -1;
  or_splitmix rng = {or_mix64(seed ^ 0x5eedULL)};
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * (n * deg != 0 ? n * deg : 1));
  uint32_t* dst = (uint32_t*)malloc(sizeof(uint32_t) * (n * deg != 0 ? n * deg : 1));
  uint32_t* picks = (uint32_t*)malloc(sizeof(uint32_t) * (deg ? deg : 1));
  uint64_t e = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t np = 0;
    while (np < deg) {
      const uint32_t w = (uint32_t)or_sm_next_below(&rng, n);
      int found = 0;
      for (uint64_t i = 0; i < np; ++i) if (picks[i] == w) { found = 1; break; }
      if (!found) picks[np++] = w;
    }
    for (uint64_t i = 0; i < np; ++i) { src[e] = (uint32_t)v; dst[e] = picks[i]; ++e; }
  }
  const int rc = or_graph_from_edges(n, src, dst, e, out);
  free(src); free(dst); free(picks);
  return rc;
}

/* graph.hpp:238-258: two k-cliques joined by a one-way l-path */
int or_gen_clique_path(uint64_t k, uint64_t l, or_graph* out) {
  if (k < 1 || l < 1) return -1;
  const uint64_t n = 2 * k + l;
  if (n > 0xffffffffULL) return -1;
  const uint64_t cap = 2 * k * (k - 1) + (l - 1) + 2 * k + 1;
  uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  uint32_t* dst = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  uint64_t e = 0;
#define ARC(a, b) do { src[e] = (uint32_t)(a); dst[e] = (uint32_t)(b); ++e; } while (0)
  for (uint64_t a = 0; a < k; ++a)
    for (uint64_t b = 0; b < k; ++b)
      if (a != b) ARC(a, b);
  for (uint64_t a = 0; a < k; ++a) ARC(a, k);
  for (uint64_t i = 0; i + 1 < l; ++i) ARC(k + i, k + i + 1);
  for (uint64_t b = 0; b < k; ++b) ARC(k + l - 1, k + l + b);
  for (uint64_t a = 0; a < k; ++a)
    for (uint64_t b = 0; b < k; ++b)
      if (a != b) ARC(k + l + a, k + l + b);
#undef ARC
  const int rc = or_graph_from_edges(n, src, dst, e, out);
  free(src); free(dst);
  return rc;
}

/* ===================================================================== */
/* engine.hpp                                                            */
/* ===================================================================== */

#define OR_KBLOCK 64 /* engine.hpp:278 */

struct or_engine {
  uint64_t* low;           /* PackedMax masks, broadword.hpp:75-87 */
  uint64_t* high;
  uint64_t* scratch;
  const uint64_t* offsets; /* borrowed, engine.hpp:281 */
  const uint32_t* succ;
  uint64_t n;
  or_config cfg;
  or_params params;
  uint64_t* current;
  uint64_t* next;
  uint8_t* modified;
  uint8_t* next_modified;
  uint8_t* signalled;
  double* block_sums;
  uint8_t* block_dirty;
  uint64_t blocks;
  or_graph transpose;
  int have_transpose;
  uint64_t t;
  int systolic;
};

/* engine.hpp:32-46 */
void or_config_default(or_config* c) {
  c->bucket_bits = 7;
  c->register_bits = 0;
  c->seed = 0;
  c->systolic_threshold = 0.25;
  c->termination = 0;
  c->eps_inc = 0.0;
  c->max_iterations = 0;
  c->track_modified = 1;
  c->use_systolic = 1;
}

/* engine.hpp:70-90 */
or_engine* or_engine_create(const uint64_t* offsets, const uint32_t* succ,
                            uint64_t n, const or_config* cfg, int* status) {
  *status = 0;
  if (cfg->systolic_threshold <= 0.0 || cfg->systolic_threshold > 1.0) { *status = 1; return NULL; }
  if (cfg->termination == 1 && cfg->eps_inc <= 0.0) { *status = 1; return NULL; }
  or_engine* e = (or_engine*)calloc(1, sizeof(or_engine));
  e->offsets = offsets;
  e->succ = succ;
  e->n = n;
  e->cfg = *cfg;
  if (e->cfg.max_iterations == 0) e->cfg.max_iterations = n + 1;
  unsigned r = e->cfg.register_bits;
  if (r == 0) r = n < (1ULL << 32) ? 5 : 6;
  if (or_params_make(e->cfg.bucket_bits, e->cfg.seed, r, &e->params) != 0) {
    free(e);
    *status = 1;
    return NULL;
  }
  e->low = (uint64_t*)malloc(sizeof(uint64_t) * e->params.words * 3);
  e->high = e->low + e->params.words;
  e->scratch = e->high + e->params.words;
  packed_masks(&e->params, e->low, e->high);
  const uint64_t words = (uint64_t)e->params.words * (n ? n : 1);
  e->current = (uint64_t*)calloc(words, sizeof(uint64_t));
  e->next = NULL;
  for (uint64_t v = 0; v < n; ++v)
    or_counter_add(e->current + v * e->params.words, &e->params, v);
  e->modified = (uint8_t*)malloc(n ? n : 1);
  memset(e->modified, 1, n);
  e->next_modified = NULL;
  e->signalled = NULL;
  e->blocks = (n + OR_KBLOCK - 1) / OR_KBLOCK;
  e->block_sums = (double*)calloc(e->blocks ? e->blocks : 1, sizeof(double));
  e->block_dirty = (uint8_t*)malloc(e->blocks ? e->blocks : 1);
  memset(e->block_dirty, 1, e->blocks);
  return e;
}

void or_engine_destroy(or_engine* e) {
  if (!e) return;
  free(e->current); free(e->next); free(e->modified); free(e->next_modified);
  free(e->signalled); free(e->block_sums); free(e->block_dirty); free(e->low);
  if (e->have_transpose) or_graph_free(&e->transpose);
  free(e);
}

const uint64_t* or_engine_counters(const or_engine* e) { return e->current; }
unsigned or_engine_words(const or_engine* e) { return e->params.words; }
uint64_t or_engine_iteration(const or_engine* e) { return e->t; }
int or_engine_systolic_active(const or_engine* e) { return e->systolic; }

/* engine.hpp:100-118: recompute dirty 64-counter blocks in index order,
 * then a sequential total over the block sums. */
double or_engine_sum_estimates(or_engine* e) {
  const unsigned w = e->params.words;
  for (uint64_t b = 0; b < e->blocks; ++b) {
    if (!e->block_dirty[b]) continue;
    const uint64_t first = b * OR_KBLOCK;
    const uint64_t last = first + OR_KBLOCK < e->n ? first + OR_KBLOCK : e->n;
    double sum = 0.0;
    for (uint64_t i = first; i < last; ++i)
      sum += or_counter_estimate(e->current + i * w, &e->params);
    e->block_sums[b] = sum;
  }
  memset(e->block_dirty, 0, e->blocks);
  double total = 0.0;
  for (uint64_t b = 0; b < e->blocks; ++b) total += e->block_sums[b];
  return total;
}

/* engine.hpp:122-228 (the spill_to_disk branch is not restated: it only
 * reroutes the same bits through a tmpfile, engine.hpp:143-197). */
void or_engine_step(or_engine* e, double* sum, uint64_t* modified) {
  const uint64_t n = e->n;
  if (n == 0) { *sum = 0.0; *modified = 0; return; }
  const unsigned words = e->params.words;
  if (!e->next) e->next = (uint64_t*)calloc((uint64_t)words * n, sizeof(uint64_t));
  if (!e->next_modified) e->next_modified = (uint8_t*)calloc(n, 1);

  for (uint64_t v = 0; v < n; ++v) {                    /* engine.hpp:160-184 */
    const int compute = !e->systolic || e->signalled[v];
    uint64_t* dst = e->next + v * words;
    memcpy(dst, e->current + v * words, words * sizeof(uint64_t));
    int changed = 0;
    if (compute) {
      for (uint64_t i = e->offsets[v]; i < e->offsets[v + 1]; ++i) {
        const uint32_t s = e->succ[i];
        if (e->cfg.track_modified && !e->modified[s]) continue;
        changed |= packed_max_with(&e->params, e->low, e->high, e->scratch, dst,
                                   e->current + (uint64_t)s * words);
      }
    }
    e->next_modified[v] = changed ? 1 : 0;
  }
  { uint64_t* tmp = e->current; e->current = e->next; e->next = tmp; }  /* :198 */
  { uint8_t* tmp = e->modified; e->modified = e->next_modified; e->next_modified = tmp; } /* :200 */

  uint64_t count = 0;                                   /* engine.hpp:202-208 */
  for (uint64_t v = 0; v < n; ++v)
    if (e->modified[v]) { ++count; e->block_dirty[v / OR_KBLOCK] = 1; }

  if (e->cfg.use_systolic) {                            /* engine.hpp:210-224 */
    if (!e->systolic && count > 0 &&
        (double)count < e->cfg.systolic_threshold * (double)n) {
      e->systolic = 1;
      if (!e->have_transpose) {
        or_graph g = {n, e->offsets[n], (uint64_t*)e->offsets, (uint32_t*)e->succ};
        or_graph_transpose(&g, &e->transpose);
        e->have_transpose = 1;
      }
      if (!e->signalled) e->signalled = (uint8_t*)calloc(n, 1);
    }
    if (e->systolic) {
      memset(e->signalled, 0, n);
      for (uint64_t v = 0; v < n; ++v)
        if (e->modified[v])
          for (uint64_t i = e->transpose.offsets[v]; i < e->transpose.offsets[v + 1]; ++i)
            e->signalled[e->transpose.succ[i]] = 1;
    }
  }
  ++e->t;
  *sum = or_engine_sum_estimates(e);
  *modified = count;
}

/* engine.hpp:233-275 */
int or_engine_run(or_engine* e, double* values, uint64_t* modified,
                  uint64_t cap, uint64_t* len) {
  *len = 0;
  if (e->n == 0) return 0;
  if (cap < 1) return 5;
  values[0] = or_engine_sum_estimates(e);
  modified[0] = e->n;
  uint64_t count = 1;
  for (;;) {
    if (count - 1 >= e->cfg.max_iterations) { *len = count; return 2; }
    double sum;
    uint64_t mod;
    or_engine_step(e, &sum, &mod);
    if (mod == 0) break;
    const double prev = values[count - 1];
    if (count >= cap) { *len = count; return 5; }
    values[count] = sum;
    modified[count] = mod;
    ++count;
    if (e->cfg.termination == 1 && prev > 0.0) {
      const double rel = (sum - prev) / prev;
      if (rel < e->cfg.eps_inc) break;
    }
  }
  for (uint64_t t = 1; t < count; ++t)                  /* :269-270 clamp */
    if (values[t] < values[t - 1]) values[t] = values[t - 1];
  *len = count;
  return 0;
}

/* ===================================================================== */
/* oracle.hpp, tests/test_util.hpp                                       */
/* ===================================================================== */

/* oracle.hpp:38-104 (single-threaded; guards not restated) */
int or_exact_nf(const uint64_t* offsets, const uint32_t* succ, uint64_t n,
                uint64_t* values, uint64_t cap, uint64_t* len) {
  *len = 0;
  if (n == 0) {
    if (cap < 1) return 5;
    values[0] = 0;
    *len = 1;
    return 0;
  }
  uint32_t* stamp = (uint32_t*)calloc(n, sizeof(uint32_t));
  uint32_t* dist = (uint32_t*)calloc(n, sizeof(uint32_t));
  uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint64_t* hist = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  uint64_t depth = 1;
  for (uint64_t src = 0; src < n; ++src) {
    const uint32_t mark = (uint32_t)src + 1;
    uint64_t head = 0, tail = 0;
    queue[tail++] = (uint32_t)src;
    stamp[src] = mark;
    dist[src] = 0;
    for (; head < tail; ++head) {
      const uint32_t v = queue[head];
      const uint32_t dv = dist[v];
      if (dv + 1 > depth) depth = dv + 1;
      ++hist[dv];
      for (uint64_t i = offsets[v]; i < offsets[v + 1]; ++i) {
        const uint32_t w = succ[i];
        if (stamp[w] == mark) continue;
        stamp[w] = mark;
        dist[w] = dv + 1;
        queue[tail++] = w;
      }
    }
  }
  *len = depth;
  int rc = 0;
  if (cap < depth) {
    rc = 5;
  } else {
    uint64_t acc = 0;
    for (uint64_t d = 0; d < depth; ++d) {
      acc += hist[d];
      values[d] = acc;
    }
  }
  free(stamp); free(dist); free(queue); free(hist);
  return rc;
}

/* oracle.hpp:107-113 */
uint64_t or_clique_path_nf(uint64_t k, uint64_t l, uint64_t t) {
  if (t == 0) return 2 * k + l;
  if (t <= l) return (t + 1) * (4 * k + 2 * l - t) / 2 - 2 * k + 2 * k * k;
  return (l + 1) * (4 * k + l) / 2 - 2 * k + 3 * k * k;
}

/* test_util.hpp:16-41: counter fed exactly B(v, radius) */
void or_counter_of_ball(const uint64_t* offsets, const uint32_t* succ, uint64_t n,
                        uint32_t v, uint64_t radius, const or_params* p, uint64_t* dst) {
  uint32_t* dist = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint64_t i = 0; i < n; ++i) dist[i] = 0xffffffffu;
  memset(dst, 0, sizeof(uint64_t) * p->words);
  uint64_t head = 0, tail = 0;
  queue[tail++] = v;
  dist[v] = 0;
  for (; head < tail; ++head) {
    const uint32_t x = queue[head];
    if (dist[x] > radius) break;
    or_counter_add(dst, p, x);
    for (uint64_t i = offsets[x]; i < offsets[x + 1]; ++i) {
      const uint32_t w = succ[i];
      if (dist[w] != 0xffffffffu) continue;
      dist[w] = dist[x] + 1;
      queue[tail++] = w;
    }
  }
  free(dist);
  free(queue);
}

/* ===================================================================== */
/* stats.hpp                                                             */
/* ===================================================================== */

/* stats.hpp:33-60: H = N/N(T); density; mean, variance, spid */
int or_distance_distribution(const double* nf, uint64_t len, double* mean_out,
                             double* variance_out, double* spid_out) {
  if (len == 0) return -1;
  const double last = nf[len - 1];
  if (!(last > 0.0)) return -1;
  double prev = 0.0, mean = 0.0, second = 0.0;
  for (uint64_t t = 0; t < len; ++t) {
    const double cdf = nf[t] / last;
    const double h = cdf - prev;
    prev = cdf;
    mean += (double)t * h;
    second += (double)t * (double)t * h;
  }
  const double var = second - mean * mean;
  *mean_out = mean;
  *variance_out = var > 0.0 ? var : 0.0;
  *spid_out = mean > 0.0 ? *variance_out / mean : 0.0;
  return 0;
}

/* stats.hpp:65-77 */
int or_effective_diameter(const double* nf, uint64_t len, double alpha,
                          int interpolated, double* out) {
  if (!(alpha > 0.0 && alpha <= 1.0)) return -1;
  if (len == 0) return -1;
  const double target = alpha * nf[len - 1];
  uint64_t t = 0;
  while (t + 1 < len && nf[t] < target) ++t;
  if (!interpolated || t == 0) { *out = (double)t; return 0; }
  const double rise = nf[t] - nf[t - 1];
  if (rise <= 0.0) { *out = (double)(t - 1); return 0; }
  *out = (double)(t - 1) + (target - nf[t - 1]) / rise;
  return 0;
}
