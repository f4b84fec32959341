/*
 * hanf_oracle_gen.c -- CPU restatements for the BASELINE-config checkers.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY (see hanf_oracle.h).  Two pieces:
 *
 *  - or_gen_rmat: the R-MAT generator of BASELINE configs 2 and 5 as the
 *    B200 package defines it (paper_1011_5599_b200/csrc/hanf_rng.h
 *    rmat_draw + Feistel, hanf_host.cpp hanf_gen_rmat): 2^scale nodes,
 *    edge_factor * 2^scale draws, ids permuted, self-loops dropped, rows
 *    sorted and deduplicated as Graph::from_edges does (graph.hpp:29-44).
 *    The reference ships no R-MAT generator (its generators are
 *    gen_clique_path / gen_uniform_random, graph.hpp:238-285), so this is
 *    the independent restatement the reference arm of bench.py uses to
 *    build config 5 without loading libhanf.so.  Pinned by
 *    tests/test_oracle_gen.py (CSR digest equal to the package's host and
 *    device generators).
 *  - or_counter_digest: an order-independent 64-bit digest of a counter
 *    array in the reference packing (CounterArray::data(), hll.hpp:224),
 *    used by the at-size parity fixtures (tests/golden/make_config_golden.py).
 *
 * Multi-threaded (pthreads); every result is independent of the thread
 * count.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "hanf_oracle.h"

/* ---- the generator streams (hanf_rng.h) ------------------------------ */
static inline uint64_t mix64(uint64_t z) { /* hash.hpp:8-15 */
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}
static inline uint64_t hash3(uint64_t seed, uint64_t key, uint64_t k) {
  return mix64(mix64(seed ^ 0x5851f42d4c957f2dULL) ^ mix64(key * 0x9e3779b97f4a7c15ULL + k));
}

typedef struct {
  uint32_t lbits, rbits;
  uint64_t keys[4];
} feistel;

static void feistel_init(feistel* f, uint32_t bits, uint64_t seed) {
  f->lbits = bits / 2;
  f->rbits = bits - bits / 2;
  for (int i = 0; i < 4; ++i) f->keys[i] = mix64(seed * 4 + (uint64_t)i + 0x7f4a7c15ULL);
}
static inline uint64_t feistel_apply(const feistel* f, uint64_t x) {
  uint64_t l = x >> f->rbits, r = x & ((1ull << f->rbits) - 1);
  uint32_t lb = f->lbits, rb = f->rbits;
  for (int i = 0; i < 4; ++i) {
    const uint64_t fx = mix64(r ^ f->keys[i]) & ((1ull << lb) - 1);
    const uint64_t nl = r, nr = l ^ fx;
    l = nl;
    r = nr;
    const uint32_t t = lb;
    lb = rb;
    rb = t;
  }
  return (l << rb) | r;
}

static inline void rmat_draw(uint64_t seed, uint64_t i, uint32_t scale, uint32_t ta,
                             uint32_t tb, uint32_t tc, uint64_t* u_out, uint64_t* v_out) {
  uint64_t u = 0, v = 0, h = 0;
  for (uint32_t level = 0; level < scale; ++level) {
    if ((level & 3) == 0) h = hash3(seed, i, level >> 2);
    const uint32_t r = (uint32_t)(h >> (16 * (level & 3))) & 0xffff;
    const uint64_t bu = r >= tb, bv = (r >= ta && r < tb) || r >= tc;
    u = (u << 1) | bu;
    v = (v << 1) | bv;
  }
  *u_out = u;
  *v_out = v;
}

/* ---- a tiny parallel-for over [0, count) ----------------------------- */
typedef void (*range_fn)(void* ctx, uint64_t lo, uint64_t hi, unsigned tid);
typedef struct {
  range_fn fn;
  void* ctx;
  uint64_t count, chunk;
  unsigned tid;
  uint64_t* cursor;
  pthread_mutex_t* mu;
  int dynamic;
  unsigned threads;
} pf_arg;

static void* pf_worker(void* p) {
  pf_arg* a = (pf_arg*)p;
  if (!a->dynamic) { /* static split: thread t gets the t-th slice */
    const uint64_t per = (a->count + a->threads - 1) / a->threads;
    const uint64_t lo = per * a->tid, hi = lo + per < a->count ? lo + per : a->count;
    if (lo < hi) a->fn(a->ctx, lo, hi, a->tid);
    return NULL;
  }
  for (;;) {
    pthread_mutex_lock(a->mu);
    const uint64_t lo = *a->cursor;
    *a->cursor += a->chunk;
    pthread_mutex_unlock(a->mu);
    if (lo >= a->count) break;
    a->fn(a->ctx, lo, lo + a->chunk < a->count ? lo + a->chunk : a->count, a->tid);
  }
  return NULL;
}

static void parallel_for(unsigned threads, uint64_t count, uint64_t chunk, int dynamic,
                         range_fn fn, void* ctx) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  pf_arg args[256];
  uint64_t cursor = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  for (unsigned t = 0; t < threads; ++t) {
    args[t] = (pf_arg){fn, ctx, count, chunk ? chunk : 1, t, &cursor, &mu, dynamic, threads};
    pthread_create(&th[t], NULL, pf_worker, &args[t]);
  }
  for (unsigned t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* ---- or_gen_rmat ------------------------------------------------------ */
#define RM_BUCKET_BITS 12u
typedef struct {
  uint32_t scale, ta, tb, tc, shift;
  uint64_t seed, draws;
  feistel perm;
  unsigned threads;
  uint64_t* counts; /* [threads][buckets] */
  uint64_t* cursor; /* [threads][buckets] */
  uint64_t* keys;   /* bucket-ordered (u << 32 | v) */
  uint64_t* tmp;
  uint64_t* bucket_lo; /* [buckets + 1] */
  uint64_t* bucket_unique;
  uint32_t nbuckets;
  uint64_t* deg;    /* [n + 1] */
  uint32_t* succ;
  uint64_t* out_lo; /* [buckets] */
} rm_ctx;

static void rm_count(void* p, uint64_t lo, uint64_t hi, unsigned tid) {
  rm_ctx* c = (rm_ctx*)p;
  uint64_t* cnt = c->counts + (uint64_t)tid * c->nbuckets;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t u, v;
    rmat_draw(c->seed, i, c->scale, c->ta, c->tb, c->tc, &u, &v);
    const uint64_t pu = feistel_apply(&c->perm, u), pv = feistel_apply(&c->perm, v);
    if (pu == pv) continue; /* self-loops dropped */
    ++cnt[pu >> c->shift];
  }
}

static void rm_scatter(void* p, uint64_t lo, uint64_t hi, unsigned tid) {
  rm_ctx* c = (rm_ctx*)p;
  uint64_t* cur = c->cursor + (uint64_t)tid * c->nbuckets;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t u, v;
    rmat_draw(c->seed, i, c->scale, c->ta, c->tb, c->tc, &u, &v);
    const uint64_t pu = feistel_apply(&c->perm, u), pv = feistel_apply(&c->perm, v);
    if (pu == pv) continue;
    c->keys[cur[pu >> c->shift]++] = (pu << 32) | pv;
  }
}

/* LSD radix sort of one bucket on its low (shift + 32) bits, 16-bit
 * digits; then unique.  The bucket's slice of tmp is its scratch. */
static void rm_sort_buckets(void* p, uint64_t lo, uint64_t hi, unsigned tid) {
  (void)tid;
  rm_ctx* c = (rm_ctx*)p;
  uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) * 65536);
  for (uint64_t b = lo; b < hi; ++b) {
    uint64_t* a = c->keys + c->bucket_lo[b];
    uint64_t* t = c->tmp + c->bucket_lo[b];
    const uint64_t m = c->bucket_lo[b + 1] - c->bucket_lo[b];
    const uint32_t bits = c->shift + 32;
    for (uint32_t sh = 0; sh < bits; sh += 16) {
      memset(hist, 0, sizeof(uint64_t) * 65536);
      for (uint64_t i = 0; i < m; ++i) ++hist[(a[i] >> sh) & 0xffff];
      uint64_t run = 0;
      for (uint32_t d = 0; d < 65536; ++d) {
        const uint64_t x = hist[d];
        hist[d] = run;
        run += x;
      }
      for (uint64_t i = 0; i < m; ++i) t[hist[(a[i] >> sh) & 0xffff]++] = a[i];
      uint64_t* s = a;
      a = t;
      t = s;
    }
    /* the sorted keys are in `a` (keys or tmp slice); unique into the
     * keys slice */
    uint64_t* dst = c->keys + c->bucket_lo[b];
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; ++i)
      if (i == 0 || a[i] != a[i - 1]) dst[k++] = a[i];
    c->bucket_unique[b] = k;
  }
  free(hist);
}

static void rm_emit(void* p, uint64_t lo, uint64_t hi, unsigned tid) {
  (void)tid;
  rm_ctx* c = (rm_ctx*)p;
  for (uint64_t b = lo; b < hi; ++b) {
    const uint64_t* a = c->keys + c->bucket_lo[b];
    uint32_t* out = c->succ + c->out_lo[b];
    for (uint64_t i = 0; i < c->bucket_unique[b]; ++i) {
      out[i] = (uint32_t)a[i];
      ++c->deg[(a[i] >> 32) + 1];
    }
  }
}

int or_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double cc,
                uint64_t seed, uint64_t permute_seed, unsigned threads, or_graph* out) {
  memset(out, 0, sizeof(*out));
  if (scale < RM_BUCKET_BITS || scale > 32) return -1;
  if (!(a >= 0 && b >= 0 && cc >= 0 && a + b + cc <= 1.0)) return -1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  rm_ctx c;
  memset(&c, 0, sizeof(c));
  const uint64_t n = 1ull << scale;
  c.scale = scale;
  c.seed = seed;
  c.draws = n * edge_factor;
  c.ta = (uint32_t)(a * 65536.0);
  c.tb = (uint32_t)((a + b) * 65536.0);
  c.tc = (uint32_t)((a + b + cc) * 65536.0);
  feistel_init(&c.perm, scale, permute_seed);
  c.threads = threads;
  c.nbuckets = 1u << RM_BUCKET_BITS;
  c.shift = scale - RM_BUCKET_BITS;
  int rc = -2;
  c.counts = (uint64_t*)calloc((size_t)threads * c.nbuckets, sizeof(uint64_t));
  c.cursor = (uint64_t*)calloc((size_t)threads * c.nbuckets, sizeof(uint64_t));
  c.bucket_lo = (uint64_t*)calloc(c.nbuckets + 1, sizeof(uint64_t));
  c.bucket_unique = (uint64_t*)calloc(c.nbuckets, sizeof(uint64_t));
  c.out_lo = (uint64_t*)calloc(c.nbuckets, sizeof(uint64_t));
  if (!c.counts || !c.cursor || !c.bucket_lo || !c.bucket_unique || !c.out_lo) goto done;
  /* pass 1: bucket counts per thread (static slices: deterministic) */
  parallel_for(threads, c.draws, 0, 0, rm_count, &c);
  {
    uint64_t run = 0;
    for (uint32_t k = 0; k < c.nbuckets; ++k) {
      c.bucket_lo[k] = run;
      for (unsigned t = 0; t < threads; ++t) {
        c.cursor[(uint64_t)t * c.nbuckets + k] = run;
        run += c.counts[(uint64_t)t * c.nbuckets + k];
      }
    }
    c.bucket_lo[c.nbuckets] = run;
  }
  c.keys = (uint64_t*)malloc(sizeof(uint64_t) * (c.bucket_lo[c.nbuckets] + 1));
  c.tmp = (uint64_t*)malloc(sizeof(uint64_t) * (c.bucket_lo[c.nbuckets] + 1));
  if (!c.keys || !c.tmp) goto done;
  /* pass 2: the same draws again, written straight to their bucket slots */
  parallel_for(threads, c.draws, 0, 0, rm_scatter, &c);
  /* per-bucket sort + unique, big buckets first is not needed: dynamic
   * chunks of 16 buckets */
  parallel_for(threads, c.nbuckets, 16, 1, rm_sort_buckets, &c);
  free(c.tmp);
  c.tmp = NULL;
  {
    uint64_t run = 0;
    for (uint32_t k = 0; k < c.nbuckets; ++k) {
      c.out_lo[k] = run;
      run += c.bucket_unique[k];
    }
    out->arcs = run;
  }
  c.deg = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  c.succ = (uint32_t*)malloc(sizeof(uint32_t) * (out->arcs ? out->arcs : 1));
  if (!c.deg || !c.succ) goto done;
  parallel_for(threads, c.nbuckets, 16, 1, rm_emit, &c);
  for (uint64_t v = 0; v < n; ++v) c.deg[v + 1] += c.deg[v];
  out->n = n;
  out->offsets = c.deg;
  out->succ = c.succ;
  c.deg = NULL;
  c.succ = NULL;
  rc = 0;
done:
  free(c.counts);
  free(c.cursor);
  free(c.bucket_lo);
  free(c.bucket_unique);
  free(c.out_lo);
  free(c.keys);
  free(c.tmp);
  free(c.deg);
  free(c.succ);
  return rc;
}

/* ---- or_counter_digest ------------------------------------------------ */
typedef struct {
  const uint64_t* words;
  unsigned W;
  uint64_t partial[256];
} dg_ctx;

static void dg_range(void* p, uint64_t lo, uint64_t hi, unsigned tid) {
  dg_ctx* c = (dg_ctx*)p;
  uint64_t acc = 0;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t h = mix64(i + 0x9e3779b97f4a7c15ULL);
    for (unsigned w = 0; w < c->W; ++w) h = mix64(h ^ c->words[i * c->W + w]) + w;
    acc += mix64(h);
  }
  c->partial[tid] += acc;
}

/* digest = sum over counters i of mix64(h_i) mod 2^64, h_i a mix chain of
 * (i, its W words).  Order-independent: equal for any thread count. */
uint64_t or_counter_digest(const uint64_t* words, uint64_t n, unsigned W, unsigned threads) {
  dg_ctx c;
  memset(&c, 0, sizeof(c));
  c.words = words;
  c.W = W;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  parallel_for(threads, n, 0, 0, dg_range, &c);
  uint64_t d = 0;
  for (unsigned t = 0; t < 256; ++t) d += c.partial[t];
  return d;
}

/* digest of a CSR (offsets, succ): pins generated graphs across builders */
uint64_t or_csr_digest(const uint64_t* offsets, const uint32_t* succ, uint64_t n) {
  uint64_t h = mix64(n ^ 0x243f6a8885a308d3ULL), acc = 0;
  for (uint64_t v = 0; v <= n; ++v) acc += mix64(offsets[v] + v * 0x9e3779b97f4a7c15ULL);
  const uint64_t a = offsets[n];
  for (uint64_t i = 0; i < a; ++i) acc += mix64(((uint64_t)succ[i] << 32 | (i & 0xffffffffu)) ^ (i >> 32) ^ h);
  return acc;
}
