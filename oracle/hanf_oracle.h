/*
 * hanf_oracle.h -- CPU restatement of the reference HyperANF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 engine: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_1011_5599_b200/, libhanf.so) never links or calls it.
 *
 * Every function restates the reference algorithm (arXiv:1011.5599
 * reference implementation, /root/reference/proj/include/hyperanf/...)
 * and cites the file:line it follows.  Plain C11, single-threaded,
 * scalar; compiled with -ffp-contract=off so floating-point evaluation
 * order equals the reference's.
 *
 * Pinning: checked against the reference compiled from its own headers
 * (oracle/_ref, see oracle/Makefile) and the golden fixtures in
 * tests/golden/ (made by tests/golden/make_golden.py from oracle/_ref).
 */
#ifndef HANF_ORACLE_H
#define HANF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- hash.hpp ------------------------------------------------------- */
uint64_t or_mix64(uint64_t z);                        /* hash.hpp:8-15  */
uint64_t or_item_hash(uint64_t item, uint64_t seed);  /* hash.hpp:20-22 */
typedef struct { uint64_t state; } or_splitmix;       /* hash.hpp:27-55 */
uint64_t or_sm_next(or_splitmix* s);
uint64_t or_sm_next_below(or_splitmix* s, uint64_t bound);

/* ---- hll.hpp -------------------------------------------------------- */
typedef struct {
  unsigned bucket_bits;    /* b */
  unsigned registers;      /* m = 2^b */
  unsigned register_bits;  /* r */
  double alpha;
  uint64_t seed;
  unsigned words;          /* W = ceil(m*r/64) */
} or_params;

double or_alpha_for_registers(unsigned m);                       /* hll.hpp:27-34 */
int or_params_make(unsigned b, uint64_t seed, unsigned r, or_params* out); /* 43-56; -1 = invalid */
unsigned or_read_register(const uint64_t* c, const or_params* p, unsigned j);  /* 75-83 */
void or_write_register(uint64_t* c, const or_params* p, unsigned j, unsigned v); /* 85-99 */
int or_counter_add(uint64_t* c, const or_params* p, uint64_t item);  /* 104-117 */
double or_counter_estimate(const uint64_t* c, const or_params* p);   /* 122-141 */
int or_naive_union(uint64_t* dst, const uint64_t* src, const or_params* p); /* 144-156 */

/* ---- broadword.hpp: PackedMax (75-130) ------------------------------ */
int or_packed_max_into(const or_params* p, uint64_t* dst, const uint64_t* src);
/* test_hll.cpp:145-169: exhaustive straddling pair, returns mismatches */
uint64_t or_selftest_straddle(void);

/* ---- graph.hpp ------------------------------------------------------ */
typedef struct {
  uint64_t n;
  uint64_t arcs;
  uint64_t* offsets; /* n+1 */
  uint32_t* succ;    /* arcs */
} or_graph;

/* graph.hpp:29-44 (sort + unique + CSR).  Returns -1 on out-of-range ids. */
int or_graph_from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst,
                        uint64_t count, or_graph* out);
int or_graph_transpose(const or_graph* g, or_graph* out);          /* 72-84 */
int or_gen_uniform_random(uint64_t n, double d, uint64_t seed, or_graph* out); /* 262-285 */
int or_gen_clique_path(uint64_t k, uint64_t l, or_graph* out);     /* 238-258 */
void or_graph_free(or_graph* g);

/* ---- engine.hpp ----------------------------------------------------- */
typedef struct {
  unsigned bucket_bits;        /* engine.hpp:33 */
  unsigned register_bits;      /* 0 = auto (5 below 2^32 nodes) */
  uint64_t seed;
  double systolic_threshold;   /* (0, 1] */
  int termination;             /* 0 stabilisation, 1 threshold */
  double eps_inc;
  uint64_t max_iterations;     /* 0 = n + 1 */
  int track_modified;
  int use_systolic;
} or_config;

void or_config_default(or_config* c);   /* EngineConfig defaults, engine.hpp:32-46 */

typedef struct or_engine or_engine;

/* Graph arrays are borrowed (non-owning, like engine.hpp:70/281).
 * status: 0 ok, 1 invalid argument. */
or_engine* or_engine_create(const uint64_t* offsets, const uint32_t* succ,
                            uint64_t n, const or_config* cfg, int* status);
void or_engine_destroy(or_engine* e);
double or_engine_sum_estimates(or_engine* e);                       /* 100-118 */
void or_engine_step(or_engine* e, double* sum, uint64_t* modified); /* 122-228 */
const uint64_t* or_engine_counters(const or_engine* e);             /* 94 */
unsigned or_engine_words(const or_engine* e);
uint64_t or_engine_iteration(const or_engine* e);
int or_engine_systolic_active(const or_engine* e);
/* engine.hpp:233-275.  Writes up to cap entries; *len = T+1.
 * returns 0 ok, 2 guard (iteration cap), 5 capacity too small. */
int or_engine_run(or_engine* e, double* values, uint64_t* modified,
                  uint64_t cap, uint64_t* len);

/* ---- oracle.hpp / tests/test_util.hpp ------------------------------- */
/* exact_nf (oracle.hpp:38-104): BFS from every source; values[t] = ordered
 * pairs within distance t.  *len = depth.  5 = capacity too small. */
int or_exact_nf(const uint64_t* offsets, const uint32_t* succ, uint64_t n,
                uint64_t* values, uint64_t cap, uint64_t* len);
/* clique_path_nf (oracle.hpp:107-113) */
uint64_t or_clique_path_nf(uint64_t k, uint64_t l, uint64_t t);
/* counter_of(ball(v, t)) (test_util.hpp:16-41): the counter a node must hold
 * after t iterations.  dst: W words. */
void or_counter_of_ball(const uint64_t* offsets, const uint32_t* succ, uint64_t n,
                        uint32_t v, uint64_t radius, const or_params* p, uint64_t* dst);

/* ---- stats.hpp ------------------------------------------------------ */
/* cdf_from_nf + distribution_from_cdf, stats.hpp:33-60. -1 on bad input. */
int or_distance_distribution(const double* nf, uint64_t len, double* mean,
                             double* variance, double* spid);
/* stats.hpp:65-77. -1 on bad input. */
int or_effective_diameter(const double* nf, uint64_t len, double alpha,
                          int interpolated, double* out);

/* ---- hanf_oracle_gen.c (multi-threaded; results thread-independent) -- */
/* BASELINE configs 2/5 R-MAT as the B200 package defines it (hanf_rng.h):
 * 2^scale nodes, edge_factor*2^scale draws, Feistel-permuted ids,
 * self-loops dropped, rows sorted + deduplicated.  -1 bad args, -2 OOM. */
int or_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                uint64_t seed, uint64_t permute_seed, unsigned threads, or_graph* out);
/* order-independent digest of n counters of W words (reference packing) */
uint64_t or_counter_digest(const uint64_t* words, uint64_t n, unsigned W, unsigned threads);
/* digest of a CSR (n+1 offsets, offsets[n] successors) */
uint64_t or_csr_digest(const uint64_t* offsets, const uint32_t* succ, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
