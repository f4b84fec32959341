// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference engine.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  This file contains no reference
// source: it #includes the reference's own headers by include path
// (-I$(REF)/proj/include, see oracle/Makefile) and exposes extern "C"
// entry points so the parity tests and bench.py's reference arm can drive
// hyperanf::NfEngine (engine.hpp:68-292) on the same CSR the B200 engine
// uses.  Output goes to oracle/_ref/ (git-ignored, travels with gpurun).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "hyperanf/engine.hpp"
#include "hyperanf/graph.hpp"
#include "hyperanf/hll.hpp"
#include "hyperanf/oracle.hpp"
#include "hyperanf/stats.hpp"

using namespace hyperanf;

namespace {
int status_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const GuardError&) {
    return 2;
  } catch (const std::out_of_range&) {
    return 1;
  } catch (...) {
    return 3;
  }
}

EngineConfig make_cfg(unsigned b, unsigned r, uint64_t seed, unsigned threads,
                      uint64_t task_size, double systolic_threshold,
                      int termination, double eps_inc, uint64_t max_iterations,
                      int track_modified, int use_systolic) {
  EngineConfig cfg;
  cfg.bucket_bits = b;
  cfg.register_bits = r;
  cfg.seed = seed;
  cfg.threads = threads;
  cfg.task_size = task_size;
  cfg.systolic_threshold = systolic_threshold;
  cfg.termination = termination ? Termination::threshold : Termination::stabilisation;
  cfg.eps_inc = eps_inc;
  cfg.max_iterations = max_iterations;
  cfg.track_modified = track_modified != 0;
  cfg.use_systolic = use_systolic != 0;
  return cfg;
}
}  // namespace

extern "C" {

// ---- graphs ---------------------------------------------------------------
void* ref_graph_from_csr(uint64_t n, const uint64_t* offsets, const uint32_t* succ) {
  std::vector<std::pair<uint32_t, uint32_t>> edges;
  edges.reserve(offsets[n]);
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t i = offsets[v]; i < offsets[v + 1]; ++i)
      edges.emplace_back(static_cast<uint32_t>(v), succ[i]);
  return new Graph(Graph::from_edges(n, std::move(edges)));
}
void* ref_gen_uniform_random(uint64_t n, double d, uint64_t seed) {
  try { return new Graph(gen_uniform_random(n, d, seed)); } catch (...) { return nullptr; }
}
void* ref_gen_clique_path(uint64_t k, uint64_t l) {
  try { return new Graph(gen_clique_path(k, l)); } catch (...) { return nullptr; }
}
uint64_t ref_graph_nodes(const void* g) { return static_cast<const Graph*>(g)->num_nodes(); }
uint64_t ref_graph_arcs(const void* g) { return static_cast<const Graph*>(g)->num_arcs(); }
void ref_graph_csr(const void* g, uint64_t* offsets, uint32_t* succ) {
  const Graph* gr = static_cast<const Graph*>(g);
  std::memcpy(offsets, gr->offsets().data(), sizeof(uint64_t) * gr->offsets().size());
  if (gr->num_arcs()) std::memcpy(succ, gr->arcs().data(), sizeof(uint32_t) * gr->num_arcs());
}
void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

// ---- engine ---------------------------------------------------------------
void* ref_engine_create(const void* g, unsigned b, unsigned r, uint64_t seed,
                        unsigned threads, uint64_t task_size,
                        double systolic_threshold, int termination,
                        double eps_inc, uint64_t max_iterations,
                        int track_modified, int use_systolic, int* status) {
  *status = 0;
  try {
    return new NfEngine(*static_cast<const Graph*>(g),
                        make_cfg(b, r, seed, threads, task_size, systolic_threshold,
                                 termination, eps_inc, max_iterations,
                                 track_modified, use_systolic));
  } catch (...) {
    *status = status_of(std::current_exception());
    return nullptr;
  }
}
void ref_engine_free(void* e) { delete static_cast<NfEngine*>(e); }
double ref_engine_sum_estimates(void* e) { return static_cast<NfEngine*>(e)->sum_estimates(); }
void ref_engine_step(void* e, double* sum, uint64_t* modified) {
  const IterationReport rep = static_cast<NfEngine*>(e)->step();
  *sum = rep.sum;
  *modified = rep.modified;
}
const uint64_t* ref_engine_counters(const void* e, uint64_t* word_count) {
  const CounterArray& c = static_cast<const NfEngine*>(e)->counters();
  *word_count = c.word_count();
  return c.data();
}
uint64_t ref_engine_iteration(const void* e) { return static_cast<const NfEngine*>(e)->iteration(); }
// hll.hpp:275-286 save_counters of the engine's current counters; 0 ok, 4 io
int ref_engine_save_counters(const void* e, const char* path) {
  try {
    hyperanf::save_counters(static_cast<const NfEngine*>(e)->counters(), path);
    return 0;
  } catch (...) {
    return 4;
  }
}
int ref_engine_systolic_active(const void* e) { return static_cast<const NfEngine*>(e)->systolic_active(); }

// NfEngine::run_to_stabilisation (engine.hpp:233-275).  0 ok, 1 invalid,
// 2 guard, 3 other, 5 capacity.
int ref_engine_run(void* e, double* values, uint64_t* modified, uint64_t cap,
                   uint64_t* len, double* wall_seconds) {
  try {
    const NfEstimate est = static_cast<NfEngine*>(e)->run_to_stabilisation();
    *len = est.values.size();
    *wall_seconds = est.wall_seconds;
    if (est.values.size() > cap) return 5;
    for (size_t i = 0; i < est.values.size(); ++i) {
      values[i] = est.values[i];
      modified[i] = est.modified[i];
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// Times one NfEngine::step() with steady_clock, as tests/acceptance.cpp:438-443.
double ref_engine_timed_step(void* e, double* sum, uint64_t* modified) {
  const auto t0 = std::chrono::steady_clock::now();
  const IterationReport rep = static_cast<NfEngine*>(e)->step();
  const auto t1 = std::chrono::steady_clock::now();
  *sum = rep.sum;
  *modified = rep.modified;
  return std::chrono::duration<double>(t1 - t0).count();
}

// ---- sketch primitives (hll.hpp) ------------------------------------------
int ref_params(unsigned b, unsigned r, uint64_t seed, unsigned* words, double* alpha) {
  try {
    const auto p = SketchParams::make(b, seed, r);
    *words = p.words_per_counter();
    *alpha = p.alpha;
    return 0;
  } catch (...) {
    return 1;
  }
}
int ref_counter_add(uint64_t* words, unsigned b, unsigned r, uint64_t seed, uint64_t item) {
  const auto p = SketchParams::make(b, seed, r);
  return counter_add(RegisterView(words, p.words_per_counter()), p, item) ? 1 : 0;
}
double ref_counter_estimate(const uint64_t* words, unsigned b, unsigned r) {
  const auto p = SketchParams::make(b, 0, r);
  return counter_estimate(ConstRegisterView(words, p.words_per_counter()), p);
}
int ref_counter_union(uint64_t* dst, const uint64_t* src, unsigned b, unsigned r) {
  const auto p = SketchParams::make(b, 0, r);
  return counter_union(RegisterView(dst, p.words_per_counter()),
                       ConstRegisterView(src, p.words_per_counter()), p) ? 1 : 0;
}
unsigned ref_read_register(const uint64_t* words, unsigned b, unsigned r, unsigned j) {
  const auto p = SketchParams::make(b, 0, r);
  return read_register(ConstRegisterView(words, p.words_per_counter()), p, j);
}
void ref_write_register(uint64_t* words, unsigned b, unsigned r, unsigned j, unsigned v) {
  const auto p = SketchParams::make(b, 0, r);
  write_register(RegisterView(words, p.words_per_counter()), p, j, v);
}

// ---- stats.hpp ---------------------------------------------------------------
int ref_distance_distribution(const double* nf, uint64_t len, double* mean,
                              double* variance, double* spid) {
  try {
    const auto d = distribution_from_cdf(cdf_from_nf(std::span<const double>(nf, len)));
    *mean = d.mean;
    *variance = d.variance;
    *spid = d.spid;
    return 0;
  } catch (...) {
    return 1;
  }
}
int ref_effective_diameter(const double* nf, uint64_t len, double alpha,
                           int interpolated, double* out) {
  try {
    *out = effective_diameter(std::span<const double>(nf, len), alpha, interpolated != 0);
    return 0;
  } catch (...) {
    return 1;
  }
}

// ---- oracle.hpp (exact NF by BFS) -------------------------------------------
int ref_exact_nf(const void* g, uint64_t* values, uint64_t cap, uint64_t* len) {
  try {
    const ExactNf ex = exact_nf(*static_cast<const Graph*>(g));
    *len = ex.values.size();
    if (ex.values.size() > cap) return 5;
    for (size_t i = 0; i < ex.values.size(); ++i) values[i] = ex.values[i];
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

unsigned ref_hardware_threads(void) { return std::thread::hardware_concurrency(); }

}  // extern "C"
