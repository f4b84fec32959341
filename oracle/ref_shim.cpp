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
// Access to the reference's private members without editing its headers:
// an explicit template instantiation may name private members (C++
// [temp.spec]), and the friend it defines hands the member pointer out.
// Used for two things only: building a hyperanf::Graph from an already
// sorted, deduplicated CSR in O(a) (from_edges' std::sort of 4.3 B pairs
// takes minutes at config 5), and running NfEngine::step's per-node body
// over a node range (ref_engine_step_sample).
template <typename Tag, typename Tag::type M>
struct Rob {
  friend typename Tag::type get(Tag) { return M; }
};
#define HANF_ROB(Name, Class, Type, Member)                   \
  struct Name {                                               \
    using type = Type Class::*;                               \
    friend type get(Name);                                    \
  };                                                          \
  template struct Rob<Name, &Class::Member>;
HANF_ROB(GraphN, Graph, std::uint64_t, n_)
HANF_ROB(GraphOff, Graph, std::vector<std::uint64_t>, offsets_)
HANF_ROB(GraphSucc, Graph, std::vector<std::uint32_t>, succ_)
HANF_ROB(EngGraph, NfEngine, const Graph*, graph_)
HANF_ROB(EngCfg, NfEngine, EngineConfig, cfg_)
HANF_ROB(EngKernel, NfEngine, PackedMax, kernel_)
HANF_ROB(EngCur, NfEngine, CounterArray, current_)
HANF_ROB(EngNext, NfEngine, CounterArray, next_)
HANF_ROB(EngParams, NfEngine, SketchParams, params_)
HANF_ROB(EngMod, NfEngine, std::vector<std::uint8_t>, modified_)
HANF_ROB(EngNextMod, NfEngine, std::vector<std::uint8_t>, next_modified_)
#undef HANF_ROB

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
// The same Graph as from_edges would build from this CSR, without the
// sort: the caller guarantees rows sorted and deduplicated with ids < n
// (checked here in O(a)).  nullptr if the CSR is not in that form.
void* ref_graph_from_sorted_csr(uint64_t n, const uint64_t* offsets, const uint32_t* succ) {
  try {
    if (offsets[0] != 0) return nullptr;
    const uint64_t a = offsets[n];
    for (uint64_t v = 0; v < n; ++v) {
      if (offsets[v + 1] < offsets[v]) return nullptr;
      for (uint64_t i = offsets[v]; i < offsets[v + 1]; ++i)
        if (succ[i] >= n || (i > offsets[v] && succ[i] <= succ[i - 1])) return nullptr;
    }
    Graph* g = new Graph();
    g->*get(GraphN{}) = n;
    (g->*get(GraphOff{})).assign(offsets, offsets + n + 1);
    (g->*get(GraphSucc{})).assign(succ, succ + a);
    return g;
  } catch (...) {
    return nullptr;
  }
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

// A bounded sample of one dense iteration of the reference engine: the
// per-node body of NfEngine::step (engine.hpp:157-184, non-systolic,
// in-memory) over nodes [lo, hi) only, dealt to `threads` workers by the
// reference's own parallel_chunks (parallel.hpp:16-48, chunk task_size),
// followed by the per-block re-sum of sum_estimates (engine.hpp:100-112)
// over the blocks of [lo, hi) on the freshly written counters.  It writes
// next_ / next_modified_ of those nodes and never swaps, so repeated
// samples all start from the same generation (the bench samples iteration
// 1 from the seeded state).  Returns the seconds (steady_clock, as
// tests/acceptance.cpp:438-443), and the sampled arcs and block sum.
double ref_engine_step_sample(void* ep, uint64_t lo, uint64_t hi, unsigned threads,
                              uint64_t* arcs_out, double* sum_out, uint64_t* changed_out) {
  NfEngine* e = static_cast<NfEngine*>(ep);
  const Graph& g = *(e->*get(EngGraph{}));
  const EngineConfig& cfg = e->*get(EngCfg{});
  const PackedMax& kernel = e->*get(EngKernel{});
  CounterArray& cur = e->*get(EngCur{});
  CounterArray& next = e->*get(EngNext{});
  const SketchParams& params = e->*get(EngParams{});
  const std::vector<std::uint8_t>& modified = e->*get(EngMod{});
  std::vector<std::uint8_t>& next_modified = e->*get(EngNextMod{});
  const uint64_t n = g.num_nodes();
  if (hi > n) hi = n;
  if (lo >= hi) {
    *arcs_out = 0;
    *sum_out = 0.0;
    *changed_out = 0;
    return 0.0;
  }
  const unsigned words = params.words_per_counter();
  if (next.size() != n) next = CounterArray(params, n);      // engine.hpp:126
  if (next_modified.size() != n) next_modified.assign(n, 0);  // engine.hpp:127
  if (threads == 0) threads = 1;
  std::vector<std::vector<std::uint64_t>> scratch(threads, std::vector<std::uint64_t>(words));
  constexpr uint64_t kBlock = 64;
  const uint64_t b0 = lo / kBlock, b1 = (hi + kBlock - 1) / kBlock;
  std::vector<double> block_sums(b1 - b0, 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  parallel_chunks(hi - lo, threads, cfg.task_size,
                  [&](std::uint64_t clo, std::uint64_t chi, unsigned id) {
    for (std::uint64_t v = lo + clo; v < lo + chi; ++v) {
      std::uint64_t* dst = next.counter(v).data();
      std::memcpy(dst, cur.counter(v).data(), words * sizeof(std::uint64_t));
      bool changed = false;
      for (std::uint32_t succ : g.successors(v)) {
        if (cfg.track_modified && !modified[succ]) continue;
        changed |= kernel.max_into(dst, cur.counter(succ).data(), scratch[id].data());
      }
      next_modified[v] = changed ? 1 : 0;
    }
  });
  parallel_chunks(b1 - b0, threads, 16, [&](std::uint64_t blo, std::uint64_t bhi, unsigned) {
    for (std::uint64_t b = b0 + blo; b < b0 + bhi; ++b) {
      const std::uint64_t first = std::max<std::uint64_t>(b * kBlock, lo);
      const std::uint64_t last = std::min<std::uint64_t>((b + 1) * kBlock, hi);
      double sum = 0.0;
      for (std::uint64_t i = first; i < last; ++i) sum += next.estimate(i);
      block_sums[b - b0] = sum;
    }
  });
  const auto t1 = std::chrono::steady_clock::now();
  double total = 0.0;
  for (double s : block_sums) total += s;
  uint64_t changed = 0;
  for (uint64_t v = lo; v < hi; ++v) changed += next_modified[v];
  *arcs_out = g.offsets()[hi] - g.offsets()[lo];
  *sum_out = total;
  *changed_out = changed;
  return std::chrono::duration<double>(t1 - t0).count();
}
// Allocates next_ / next_modified_ as step() would (engine.hpp:126-127) and
// touches every page with `threads` workers, so step samples measure the
// steady state rather than first-touch page faults of iteration 1.
void ref_engine_prefault(void* ep, unsigned threads) {
  NfEngine* e = static_cast<NfEngine*>(ep);
  const uint64_t n = (e->*get(EngGraph{}))->num_nodes();
  const SketchParams& params = e->*get(EngParams{});
  CounterArray& next = e->*get(EngNext{});
  std::vector<std::uint8_t>& next_modified = e->*get(EngNextMod{});
  if (next.size() != n) next = CounterArray(params, n);
  if (next_modified.size() != n) next_modified.assign(n, 0);
  const unsigned words = params.words_per_counter();
  parallel_chunks(n, threads ? threads : 1, 1 << 16,
                  [&](std::uint64_t lo, std::uint64_t hi, unsigned) {
    std::memset(next.counter(lo).data(), 0, (hi - lo) * words * sizeof(std::uint64_t));
  });
}
// next_ after samples (the sampled rows are the step's rows)
const uint64_t* ref_engine_next_counters(const void* ep, uint64_t* word_count) {
  const NfEngine* e = static_cast<const NfEngine*>(ep);
  const CounterArray& c = const_cast<NfEngine*>(e)->*get(EngNext{});
  *word_count = c.word_count();
  return c.data();
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
