// hyperanf_b200/engine.hpp -- C++ drop-in for the reference engine surface
// (/root/reference/proj/include/hyperanf/engine.hpp) over the C-ABI of
// libhanf.so (include/hanf.h).  Header-only; link with -lhanf.
//
// Replacing the reference path is a namespace change:
//
//     const hyperanf::Graph g = ...;                    // unchanged
//     hyperanf::EngineConfig cfg = ...;                 // unchanged
//     auto est = hyperanf_b200::estimate_nf(g, hyperanf_b200::from_reference(cfg));
//
// Any graph type with num_nodes(), offsets() (u64, n+1) and arcs() (u32)
// is accepted (graph.hpp:46-57), hyperanf::Graph included.  Types, member
// names, argument meaning and exception types follow the reference:
//   EngineConfig      engine.hpp:32-46      IterationReport  engine.hpp:48-51
//   NfEstimate        engine.hpp:53-66      NfEngine         engine.hpp:68-292
//   estimate_nf       engine.hpp:295-298    SketchParams     hll.hpp:36-70
//   std::invalid_argument / GuardError / std::out_of_range / IoError /
//   ParseError as the reference throws them (errors.hpp, hll.hpp:233-235).
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hanf.h"

// With the reference's headers on the include path, its exception types
// are used directly (errors.hpp:8-20): a caller catching
// hyperanf::GuardError catches this engine's iteration-cap error too.
#if defined(__has_include)
#if __has_include(<hyperanf/errors.hpp>)
#include <hyperanf/errors.hpp>
#define HANF_HAVE_REFERENCE_ERRORS 1
#endif
#endif

namespace hyperanf_b200 {

#ifdef HANF_HAVE_REFERENCE_ERRORS
using ParseError = hyperanf::ParseError;
using IoError = hyperanf::IoError;
using GuardError = hyperanf::GuardError;
#else
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct GuardError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#endif
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(hanf_status st) {
  if (st == HANF_OK) return;
  const std::string msg = hanf_last_error();
  switch (st) {
    case HANF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case HANF_GUARD: throw GuardError(msg);
    case HANF_OUT_OF_RANGE: throw std::out_of_range(msg);
    case HANF_OUT_OF_MEMORY: throw std::bad_alloc();
    case HANF_IO_ERROR: throw IoError(msg);
    case HANF_PARSE_ERROR: throw ParseError(msg);
    default: throw DeviceError(msg);
  }
}

enum class Termination { stabilisation, threshold };

inline const char* to_string(Termination t) {
  return t == Termination::stabilisation ? "stabilisation" : "threshold";
}

struct EngineConfig {
  unsigned bucket_bits = 7;
  unsigned register_bits = 0;
  std::uint64_t seed = 0;
  unsigned threads = 1;           // CPU knob, accepted (no effect on the GPU)
  std::uint64_t task_size = 0;    // CPU knob, accepted
  double systolic_threshold = 0.25;
  Termination termination = Termination::stabilisation;
  double eps_inc = 0.0;
  std::uint64_t max_iterations = 0;
  bool spill_to_disk = false;     // accepted: HBM holds both generations
  bool track_modified = true;
  bool use_systolic = true;
  // B200 options (never change a result bit)
  int device = 0;
  bool exact_sum = true;
  std::uint64_t shard_begin = 0, shard_end = 0;
  std::uint32_t shard_count = 0;
  // runs planned on this engine (reseed() between them, main.cpp:263-283);
  // schedules only: from 20, large engines build their source-blocked dense
  // sweeps at construction (hanf_block_stats)
  std::uint32_t expected_runs = 0;
  // several GPUs of this process, one node-range shard each (repeats
  // allowed): NfEngine then drives them all (hanf_create_multi), as the
  // reference's NfEngine keeps its threads internal (engine.hpp:157)
  std::vector<int> devices;

  hanf_config to_c() const {
    hanf_config c;
    check(hanf_config_init(&c));
    c.bucket_bits = bucket_bits;
    c.register_bits = register_bits;
    c.seed = seed;
    c.threads = threads;
    c.task_size = task_size;
    c.systolic_threshold = systolic_threshold;
    c.termination = termination == Termination::threshold ? 1 : 0;
    c.eps_inc = eps_inc;
    c.max_iterations = max_iterations;
    c.spill_to_disk = spill_to_disk;
    c.track_modified = track_modified;
    c.use_systolic = use_systolic;
    c.device = device;
    c.exact_sum = exact_sum;
    c.shard_begin = shard_begin;
    c.shard_end = shard_end;
    c.shard_count = shard_count;
    c.expected_runs = expected_runs;
    return c;
  }
};

// Converts a reference hyperanf::EngineConfig (any type with the same
// member names) field by field.
template <class RefConfig>
EngineConfig from_reference(const RefConfig& r) {
  EngineConfig c;
  c.bucket_bits = r.bucket_bits;
  c.register_bits = r.register_bits;
  c.seed = r.seed;
  c.threads = r.threads;
  c.task_size = r.task_size;
  c.systolic_threshold = r.systolic_threshold;
  c.termination = static_cast<int>(r.termination) == 0 ? Termination::stabilisation
                                                       : Termination::threshold;
  c.eps_inc = r.eps_inc;
  c.max_iterations = r.max_iterations;
  c.spill_to_disk = r.spill_to_disk;
  c.track_modified = r.track_modified;
  c.use_systolic = r.use_systolic;
  return c;
}

struct IterationReport {
  double sum = 0.0;
  std::uint64_t modified = 0;
};

struct NfEstimate {
  std::uint64_t n = 0;
  unsigned m = 0;
  std::uint64_t seed = 0;
  Termination termination = Termination::stabilisation;
  std::vector<double> values;
  std::vector<std::uint64_t> modified;
  double wall_seconds = 0.0;
  bool exact = false;
  std::uint64_t iterations() const noexcept { return values.empty() ? 0 : values.size() - 1; }
};

struct SketchParams {
  unsigned bucket_bits = 7, registers = 128, register_bits = 5;
  double alpha = 0.0;
  std::uint64_t seed = 0;
  unsigned words = 10;
  static SketchParams make(unsigned b, std::uint64_t seed, unsigned r = 5) {
    hanf_sketch_params p;
    check(hanf_sketch_params_make(b, seed, r, &p));
    return from_c(p);
  }
  static SketchParams from_c(const hanf_sketch_params& p) {
    SketchParams s;
    s.bucket_bits = p.bucket_bits;
    s.registers = p.registers;
    s.register_bits = p.register_bits;
    s.alpha = p.alpha;
    s.seed = p.seed;
    s.words = p.words_per_counter;
    return s;
  }
  unsigned words_per_counter() const noexcept { return words; }
  unsigned max_register_value() const noexcept { return (1u << register_bits) - 1; }
};

template <class G>
hanf_graph_view view_of(const G& g) {
  hanf_graph_view v;
  v.n = g.num_nodes();
  v.num_arcs = g.arcs().size();
  v.offsets = g.offsets().data();
  v.arcs = g.arcs().data();
  return v;
}

class NfEngine {
 public:
  template <class G>
  NfEngine(const G& graph, EngineConfig cfg) : cfg_(cfg), n_(graph.num_nodes()) {
    const hanf_graph_view v = view_of(graph);
    const hanf_config c = cfg_.to_c();
    if (cfg_.devices.empty())
      check(hanf_create(&v, &c, &h_));
    else
      check(hanf_create_multi(&v, &c, cfg_.devices.data(),
                              static_cast<std::uint32_t>(cfg_.devices.size()), &h_));
    hanf_sketch_params p;
    check(hanf_params(h_, &p));
    params_ = SketchParams::from_c(p);
  }
  NfEngine(const NfEngine&) = delete;
  NfEngine& operator=(const NfEngine&) = delete;
  ~NfEngine() { hanf_destroy(h_); }

  const SketchParams& params() const noexcept { return params_; }
  const EngineConfig& config() const noexcept { return cfg_; }
  // NfEngine::counters() (engine.hpp:94): the current generation in the
  // reference packing (CounterArray::data(), hll.hpp:224), as a stable
  // reference to a host mirror that is refreshed from HBM only after the
  // counters changed (step, reset, reseed, restore)
  const std::vector<std::uint64_t>& counters() const {
    if (mirror_version_ != version_) {
      mirror_.resize(static_cast<size_t>(n_) * params_.words);
      check(hanf_read_counters(h_, 0, n_, mirror_.data()));
      mirror_version_ = version_;
    }
    return mirror_;
  }
  std::vector<std::uint64_t> counter(std::uint64_t i) const {
    std::vector<std::uint64_t> out(params_.words);
    check(hanf_read_counters(h_, i, 1, out.data()));
    return out;
  }
  std::uint64_t iteration() const {
    std::uint64_t t = 0;
    check(hanf_iteration(h_, &t));
    return t;
  }
  bool systolic_active() const {
    int32_t a = 0;
    check(hanf_systolic_active(h_, &a));
    return a != 0;
  }
  double sum_estimates() {
    double s = 0.0;
    check(hanf_sum_estimates(h_, &s));
    return s;
  }
  IterationReport step() {
    hanf_iteration_report r;
    ++version_;
    check(hanf_step(h_, &r));
    return {r.sum, r.modified};
  }
  NfEstimate run_to_stabilisation() {
    ++version_;
    NfEstimate est;
    est.n = n_;
    est.m = params_.registers;
    est.seed = params_.seed;
    est.termination = cfg_.termination;
    std::uint64_t len = 0;
    double wall = 0.0;
    std::vector<double> vals(64);
    std::vector<std::uint64_t> mods(64);
    hanf_status st = hanf_run_to_stabilisation(h_, vals.data(), mods.data(), vals.size(), &len, &wall);
    if (st == HANF_CAPACITY) {
      vals.resize(len);
      mods.resize(len);
      st = hanf_last_result(h_, vals.data(), mods.data(), len, &len);
    }
    check(st);
    vals.resize(len);
    mods.resize(len);
    est.values = std::move(vals);
    est.modified = std::move(mods);
    est.wall_seconds = wall;
    return est;
  }
  void reset() {
    ++version_;
    check(hanf_reset(h_));
  }
  // the next run of a multi-seed experiment on the uploaded graph (new)
  void reseed(std::uint64_t seed) {
    ++version_;
    check(hanf_reseed(h_, seed));
    cfg_.seed = seed;
    params_.seed = seed;
  }
  // (new) items and arcs of the engine's source-blocked dense sweeps, {0, 0}
  // on the plain schedule (hanf_block_stats; results never depend on it)
  std::pair<std::uint64_t, std::uint64_t> block_stats() const {
    std::uint64_t items = 0, arcs = 0;
    check(hanf_block_stats(h_, &items, &arcs));
    return {items, arcs};
  }
  // hll.hpp:275-286 save_counters of the current counters (same bytes)
  void save_counters(const std::string& path) const { check(hanf_save_counters(h_, path.c_str())); }
  // resume from an HCA1 snapshot taken at `iteration` (new; hll.hpp:288-303 format)
  void restore_counters(const std::string& path, std::uint64_t iteration) {
    ++version_;
    check(hanf_restore_counters(h_, path.c_str(), iteration));
    hanf_sketch_params p;
    check(hanf_params(h_, &p));
    params_ = SketchParams::from_c(p);
    cfg_.seed = params_.seed;
  }
  hanf_engine* handle() noexcept { return h_; }

 private:
  EngineConfig cfg_;
  std::uint64_t n_ = 0;
  SketchParams params_;
  hanf_engine* h_ = nullptr;
  std::uint64_t version_ = 0;                      // bumped by every mutating call
  mutable std::uint64_t mirror_version_ = ~0ull;
  mutable std::vector<std::uint64_t> mirror_;
};

// One node range of a multi-GPU run (new; the reference has no distributed
// engine).  Peer-push exchange (hanf.h): every rank exports its arena,
// the caller's transport (MPI, sockets, torch.distributed) all-gathers the
// descriptors, attach() maps the peers; a step is compute(), a barrier
// across the ranks after compute() returned, then commit() - the same
// IterationReport on every rank, equal to the single engine's bit for bit.
class ShardEngine {
 public:
  template <class G>
  ShardEngine(const G& graph, EngineConfig cfg, std::uint64_t begin, std::uint64_t end,
              std::uint32_t shards)
      : n_(graph.num_nodes()) {
    const hanf_graph_view v = view_of(graph);
    hanf_config c = cfg.to_c();
    c.shard_begin = begin;
    c.shard_end = end;
    c.shard_count = shards;
    check(hanf_create(&v, &c, &h_));
  }
  ShardEngine(const ShardEngine&) = delete;
  ShardEngine& operator=(const ShardEngine&) = delete;
  ~ShardEngine() {
    hanf_shard_detach(h_);
    hanf_destroy(h_);
  }
  hanf_shard_peer export_peer() const {
    hanf_shard_peer p;
    check(hanf_shard_export(h_, &p));
    return p;
  }
  // peers = every rank's export_peer(), in rank order; self = this rank
  void attach(const std::vector<hanf_shard_peer>& peers, std::uint32_t self) {
    check(hanf_shard_attach(h_, peers.data(), static_cast<std::uint32_t>(peers.size()), self));
  }
  // shards of one process (same device, or peer access between them)
  static void attach_local(const std::vector<ShardEngine*>& shards) {
    std::vector<hanf_engine*> hs;
    for (auto* s : shards) hs.push_back(s->h_);
    for (std::uint32_t k = 0; k < hs.size(); ++k)
      check(hanf_shard_attach_local(hs[k], hs.data(), static_cast<std::uint32_t>(hs.size()), k));
  }
  // enqueue this range's sweep (rows pushed to the peers) and wait for it
  void compute() {
    check(hanf_shard_compute(h_));
    check(hanf_shard_wait(h_));
  }
  // relabelled shards, optional, between compute's barrier and a second
  // one: re-sum this rank's slice of the block sums (hanf_shard_reduce)
  void reduce() {
    check(hanf_shard_reduce(h_));
    check(hanf_shard_wait(h_));
  }
  IterationReport commit() {
    hanf_iteration_report r;
    check(hanf_shard_commit(h_, &r));
    return {r.sum, r.modified};
  }
  double sum_estimates() {
    double s = 0.0;
    check(hanf_sum_estimates(h_, &s));
    return s;
  }
  std::vector<std::uint64_t> counters() const {
    hanf_sketch_params p;
    check(hanf_params(h_, &p));
    std::vector<std::uint64_t> out(static_cast<size_t>(n_) * p.words_per_counter);
    check(hanf_read_counters(h_, 0, n_, out.data()));
    return out;
  }
  void detach() { check(hanf_shard_detach(h_)); }
  hanf_engine* handle() noexcept { return h_; }

 private:
  std::uint64_t n_ = 0;
  hanf_engine* h_ = nullptr;
};

template <class G>
NfEstimate estimate_nf(const G& g, const EngineConfig& cfg) {
  NfEngine engine(g, cfg);
  return engine.run_to_stabilisation();
}

// main.cpp:263-283 multirun: estimate_nf for seeds base + i, on one engine
template <class G>
std::vector<NfEstimate> multirun(const G& g, EngineConfig cfg, std::uint64_t runs,
                                 std::uint64_t base_seed) {
  std::vector<NfEstimate> out;
  if (runs == 0) return out;
  cfg.seed = base_seed;
  NfEngine engine(g, cfg);
  for (std::uint64_t i = 0; i < runs; ++i) {
    if (i) engine.reseed(base_seed + i);
    out.push_back(engine.run_to_stabilisation());
  }
  return out;
}

// oracle.hpp:24-104: the exact neighbourhood function, on the GPU, with the
// reference's guard (GuardError past max_nodes / max_work = n * arcs)
struct ExactNf {
  std::uint64_t n = 0;
  std::vector<std::uint64_t> values;
  std::uint64_t diameter() const noexcept { return values.empty() ? 0 : values.size() - 1; }
  std::vector<double> as_doubles() const { return {values.begin(), values.end()}; }
};
template <class G>
ExactNf exact_nf(const G& g, int device = 0, std::uint64_t max_nodes = 1'000'000,
                 std::uint64_t max_work = 100'000'000'000ULL) {
  const hanf_graph_view v = view_of(g);
  ExactNf out;
  out.n = v.n;
  std::uint64_t len = 0;
  std::vector<std::uint64_t> vals(64);
  hanf_status st = hanf_exact_nf(&v, device, max_nodes, max_work, vals.data(), vals.size(), &len);
  if (st == HANF_CAPACITY) {
    vals.resize(len);
    st = hanf_exact_nf(&v, device, max_nodes, max_work, vals.data(), vals.size(), &len);
  }
  check(st);
  vals.resize(len);
  out.values = std::move(vals);
  return out;
}

// stats.hpp:44-77 on an N(t) vector
struct DistanceDistribution {
  double mean = 0.0, variance = 0.0, spid = 0.0;
};
inline DistanceDistribution distance_distribution(const std::vector<double>& nf) {
  DistanceDistribution d;
  check(hanf_distance_distribution(nf.data(), nf.size(), &d.mean, &d.variance, &d.spid));
  return d;
}
inline double effective_diameter(const std::vector<double>& nf, double alpha = 0.9,
                                 bool interpolated = false) {
  double out = 0.0;
  check(hanf_effective_diameter(nf.data(), nf.size(), alpha, interpolated ? 1 : 0, &out));
  return out;
}

}  // namespace hyperanf_b200
