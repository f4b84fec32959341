// dropin_test.cpp -- the C++ drop-in check: the reference engine
// (hyperanf::NfEngine, compiled from the reference's own headers) and the
// B200 engine behind include/hyperanf_b200/engine.hpp run on the SAME
// hyperanf::Graph objects, in lockstep.  Test infrastructure: built by
// oracle/Makefile into oracle/_ref/ (it contains reference code), run by
// tests/test_gpu_dropin.py on the GPU box.  Exit 0 = every check passed.
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hyperanf/engine.hpp"
#include "hyperanf/graph.hpp"
#include "hyperanf/hll.hpp"
#include "hyperanf/oracle.hpp"
#include "hyperanf/stats.hpp"
#include "hyperanf_b200/engine.hpp"

namespace {
int failures = 0;
void expect(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("FAIL %s\n", what.c_str());
  }
}

void lockstep(const hyperanf::Graph& g, const hyperanf::EngineConfig& cfg, const char* name) {
  hyperanf::NfEngine ref(g, cfg);
  hyperanf_b200::NfEngine gpu(g, hyperanf_b200::from_reference(cfg));
  const auto& rc = ref.counters();
  expect(ref.sum_estimates() == gpu.sum_estimates(), std::string(name) + " N(0)");
  expect(std::vector<std::uint64_t>(rc.data(), rc.data() + rc.word_count()) == gpu.counters(),
         std::string(name) + " seeded counters");
  for (std::uint64_t t = 1; t <= g.num_nodes() + 1; ++t) {
    const auto a = ref.step();
    const auto b = gpu.step();
    const auto& c = ref.counters();
    const bool same = a.sum == b.sum && a.modified == b.modified &&
                      std::vector<std::uint64_t>(c.data(), c.data() + c.word_count()) ==
                          gpu.counters() &&
                      ref.systolic_active() == gpu.systolic_active() &&
                      ref.iteration() == gpu.iteration();
    expect(same, std::string(name) + " step " + std::to_string(t));
    if (!same || a.modified == 0) break;
  }
  const auto ea = hyperanf::estimate_nf(g, cfg);
  const auto eb = hyperanf_b200::estimate_nf(g, hyperanf_b200::from_reference(cfg));
  expect(ea.values == eb.values && ea.modified == eb.modified, std::string(name) + " estimate_nf");
  if (!ea.values.empty() && ea.values.back() > 0) {
    const auto da = hyperanf::distribution_from_cdf(hyperanf::cdf_from_nf(ea.values));
    const auto db = hyperanf_b200::distance_distribution(eb.values);
    expect(da.spid == db.spid && da.mean == db.mean, std::string(name) + " spid");
    expect(hyperanf::effective_diameter(ea.values, 0.9, true) ==
               hyperanf_b200::effective_diameter(eb.values, 0.9, true),
           std::string(name) + " interpolated effective diameter");
  }
}
// hanf_create_multi through the drop-in: EngineConfig::devices lists one
// device per shard (here repeats of device 0: one GPU on the test box)
void lockstep_multi(const hyperanf::Graph& g, const hyperanf::EngineConfig& cfg,
                    std::vector<int> devices, const std::string& name) {
  hyperanf::NfEngine ref(g, cfg);
  hyperanf_b200::EngineConfig bc = hyperanf_b200::from_reference(cfg);
  bc.devices = devices;
  hyperanf_b200::NfEngine gpu(g, bc);
  const auto& rc0 = ref.counters();
  expect(ref.sum_estimates() == gpu.sum_estimates(), name + " N(0)");
  expect(std::vector<std::uint64_t>(rc0.data(), rc0.data() + rc0.word_count()) == gpu.counters(),
         name + " seeded counters");
  for (std::uint64_t t = 1; t <= g.num_nodes() + 1; ++t) {
    const auto a = ref.step();
    const auto b = gpu.step();
    const auto& c = ref.counters();
    const bool same = a.sum == b.sum && a.modified == b.modified &&
                      std::vector<std::uint64_t>(c.data(), c.data() + c.word_count()) ==
                          gpu.counters() &&
                      ref.iteration() == gpu.iteration();
    expect(same, name + " step " + std::to_string(t));
    if (!same || a.modified == 0) break;
  }
  const auto ea = hyperanf::estimate_nf(g, cfg);
  gpu.reset();
  const auto eb = gpu.run_to_stabilisation();
  expect(ea.values == eb.values && ea.modified == eb.modified, name + " reset + run");
  const auto ec = hyperanf_b200::estimate_nf(g, bc);
  expect(ea.values == ec.values, name + " estimate_nf");
}
}  // namespace

int main() {
  struct Case {
    hyperanf::Graph g;
    unsigned b, r;
    std::uint64_t seed;
    const char* name;
  };
  std::vector<std::pair<std::uint32_t, std::uint32_t>> path;
  for (std::uint32_t v = 0; v + 1 < 64; ++v) path.emplace_back(v, v + 1);
  std::vector<Case> cases;
  cases.push_back({hyperanf::gen_uniform_random(60, 3, 21), 6, 6, 77, "balls60 r6"});
  cases.push_back({hyperanf::gen_uniform_random(500, 5, 31), 7, 0, 8, "ur500"});
  cases.push_back({hyperanf::gen_clique_path(260, 10), 8, 0, 42, "clique-path 260/10"});
  cases.push_back({hyperanf::gen_clique_path(1100, 3), 6, 0, 42, "clique-path 1100/3 (hubs)"});
  cases.push_back({hyperanf::Graph::from_edges(64, path), 6, 0, 2, "64-path"});
  cases.push_back({hyperanf::gen_uniform_random(20000, 12, 5), 5, 0, 1, "ur20000 b5"});
  cases.push_back({hyperanf::gen_uniform_random(3000, 7, 9), 9, 0, 3, "ur3000 b9"});
  for (const auto& c : cases) {
    hyperanf::EngineConfig cfg;
    cfg.bucket_bits = c.b;
    cfg.register_bits = c.r;
    cfg.seed = c.seed;
    lockstep(c.g, cfg, c.name);
  }
  // error behaviour: same exception types as the reference
  const hyperanf::Graph one = hyperanf::Graph::from_edges(1, {});
  hyperanf::EngineConfig bad;
  bad.systolic_threshold = 0.0;
  try {
    hyperanf_b200::NfEngine e(one, hyperanf_b200::from_reference(bad));
    expect(false, "invalid systolic threshold accepted");
  } catch (const std::invalid_argument&) {
  }
  hyperanf::EngineConfig capped;
  capped.bucket_bits = 6;
  capped.seed = 1;
  capped.max_iterations = 2;
  try {
    hyperanf_b200::estimate_nf(hyperanf::gen_clique_path(4, 8),
                               hyperanf_b200::from_reference(capped));
    expect(false, "iteration cap not enforced");
  } catch (const hyperanf::GuardError&) {  // the reference's own type (aliased)
  }
  // exact NF (oracle.hpp) against the reference's all-pairs BFS
  for (const auto& g : {hyperanf::gen_uniform_random(2000, 4, 3), hyperanf::gen_clique_path(20, 9)}) {
    const auto want = hyperanf::exact_nf(g);
    const auto got = hyperanf_b200::exact_nf(g);
    expect(got.values == want.values, "exact_nf values");
  }
  try {
    hyperanf_b200::exact_nf(hyperanf::gen_uniform_random(2000, 4, 3), 0, 100);
    expect(false, "exact_nf guard not enforced");
  } catch (const hyperanf_b200::GuardError&) {
  }
  // multirun: every seed equals its own estimate_nf; snapshots equal the
  // reference's save_counters bytes
  {
    const hyperanf::Graph g = hyperanf::gen_uniform_random(3000, 6, 2);
    hyperanf::EngineConfig cfg;
    cfg.bucket_bits = 6;
    const auto runs = hyperanf_b200::multirun(g, hyperanf_b200::from_reference(cfg), 3, 50);
    for (std::uint64_t i = 0; i < runs.size(); ++i) {
      hyperanf::EngineConfig c = cfg;
      c.seed = 50 + i;
      const auto ref_est = hyperanf::estimate_nf(g, c);
      expect(runs[i].values == ref_est.values, "multirun seed " + std::to_string(50 + i));
    }
    hyperanf::EngineConfig c = cfg;
    c.seed = 7;
    hyperanf::NfEngine ref(g, c);
    hyperanf_b200::NfEngine gpu(g, hyperanf_b200::from_reference(c));
    ref.step();
    gpu.step();
    const std::string a = "/tmp/dropin_ref.hca", b = "/tmp/dropin_gpu.hca";
    hyperanf::save_counters(ref.counters(), a);
    gpu.save_counters(b);
    auto slurp = [](const std::string& p) {
      std::FILE* f = std::fopen(p.c_str(), "rb");
      std::string d;
      if (!f) return d;
      char buf[4096];
      size_t k;
      while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) d.append(buf, k);
      std::fclose(f);
      return d;
    };
    expect(!slurp(a).empty() && slurp(a) == slurp(b), "HCA1 snapshot bytes");
    std::remove(a.c_str());
    std::remove(b.c_str());
  }
  {  // multi-GPU path in C++: 2 and 3 peer-push shards of one process
     // against the reference engine, every iteration
    const auto g = hyperanf::gen_uniform_random(3000, 6.0, 17);
    hyperanf::EngineConfig c;
    c.bucket_bits = 6;
    c.seed = 5;
    for (std::uint32_t k : {2u, 3u}) {
      const std::uint64_t n = g.num_nodes(), per = ((n + k - 1) / k + 63) / 64 * 64;
      std::vector<std::unique_ptr<hyperanf_b200::ShardEngine>> own;
      std::vector<hyperanf_b200::ShardEngine*> shards;
      for (std::uint32_t r = 0; r < k; ++r) {
        own.emplace_back(new hyperanf_b200::ShardEngine(
            g, hyperanf_b200::from_reference(c), std::min(n, r * per), std::min(n, (r + 1) * per), k));
        shards.push_back(own.back().get());
      }
      hyperanf_b200::ShardEngine::attach_local(shards);
      hyperanf::NfEngine ref(g, c);
      bool same = true;
      for (std::uint64_t t = 1; t <= n + 1 && same; ++t) {
        for (auto* s : shards) s->compute();
        for (auto* s : shards) s->reduce();  // (a no-op: these shards are not relabelled)
        std::vector<hyperanf_b200::IterationReport> reps;
        for (auto* s : shards) reps.push_back(s->commit());
        const auto a = ref.step();
        const auto& rc = ref.counters();
        for (auto& r : reps) same = same && r.sum == a.sum && r.modified == a.modified;
        same = same && std::vector<std::uint64_t>(rc.data(), rc.data() + rc.word_count()) ==
                           shards.back()->counters();
        if (a.modified == 0) break;
      }
      expect(same, "peer-push shards x" + std::to_string(k));
      for (auto* s : shards) s->detach();
    }
  }
  {  // one engine over several devices (hanf_create_multi), plain and
     // relabelled (interleaved) shards
    hyperanf::EngineConfig c;
    c.bucket_bits = 6;
    c.seed = 9;
    const auto g = hyperanf::gen_uniform_random(4096, 7.0, 23);
    lockstep_multi(g, c, {0, 0}, "multi x2");
    lockstep_multi(g, c, {0, 0, 0}, "multi x3");
    setenv("HANF_RELABEL", "1", 1);
    lockstep_multi(g, c, {0, 0, 0, 0}, "multi x4 relabelled");
    unsetenv("HANF_RELABEL");
    lockstep_multi(hyperanf::gen_uniform_random(100, 3.0, 2), c, {0, 0}, "multi tiny (one shard)");
  }
  {  // source-blocked dense sweeps (hanf_block.cu) forced on small shapes,
     // mapped arc chunks at upload: the reference's bits through the drop-in
    hyperanf::EngineConfig c;
    c.bucket_bits = 6;
    c.seed = 31;
    const auto g = hyperanf::gen_uniform_random(5000, 12.0, 4);
    setenv("HANF_RELABEL", "1", 1);
    setenv("HANF_LAYOUT", "packed", 1);
    setenv("HANF_BLOCK", "1", 1);
    setenv("HANF_BLOCK_S", "6", 1);
    setenv("HANF_BLOCK_T", "7", 1);
    setenv("HANF_BLOCK_SEG", "6", 1);
    setenv("HANF_BLOCK_GROUP", "6", 1);
    setenv("HANF_MAP_CHUNK", "1000", 1);
    {
      auto bc = hyperanf_b200::from_reference(c);
      bc.expected_runs = 32;
      hyperanf_b200::NfEngine probe(g, bc);
      expect(probe.block_stats().first > 0, "blocked engine has items");
    }
    lockstep(g, c, "source-blocked sweeps");
    for (const char* k : {"HANF_RELABEL", "HANF_LAYOUT", "HANF_BLOCK", "HANF_BLOCK_S", "HANF_BLOCK_T",
                          "HANF_BLOCK_SEG", "HANF_BLOCK_GROUP", "HANF_MAP_CHUNK"})
      unsetenv(k);
  }
  std::printf("dropin_test: %zu graphs, %d failures\n", cases.size(), failures);
  return failures == 0 ? 0 : 1;
}
