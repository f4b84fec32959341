// hanf_engine.cu -- host engine behind the C-ABI (include/hanf.h).
//
// Restates the NfEngine surface (engine.hpp:68-298) over device state:
//   - CSR of the node range this engine updates, resident in HBM;
//   - two counter generations (reference packing, hll.hpp:183-240);
//   - two "modified" bitmaps (bit v <-> modified_[v], engine.hpp:287), word
//     i of which is exactly the dirty flag of 64-counter block i (:206);
//   - cached per-counter estimates and per-block sums (engine.hpp:288).
// The union/estimate/reduce kernels live in hanf_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <thread>
#include <new>
#include <string>
#include <vector>

#include "../../include/hanf.h"
#include "hanf_internal.h"

namespace {

thread_local std::string g_last_error;

hanf_status fail(hanf_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

hanf_status cuda_fail(cudaError_t e, const char* what) {
  const hanf_status st =
      e == cudaErrorMemoryAllocation ? HANF_OUT_OF_MEMORY : HANF_CUDA_ERROR;
  return fail(st, std::string(what) + ": " + cudaGetErrorString(e));
}

#define HANF_CUDA(expr)                                   \
  do {                                                    \
    const cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);   \
  } while (0)

// hll.hpp:27-34
double alpha_for_registers(unsigned m) {
  switch (m) {
    case 16: return 0.673;
    case 32: return 0.697;
    case 64: return 0.709;
    default: return 0.7213 / (1.0 + 1.079 / static_cast<double>(m));
  }
}

// SketchParams::make, hll.hpp:43-56 (same messages)
hanf_status make_params(uint32_t b, uint64_t seed, uint32_t r, hanf_sketch_params* p) {
  if (b < 4 || b > 20) return fail(HANF_INVALID_ARGUMENT, "bucket bits must be in [4, 20]");
  if (r < 5 || r > 8) return fail(HANF_INVALID_ARGUMENT, "register width must be in [5, 8]");
  p->bucket_bits = b;
  p->registers = 1u << b;
  p->register_bits = r;
  p->words_per_counter = (p->registers * r + 63) / 64;
  p->alpha = alpha_for_registers(p->registers);
  p->seed = seed;
  return HANF_OK;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  cudaError_t alloc(size_t n) {
    count = n;
    return cudaMalloc(&p, sizeof(T) * (n ? n : 1));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
  }
};

}  // namespace

namespace hanf_host_detail {
void set_error(const std::string& s) { g_last_error = s; }
}  // namespace hanf_host_detail

struct hanf_engine {
  hanf_config cfg{};
  hanf_sketch_params params{};
  uint64_t n = 0;
  uint64_t lo = 0, hi = 0;   // node shard [lo, hi)
  uint64_t blocks = 0;       // ceil(n / 64)
  uint64_t words = 0;        // W
  int device = 0;
  cudaStream_t stream = nullptr;

  DevBuf<uint64_t> cnt[2];
  DevBuf<uint64_t> mod[2];
  DevBuf<double> est;
  DevBuf<double> block_sums;
  DevBuf<double> log_table;
  DevBuf<uint32_t> order;     // light nodes, descending out-degree
  DevBuf<hanf::WarpTask> wtasks;
  DevBuf<uint32_t> tos;       // task-ordered successor ids (see build_tasks)
  uint64_t tos_words = 0;
  uint32_t num_wtasks = 0;
  DevBuf<uint32_t> hub_node;  // per hub chunk
  DevBuf<uint64_t> partials;
  DevBuf<uint32_t> hub_nodes, hub_first, hub_count, chunk_hub, hub_ticket;
  DevBuf<hanf::ReduceOut> reduce;
  DevBuf<double> reduce_sums;
  DevBuf<unsigned long long> reduce_counts;
  uint32_t num_hubs = 0;
  int gather_mode = -1;       // union kernel variant (-1: per-layout default)

  hanf::ReduceOut* h_reduce = nullptr;  // pinned: total + count
  double* h_block_sums = nullptr;       // pinned: exact_sum mode

  int cur = 0;               // index of the current generation
  uint64_t t = 0;            // iteration()
  bool stale_valid = false;  // next[v] may lag where mod[cur] is set
  bool systolic = false;     // systolic_active(), engine.hpp:210-216
  double last_sum = 0.0;     // sum_estimates() of the current generation
  uint64_t last_count = 0;   // modified count of the last step (n after seeding)
  std::vector<double> result_values;      // last run_to_stabilisation
  std::vector<uint64_t> result_modified;
  uint64_t launches = 0;
  // phase timing (hanf_set_timing)
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double union_ms = 0.0, estimate_ms = 0.0, reduce_ms = 0.0;
  uint64_t timed_steps = 0;
  // CUDA graphs of the single-GPU step: [cur][check_mod][stale_valid]
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    uint64_t kernels = 0;
  };
  StepGraph graphs[2][2][2];
  bool use_graphs = true;

  ~hanf_engine() {
    for (auto& a : graphs)
      for (auto& b : a)
        for (auto& c : b)
          if (c.exec) cudaGraphExecDestroy(c.exec);
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
    if (device >= 0) cudaSetDevice(device);
    for (int i = 0; i < 2; ++i) { cnt[i].free(); mod[i].free(); }
    est.free(); block_sums.free(); log_table.free(); order.free();
    wtasks.free(); tos.free(); hub_node.free(); partials.free();
    hub_nodes.free(); hub_first.free(); hub_count.free(); chunk_hub.free(); hub_ticket.free();
    reduce.free(); reduce_sums.free(); reduce_counts.free();
    if (h_reduce) cudaFreeHost(h_reduce);
    if (h_block_sums) cudaFreeHost(h_block_sums);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// Builds the union sweep's work for nodes [lo, hi) (once per graph):
//  - nodes with out-degree > kHubDegree: chunks of kHubChunk arcs, one warp
//    each, plus one finalize warp per node (hub_nodes/first/count);
//  - nodes with out-degree 1..kHubDegree ("light"): sorted by descending
//    degree (stable in id), G = next_pow2(ceil(deg/32)) lanes per node,
//    32/G nodes of one class per warp;
//  - the task-ordered successor array: warp w owns rows [tos/32, +trips) of
//    32 ids; lane (node slot j, sub) reads successor i*G + sub of node j in
//    row i, or the zero row n past the end of the list.
// Degree-0 nodes get no task: their counters never change and both
// generations hold them from seeding.
hanf_status build_tasks(hanf_engine* e, const uint64_t* offsets, const uint32_t* succ) {
  const uint64_t lo = e->lo, hi = e->hi;
  const uint32_t maxd = hanf::kHubDegree;
  const uint32_t zero = static_cast<uint32_t>(e->n);
  std::vector<uint64_t> hist(maxd + 2, 0);
  std::vector<std::pair<uint64_t, uint32_t>> hub_list;
  uint64_t hub_chunks = 0;
  for (uint64_t v = lo; v < hi; ++v) {
    const uint64_t d = offsets[v + 1] - offsets[v];
    if (d == 0) continue;
    if (d > maxd) {
      hub_list.emplace_back(d, static_cast<uint32_t>(v));
      hub_chunks += (d + hanf::kHubChunk - 1) / hanf::kHubChunk;
    } else {
      ++hist[d];
    }
  }
  std::stable_sort(hub_list.begin(), hub_list.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<uint64_t> pos(maxd + 2, 0);
  uint64_t light = 0;
  for (uint64_t d = maxd; d >= 1; --d) {
    pos[d] = light;
    light += hist[d];
  }
  if (light > 0xffffffffull || hub_chunks > 0xffffffffull)
    return fail(HANF_INVALID_ARGUMENT, "too many nodes in one engine shard");
  std::vector<uint32_t> order(light ? light : 1);
  std::vector<uint32_t> ldeg(light ? light : 1);
  for (uint64_t v = lo; v < hi; ++v) {
    const uint64_t d = offsets[v + 1] - offsets[v];
    if (d == 0 || d > maxd) continue;
    ldeg[pos[d]] = static_cast<uint32_t>(d);
    order[pos[d]++] = static_cast<uint32_t>(v);
  }
  auto log2g_of = [](uint64_t d) {
    uint32_t g = 0;
    while ((32ull << g) < d) ++g;  // G = 2^g lanes, each <= 32 arcs
    return g;
  };
  // warp tasks: hub chunks first (longest nodes first), then light classes
  std::vector<hanf::WarpTask> tasks;
  tasks.reserve(hub_chunks + light / 1 + 1);
  std::vector<uint32_t> hub_node(hub_chunks ? hub_chunks : 1);
  std::vector<uint32_t> chunk_hub(hub_chunks ? hub_chunks : 1);
  std::vector<uint64_t> chunk_begin(hub_chunks ? hub_chunks : 1);
  std::vector<uint32_t> hubs_v(hub_list.size() + 1), hubs_first(hub_list.size() + 1),
      hubs_count(hub_list.size() + 1);
  uint64_t tos = 0, c = 0;
  for (size_t h = 0; h < hub_list.size(); ++h) {
    const uint32_t v = hub_list[h].second;
    const uint64_t s = offsets[v], en = offsets[v + 1];
    hubs_v[h] = v;
    hubs_first[h] = static_cast<uint32_t>(c);
    uint32_t k = 0;
    for (uint64_t a = s; a < en; a += hanf::kHubChunk, ++k, ++c) {
      const uint64_t len = std::min<uint64_t>(hanf::kHubChunk, en - a);
      hub_node[c] = v;
      chunk_hub[c] = static_cast<uint32_t>(h);
      chunk_begin[c] = a;
      const uint16_t trips = static_cast<uint16_t>((len + 31) / 32);
      tasks.push_back(hanf::WarpTask{tos, static_cast<uint32_t>(c), trips, 5, 0});
      tos += 32ull * trips;
    }
    hubs_count[h] = k;
  }
  for (uint64_t i = 0; i < light;) {
    const uint32_t lg = log2g_of(ldeg[i]);
    const uint32_t per = 32u >> lg;
    uint64_t cnt = 0;
    while (cnt < per && i + cnt < light && log2g_of(ldeg[i + cnt]) == lg) ++cnt;
    const uint32_t G = 1u << lg;
    const uint16_t trips = static_cast<uint16_t>((ldeg[i] + G - 1) / G);
    tasks.push_back(hanf::WarpTask{tos, static_cast<uint32_t>(i), trips,
                                   static_cast<uint8_t>(lg), static_cast<uint8_t>(cnt)});
    tos += 32ull * trips;
    i += cnt;
  }
  if (tasks.size() > 0x7fffffffull / 32) return fail(HANF_INVALID_ARGUMENT, "task table overflow");
  std::vector<uint32_t> tos_ids;
  try {
    tos_ids.assign(tos ? tos : 1, zero);
  } catch (const std::bad_alloc&) {
    return fail(HANF_OUT_OF_MEMORY, "task-ordered successor array allocation failed");
  }
  auto fill = [&](uint64_t t0, uint64_t t1) {
    for (uint64_t t = t0; t < t1; ++t) {
      const hanf::WarpTask& w = tasks[t];
      uint32_t* dst = tos_ids.data() + w.tos;
      if (w.nodes == 0) {
        const uint64_t a = chunk_begin[w.item];
        const uint64_t len = std::min<uint64_t>(hanf::kHubChunk, offsets[hub_node[w.item] + 1] - a);
        for (uint64_t k = 0; k < len; ++k) dst[k] = succ[a + k];
      } else {
        const uint32_t G = 1u << w.lg;
        for (uint32_t j = 0; j < w.nodes; ++j) {
          const uint32_t v = order[w.item + j];
          const uint64_t s = offsets[v], d = offsets[v + 1] - s;
          for (uint64_t k = 0; k < d; ++k) {
            const uint64_t i = k / G, sub = k % G;
            dst[32 * i + j * G + sub] = succ[s + k];
          }
        }
      }
    }
  };
  {
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const uint64_t T = tasks.size();
    if (T > 4096 && nt > 1) {
      std::vector<std::thread> pool;
      for (unsigned p = 0; p < nt; ++p) pool.emplace_back(fill, T * p / nt, T * (p + 1) / nt);
      for (auto& th : pool) th.join();
    } else {
      fill(0, T);
    }
  }
  e->num_wtasks = static_cast<uint32_t>(tasks.size());
  e->num_hubs = static_cast<uint32_t>(hub_list.size());
  e->tos_words = tos;
  cudaStream_t st = e->stream;
  HANF_CUDA(e->order.alloc(order.size()));
  HANF_CUDA(cudaMemcpyAsync(e->order.p, order.data(), sizeof(uint32_t) * order.size(),
                            cudaMemcpyHostToDevice, st));
  HANF_CUDA(e->wtasks.alloc(tasks.size()));
  if (!tasks.empty())
    HANF_CUDA(cudaMemcpyAsync(e->wtasks.p, tasks.data(), sizeof(hanf::WarpTask) * tasks.size(),
                              cudaMemcpyHostToDevice, st));
  HANF_CUDA(e->tos.alloc(tos_ids.size()));
  HANF_CUDA(cudaMemcpyAsync(e->tos.p, tos_ids.data(), sizeof(uint32_t) * tos_ids.size(),
                            cudaMemcpyHostToDevice, st));
  HANF_CUDA(e->hub_node.alloc(hub_node.size()));
  HANF_CUDA(cudaMemcpyAsync(e->hub_node.p, hub_node.data(), sizeof(uint32_t) * hub_node.size(),
                            cudaMemcpyHostToDevice, st));
  HANF_CUDA(e->partials.alloc(static_cast<size_t>(hub_chunks ? hub_chunks : 1) * e->words));
  HANF_CUDA(e->chunk_hub.alloc(chunk_hub.size()));
  HANF_CUDA(cudaMemcpyAsync(e->chunk_hub.p, chunk_hub.data(), sizeof(uint32_t) * chunk_hub.size(),
                            cudaMemcpyHostToDevice, st));
  HANF_CUDA(e->hub_ticket.alloc(hubs_v.size()));
  HANF_CUDA(cudaMemsetAsync(e->hub_ticket.p, 0, sizeof(uint32_t) * hubs_v.size(), st));
  HANF_CUDA(e->hub_nodes.alloc(hubs_v.size()));
  HANF_CUDA(e->hub_first.alloc(hubs_first.size()));
  HANF_CUDA(e->hub_count.alloc(hubs_count.size()));
  HANF_CUDA(cudaMemcpyAsync(e->hub_nodes.p, hubs_v.data(), sizeof(uint32_t) * hubs_v.size(),
                            cudaMemcpyHostToDevice, st));
  HANF_CUDA(cudaMemcpyAsync(e->hub_first.p, hubs_first.data(), sizeof(uint32_t) * hubs_first.size(),
                            cudaMemcpyHostToDevice, st));
  HANF_CUDA(cudaMemcpyAsync(e->hub_count.p, hubs_count.data(), sizeof(uint32_t) * hubs_count.size(),
                            cudaMemcpyHostToDevice, st));
  // the staging vectors are freed on return: make sure the copies are done
  HANF_CUDA(cudaStreamSynchronize(st));
  return HANF_OK;
}

// Recomputes estimates of the counters flagged in `dirty` (all when null)
// for blocks [b0, b1) of generation g.
hanf_status run_estimates(hanf_engine* e, int g, const uint64_t* dirty, uint64_t b0, uint64_t b1) {
  hanf::EstimateArgs a{};
  a.counters = e->cnt[g].p;
  a.dirty = dirty;
  a.est = e->est.p;
  a.block_sums = e->block_sums.p;
  a.n = e->n;
  a.block_begin = b0;
  a.block_end = b1;
  a.alpha = e->params.alpha;
  a.m = static_cast<double>(e->params.registers);
  a.registers = e->params.registers;
  a.register_bits = e->params.register_bits;
  a.words = e->params.words_per_counter;
  a.log_table = e->log_table.p;
  HANF_CUDA(hanf::launch_estimate(a, e->stream, &e->launches));
  return HANF_OK;
}

// Block sums of [b0, b1) from the cached estimates (when `recompute`), then
// the total of all block sums and the popcount of `bits`; waits for the
// stream.  exact_sum: the total is redone on the host in the reference's
// order (engine.hpp:115-117).
hanf_status finish_enqueue(hanf_engine* e, const uint64_t* bits, bool recompute, uint64_t b0,
                           uint64_t b1, bool in_step) {
  hanf::FinishArgs f{};
  f.est = recompute ? e->est.p : nullptr;
  f.bits = bits;
  f.block_sums = e->block_sums.p;
  f.out = e->reduce.p;
  f.n = e->n;
  f.blocks = e->blocks;
  f.b0 = b0;
  f.b1 = b1;
  if (in_step && e->timing) HANF_CUDA(cudaEventRecord(e->ev[2], e->stream));
  HANF_CUDA(hanf::launch_finish(f, e->stream, &e->launches));
  if (in_step && e->timing) HANF_CUDA(cudaEventRecord(e->ev[3], e->stream));
  HANF_CUDA(cudaMemcpyAsync(e->h_reduce, e->reduce.p, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                            e->stream));
  if (e->cfg.exact_sum)
    HANF_CUDA(cudaMemcpyAsync(e->h_block_sums, e->block_sums.p, sizeof(double) * e->blocks,
                              cudaMemcpyDeviceToHost, e->stream));
  return HANF_OK;
}

hanf_status finish_complete(hanf_engine* e, double* total, uint64_t* count, bool in_step) {
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  if (in_step && e->timing) {
    float a = 0.f, b = 0.f, c = 0.f;
    HANF_CUDA(cudaEventElapsedTime(&a, e->ev[0], e->ev[1]));
    HANF_CUDA(cudaEventElapsedTime(&b, e->ev[1], e->ev[2]));
    HANF_CUDA(cudaEventElapsedTime(&c, e->ev[2], e->ev[3]));
    e->union_ms += a;
    e->estimate_ms += b;
    e->reduce_ms += c;
    ++e->timed_steps;
  }
  if (e->cfg.exact_sum) {
    double s = 0.0;
    for (uint64_t b = 0; b < e->blocks; ++b) s += e->h_block_sums[b];
    *total = s;
  } else {
    *total = e->h_reduce->total;
  }
  *count = e->h_reduce->count;
  return HANF_OK;
}

hanf_status finish(hanf_engine* e, const uint64_t* bits, bool recompute, uint64_t b0, uint64_t b1,
                   double* total, uint64_t* count, bool in_step = false) {
  const hanf_status st = finish_enqueue(e, bits, recompute, b0, b1, in_step);
  if (st != HANF_OK) return st;
  return finish_complete(e, total, count, in_step);
}

// Seeds both generations (every engine seeds all n counters: seeding is a
// pure function of (v, seed), so shards need no exchange) and computes N(0).
hanf_status seed_all(hanf_engine* e) {
  e->cur = 0;
  e->t = 0;
  e->stale_valid = false;
  e->systolic = false;
  HANF_CUDA(hanf::launch_seed(e->cnt[0].p, e->cnt[1].p, e->mod[0].p, e->n, 0, e->n,
                              e->params.bucket_bits, e->params.register_bits,
                              e->params.words_per_counter, e->params.seed, e->stream,
                              &e->launches));
  HANF_CUDA(cudaMemsetAsync(e->mod[1].p, 0, sizeof(uint64_t) * e->blocks, e->stream));
  hanf_status st = run_estimates(e, 0, nullptr, 0, e->blocks);
  if (st != HANF_OK) return st;
  uint64_t count = 0;
  e->last_count = e->n;
  return finish(e, e->mod[0].p, false, 0, 0, &e->last_sum, &count);
}

hanf_status validate_config(const hanf_config* cfg) {
  if (cfg->systolic_threshold <= 0.0 || cfg->systolic_threshold > 1.0)
    return fail(HANF_INVALID_ARGUMENT, "systolic threshold must be in (0, 1]");
  if (cfg->termination == 1 && cfg->eps_inc <= 0.0)
    return fail(HANF_INVALID_ARGUMENT, "threshold termination needs eps_inc > 0");
  if (cfg->termination != 0 && cfg->termination != 1)
    return fail(HANF_INVALID_ARGUMENT, "termination must be 0 (stabilisation) or 1 (threshold)");
  return HANF_OK;
}

hanf_status compute_local(hanf_engine* e) {
  const int g = e->cur, ng = 1 - e->cur;
  const uint64_t w0 = e->lo >> 6, w1 = (e->hi + 63) >> 6;
  HANF_CUDA(cudaMemsetAsync(e->mod[ng].p + w0, 0, sizeof(uint64_t) * (w1 - w0), e->stream));
  if (e->timing) HANF_CUDA(cudaEventRecord(e->ev[0], e->stream));
  hanf::UnionArgs a{};
  a.tos = e->tos.p;
  a.wtasks = e->wtasks.p;
  a.num_wtasks = e->num_wtasks;
  a.zero_row = static_cast<uint32_t>(e->n);
  const bool fused = hanf::fused_estimates(e->params.register_bits, e->params.registers);
  a.est = fused ? e->est.p : nullptr;
  a.ep = hanf::EstimateParams{e->params.alpha, static_cast<double>(e->params.registers),
                              e->params.registers, e->params.register_bits,
                              e->params.words_per_counter, e->log_table.p};
  a.cur = e->cnt[g].p;
  a.next = e->cnt[ng].p;
  a.mod_cur = e->mod[g].p;
  a.mod_next = e->mod[ng].p;
  a.order = e->order.p;
  a.hub_node = e->hub_node.p;
  a.partials = e->partials.p;
  a.chunk_hub = e->chunk_hub.p;
  a.hub_nodes = e->hub_nodes.p;
  a.hub_first = e->hub_first.p;
  a.hub_count = e->hub_count.p;
  a.hub_ticket = e->hub_ticket.p;
  a.words = e->params.words_per_counter;
  // skipping unmodified successors costs a bitmap probe per arc and saves
  // a counter gather per skipped arc: worth it once most counters settled
  a.check_mod = (e->cfg.track_modified && e->t > 0 &&
                 2 * e->last_count < e->n) ? 1 : 0;
  a.stale_valid = e->stale_valid ? 1 : 0;
  HANF_CUDA(hanf::launch_union(a, e->params.register_bits, e->params.registers,
                               e->gather_mode, e->stream, &e->launches));
  if (e->timing) HANF_CUDA(cudaEventRecord(e->ev[1], e->stream));
  const bool sharded = e->lo != 0 || e->hi != e->n;
  if (!fused) {
    const hanf_status st = run_estimates(e, ng, e->mod[ng].p, w0, w1);
    if (st != HANF_OK) return st;
  } else if (sharded) {
    // block sums of this shard now: they are exchanged before commit
    hanf::FinishArgs f{e->est.p, e->mod[ng].p, e->block_sums.p, e->reduce.p, e->n, e->blocks, w0, w1};
    HANF_CUDA(hanf::launch_finish(f, e->stream, &e->launches));
  }
  return HANF_OK;
}

bool commit_recomputes(const hanf_engine* e) {
  // single GPU with fused estimates: the block sums are recomputed in the
  // same launch as the totals
  const bool sharded = e->lo != 0 || e->hi != e->n;
  return !sharded && hanf::fused_estimates(e->params.register_bits, e->params.registers);
}

hanf_status commit_enqueue(hanf_engine* e) {
  const int ng = 1 - e->cur;
  return finish_enqueue(e, e->mod[ng].p, commit_recomputes(e), 0, e->blocks, true);
}

hanf_status commit_complete(hanf_engine* e, hanf_iteration_report* rep) {
  double total = 0.0;
  uint64_t count = 0;
  const hanf_status st = finish_complete(e, &total, &count, true);
  if (st != HANF_OK) return st;
  e->cur = 1 - e->cur;                             // std::swap, engine.hpp:198-200
  e->stale_valid = true;
  if (e->cfg.use_systolic && !e->systolic && count > 0 &&
      static_cast<double>(count) < e->cfg.systolic_threshold * static_cast<double>(e->n))
    e->systolic = true;                            // engine.hpp:211-216
  ++e->t;
  e->last_sum = total;
  e->last_count = count;
  rep->sum = total;
  rep->modified = count;
  return HANF_OK;
}

hanf_status commit(hanf_engine* e, hanf_iteration_report* rep) {
  const hanf_status st = commit_enqueue(e);
  if (st != HANF_OK) return st;
  return commit_complete(e, rep);
}

// One single-GPU step as a CUDA graph (memset + union + finish + read-back),
// captured once per (generation parity, check_mod, stale_valid) and replayed.
hanf_status step_graphed(hanf_engine* e, hanf_iteration_report* rep) {
  const int check = (e->cfg.track_modified && e->t > 0 && 2 * e->last_count < e->n) ? 1 : 0;
  hanf_engine::StepGraph& G = e->graphs[e->cur][check][e->stale_valid ? 1 : 0];
  if (!G.exec) {
    const uint64_t before = e->launches;
    cudaGraph_t graph = nullptr;
    HANF_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    hanf_status st = compute_local(e);
    if (st == HANF_OK) st = commit_enqueue(e);
    const cudaError_t ce = cudaStreamEndCapture(e->stream, &graph);
    if (st != HANF_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
    const cudaError_t ie = cudaGraphInstantiate(&G.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return cuda_fail(ie, "cudaGraphInstantiate");
    G.kernels = e->launches - before;
    e->launches = before;
  }
  HANF_CUDA(cudaGraphLaunch(G.exec, e->stream));
  e->launches += G.kernels;
  return commit_complete(e, rep);
}

}  // namespace

extern "C" {

const char* hanf_last_error(void) { return g_last_error.c_str(); }

hanf_status hanf_config_init(hanf_config* cfg) {
  if (!cfg) return fail(HANF_INVALID_ARGUMENT, "null config");
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->bucket_bits = 7;          // engine.hpp:33-45
  cfg->register_bits = 0;
  cfg->seed = 0;
  cfg->threads = 1;
  cfg->task_size = 0;
  cfg->systolic_threshold = 0.25;
  cfg->termination = 0;
  cfg->eps_inc = 0.0;
  cfg->max_iterations = 0;
  cfg->spill_to_disk = 0;
  cfg->track_modified = 1;
  cfg->use_systolic = 1;
  cfg->device = 0;
  cfg->exact_sum = 1;
  cfg->shard_begin = 0;
  cfg->shard_end = 0;
  return HANF_OK;
}

hanf_status hanf_sketch_params_make(uint32_t b, uint64_t seed, uint32_t r, hanf_sketch_params* out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null output");
  return make_params(b, seed, r, out);
}

hanf_status hanf_create(const hanf_graph_view* g, const hanf_config* cfg_in, hanf_engine** out) {
  if (!g || !cfg_in || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  hanf_status st = validate_config(cfg_in);
  if (st != HANF_OK) return st;
  const uint64_t n = g->n;
  if (n > (1ull << 32)) return fail(HANF_INVALID_ARGUMENT, "graph too large for 32-bit node ids");
  if (n > 0 && !g->offsets) return fail(HANF_INVALID_ARGUMENT, "null offsets");
  if (n > 0 && g->offsets[n] != g->num_arcs)
    return fail(HANF_INVALID_ARGUMENT, "offsets[n] must equal the arc count");
  if (g->num_arcs > 0 && !g->arcs) return fail(HANF_INVALID_ARGUMENT, "null arcs");

  hanf_config cfg = *cfg_in;
  if (cfg.max_iterations == 0) cfg.max_iterations = n + 1;  // engine.hpp:78
  uint32_t r = cfg.register_bits;
  if (r == 0) r = n < (1ull << 32) ? 5 : 6;                  // engine.hpp:79-80
  hanf_sketch_params params;
  st = make_params(cfg.bucket_bits, cfg.seed, r, &params);
  if (st != HANF_OK) return st;
  uint64_t lo = cfg.shard_begin, hi = cfg.shard_end;
  if (lo == 0 && hi == 0) hi = n;
  if (lo > hi || hi > n) return fail(HANF_INVALID_ARGUMENT, "shard range outside [0, n]");
  if ((lo & 63) != 0 || ((hi & 63) != 0 && hi != n))
    return fail(HANF_INVALID_ARGUMENT, "shard boundaries must be multiples of 64 nodes");

  hanf_engine* e = new (std::nothrow) hanf_engine();
  if (!e) return fail(HANF_OUT_OF_MEMORY, "engine allocation failed");
  e->device = cfg.device;
  e->cfg = cfg;
  e->params = params;
  e->n = n;
  e->lo = lo;
  e->hi = hi;
  e->blocks = (n + 63) / 64;
  e->words = params.words_per_counter;

  auto bail = [&](hanf_status s) {
    const std::string msg = g_last_error;
    delete e;
    g_last_error = msg;
    return s;
  };
#define HANF_TRY(expr)                                                  \
  do {                                                                  \
    const cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) return bail(cuda_fail(_e, #expr));           \
  } while (0)

  HANF_TRY(cudaSetDevice(cfg.device));
  HANF_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  // row n is an all-zero counter (the union kernels' padding target); 8
  // extra words keep the 256-bit window loads of the last rows in bounds
  const uint64_t nw = (n + 1) * e->words + 8;
  HANF_TRY(e->cnt[0].alloc(nw));
  HANF_TRY(e->cnt[1].alloc(nw));
  HANF_TRY(cudaMemsetAsync(e->cnt[0].p + n * e->words, 0, sizeof(uint64_t) * (e->words + 8),
                           e->stream));
  HANF_TRY(cudaMemsetAsync(e->cnt[1].p + n * e->words, 0, sizeof(uint64_t) * (e->words + 8),
                           e->stream));
  HANF_TRY(e->mod[0].alloc(e->blocks));
  HANF_TRY(e->mod[1].alloc(e->blocks));
  HANF_TRY(e->est.alloc(n));
  HANF_TRY(e->block_sums.alloc(e->blocks));
  HANF_TRY(e->reduce.alloc(1));
  {
    const uint64_t ctas = (e->blocks + hanf::kFinishThreads - 1) / hanf::kFinishThreads;
    HANF_TRY(e->reduce_sums.alloc(ctas));
    HANF_TRY(e->reduce_counts.alloc(ctas));
    hanf::ReduceOut init{};
    init.partial_sum = e->reduce_sums.p;
    init.partial_count = e->reduce_counts.p;
    HANF_TRY(cudaMemcpy(e->reduce.p, &init, sizeof(init), cudaMemcpyHostToDevice));
  }
  HANF_TRY(cudaMallocHost(&e->h_reduce, sizeof(hanf::ReduceOut)));
  if (cfg.exact_sum)
    HANF_TRY(cudaMallocHost(&e->h_block_sums, sizeof(double) * (e->blocks ? e->blocks : 1)));

  // the CSR itself is not kept on the device: build_tasks lays the shard's
  // successor ids out in task order (the only form the union sweep reads)
  if (n > 0) {
    for (uint64_t v = lo; v < hi; ++v)
      if (g->offsets[v + 1] < g->offsets[v])
        return bail(fail(HANF_INVALID_ARGUMENT, "offsets must be non-decreasing"));
    for (uint64_t i = g->offsets[lo]; i < g->offsets[hi]; ++i)
      if (g->arcs[i] >= n) return bail(fail(HANF_INVALID_ARGUMENT, "arc endpoint out of range"));
  }
  if (const char* gm = std::getenv("HANF_GATHER")) e->gather_mode = std::atoi(gm);
  if (const char* ng = std::getenv("HANF_NO_GRAPHS")) e->use_graphs = std::atoi(ng) == 0;
  if (lo != 0 || hi != n) e->use_graphs = false;  // sharded steps are split around the exchange

  // linear-counting table m*log(m/z), same expression as hll.hpp:139
  {
    const double m = static_cast<double>(params.registers);
    std::vector<double> table(params.registers + 1, 0.0);
    for (uint32_t z = 1; z <= params.registers; ++z)
      table[z] = m * std::log(m / static_cast<double>(z));
    HANF_TRY(e->log_table.alloc(table.size()));
    HANF_TRY(cudaMemcpy(e->log_table.p, table.data(), sizeof(double) * table.size(),
                        cudaMemcpyHostToDevice));
  }
  if (n > 0) {
    st = build_tasks(e, g->offsets, g->arcs);
    if (st != HANF_OK) return bail(st);
    st = seed_all(e);
    if (st != HANF_OK) return bail(st);
  }
#undef HANF_TRY
  *out = e;
  return HANF_OK;
}

void hanf_destroy(hanf_engine* e) { delete e; }

hanf_status hanf_reset(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (e->n == 0) {
    e->t = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  return seed_all(e);
}

hanf_status hanf_sum_estimates(hanf_engine* e, double* sum) {
  if (!e || !sum) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *sum = e->n == 0 ? 0.0 : e->last_sum;
  return HANF_OK;
}

hanf_status hanf_step(hanf_engine* e, hanf_iteration_report* rep) {
  if (!e || !rep) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->n == 0) {                       // engine.hpp:124
    rep->sum = 0.0;
    rep->modified = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  // phase timing needs events between the kernels: run ungraphed then
  if (e->use_graphs && !e->timing) return step_graphed(e, rep);
  hanf_status st = compute_local(e);
  if (st != HANF_OK) return st;
  return commit(e, rep);
}

hanf_status hanf_shard_compute(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (e->n == 0) return HANF_OK;
  HANF_CUDA(cudaSetDevice(e->device));
  return compute_local(e);
}

hanf_status hanf_shard_commit(hanf_engine* e, hanf_iteration_report* rep) {
  if (!e || !rep) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->n == 0) {
    rep->sum = 0.0;
    rep->modified = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  return commit(e, rep);
}

hanf_status hanf_run_to_stabilisation(hanf_engine* e, double* values, uint64_t* modified,
                                      uint64_t capacity, uint64_t* length, double* wall) {
  if (!e || !length) return fail(HANF_INVALID_ARGUMENT, "null argument");
  const auto start = std::chrono::steady_clock::now();
  *length = 0;
  if (wall) *wall = 0.0;
  if (e->n == 0) return HANF_OK;         // engine.hpp:240
  if (e->cfg.termination == 1) {         // engine.hpp:242-250
    std::cerr << "warning: threshold termination can stop before the counters "
                 "stabilise and truncate the neighbourhood function; on graphs "
                 "where large components hang off a narrow path (two cliques "
                 "joined by a one-way path) the resulting cdf and effective "
                 "diameter are arbitrarily wrong. Use stabilisation for "
                 "trustworthy results.\n";
  }
  std::vector<double> vals;
  std::vector<uint64_t> mods;
  vals.push_back(e->last_sum);
  mods.push_back(e->n);
  for (;;) {
    if (vals.size() - 1 >= e->cfg.max_iterations)
      return fail(HANF_GUARD, "engine: iteration cap " + std::to_string(e->cfg.max_iterations) +
                                  " exceeded; pathological input or bug");
    hanf_iteration_report rep;
    const hanf_status st = hanf_step(e, &rep);
    if (st != HANF_OK) return st;
    if (rep.modified == 0) break;
    const double prev = vals.back();
    vals.push_back(rep.sum);
    mods.push_back(rep.modified);
    if (e->cfg.termination == 1 && prev > 0.0) {
      const double rel = (rep.sum - prev) / prev;
      if (rel < e->cfg.eps_inc) break;
    }
  }
  for (size_t t = 1; t < vals.size(); ++t) vals[t] = std::max(vals[t], vals[t - 1]);
  *length = vals.size();
  e->result_values = vals;
  e->result_modified = mods;
  if (wall)
    *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  if (capacity < vals.size())
    return fail(HANF_CAPACITY, "output capacity " + std::to_string(capacity) + " < " +
                                   std::to_string(vals.size()) + " values");
  if (values) std::copy(vals.begin(), vals.end(), values);
  if (modified) std::copy(mods.begin(), mods.end(), modified);
  return HANF_OK;
}

hanf_status hanf_last_result(const hanf_engine* e, double* values, uint64_t* modified,
                             uint64_t capacity, uint64_t* length) {
  if (!e || !length) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *length = e->result_values.size();
  if (capacity < e->result_values.size())
    return fail(HANF_CAPACITY, "output capacity too small");
  if (values) std::copy(e->result_values.begin(), e->result_values.end(), values);
  if (modified) std::copy(e->result_modified.begin(), e->result_modified.end(), modified);
  return HANF_OK;
}

hanf_status hanf_estimate_nf(const hanf_graph_view* g, const hanf_config* cfg, double* values,
                             uint64_t* modified, uint64_t capacity, uint64_t* length,
                             double* wall) {
  const auto start = std::chrono::steady_clock::now();
  hanf_engine* e = nullptr;
  hanf_status st = hanf_create(g, cfg, &e);
  if (st != HANF_OK) return st;
  st = hanf_run_to_stabilisation(e, values, modified, capacity, length, nullptr);
  hanf_destroy(e);
  if (wall)
    *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  return st;
}

hanf_status hanf_read_counters(hanf_engine* e, uint64_t first, uint64_t count, uint64_t* dst) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (first > e->n || count > e->n - first)
    return fail(HANF_OUT_OF_RANGE, "counter index out of range");
  if (count == 0) return HANF_OK;
  if (!dst) return fail(HANF_INVALID_ARGUMENT, "null destination");
  HANF_CUDA(cudaSetDevice(e->device));
  HANF_CUDA(cudaMemcpyAsync(dst, e->cnt[e->cur].p + first * e->words,
                            sizeof(uint64_t) * count * e->words, cudaMemcpyDeviceToHost,
                            e->stream));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  return HANF_OK;
}

hanf_status hanf_params(const hanf_engine* e, hanf_sketch_params* out) {
  if (!e || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *out = e->params;
  return HANF_OK;
}

hanf_status hanf_iteration(const hanf_engine* e, uint64_t* t) {
  if (!e || !t) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *t = e->t;
  return HANF_OK;
}

hanf_status hanf_systolic_active(const hanf_engine* e, int32_t* active) {
  if (!e || !active) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *active = e->systolic ? 1 : 0;
  return HANF_OK;
}

hanf_status hanf_num_nodes(const hanf_engine* e, uint64_t* n) {
  if (!e || !n) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *n = e->n;
  return HANF_OK;
}

hanf_status hanf_stream(const hanf_engine* e, void** stream) {
  if (!e || !stream) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *stream = static_cast<void*>(e->stream);
  return HANF_OK;
}

hanf_status hanf_launch_count(const hanf_engine* e, uint64_t* launches) {
  if (!e || !launches) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *launches = e->launches;
  return HANF_OK;
}

hanf_status hanf_set_timing(hanf_engine* e, int32_t enable) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  HANF_CUDA(cudaSetDevice(e->device));
  for (auto& x : e->ev)
    if (!x) HANF_CUDA(cudaEventCreate(&x));
  e->timing = enable != 0;
  e->union_ms = e->estimate_ms = e->reduce_ms = 0.0;
  e->timed_steps = 0;
  return HANF_OK;
}

hanf_status hanf_timing(const hanf_engine* e, double* union_ms, double* estimate_ms,
                        double* reduce_ms, uint64_t* steps) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (union_ms) *union_ms = e->union_ms;
  if (estimate_ms) *estimate_ms = e->estimate_ms;
  if (reduce_ms) *reduce_ms = e->reduce_ms;
  if (steps) *steps = e->timed_steps;
  return HANF_OK;
}

hanf_status hanf_device_buffers(hanf_engine* e, hanf_buffers* out) {
  if (!e || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  const int ng = 1 - e->cur;
  out->next_counters = e->cnt[ng].p;
  out->next_modified = e->mod[ng].p;
  out->block_sums = e->block_sums.p;
  out->words_per_counter = e->words;
  out->blocks = e->blocks;
  out->shard_begin = e->lo;
  out->shard_end = e->hi;
  return HANF_OK;
}

}  // extern "C"
