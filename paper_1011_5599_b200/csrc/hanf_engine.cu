// hanf_engine.cu -- host engine behind the C-ABI (include/hanf.h).
//
// Restates the NfEngine surface (engine.hpp:68-298) over device state:
//   - the union sweep's work, built on the device from the caller's CSR
//     (hanf_build.cu); the CSR itself is not kept;
//   - two counter generations (reference packing, hll.hpp:183-240) plus an
//     all-zero row n;
//   - two "modified" bitmaps (bit v <-> modified_[v], engine.hpp:287), word
//     i of which is exactly the dirty flag of 64-counter block i (:206);
//   - cached per-counter estimates and per-block sums (engine.hpp:288).
// Device memory comes from the stream-ordered pool (cudaMallocAsync, kept
// cached across engines), pinned host staging from a process-wide cache, so
// creating and destroying engines (estimate_nf) costs no allocator syncs.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/hanf.h"
#include "hanf_internal.h"
#include "hanf_rng.h"

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
cudaError_t palloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1), s);
}
template <class T>
void pfree(T*& p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
  p = nullptr;
}

// Keep freed device memory in the pool (no release at synchronisation).
void configure_pool(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  done.push_back(device);
}

// Process-wide cache of non-blocking streams per device (creating and
// destroying a stream costs ~0.05 ms each, a measurable share of a
// one-shot estimate_nf).  Streams are returned idle (synchronised).
class StreamCache {
 public:
  cudaError_t get(int device, cudaStream_t* s) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      auto& v = free_[device];
      if (!v.empty()) {
        *s = v.back();
        v.pop_back();
        return cudaSuccess;
      }
    }
    return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
  }
  void put(int device, cudaStream_t s) {
    std::lock_guard<std::mutex> lock(mu_);
    free_[device].push_back(s);
  }

 private:
  std::mutex mu_;
  std::map<int, std::vector<cudaStream_t>> free_;
};
StreamCache& streams() {
  static StreamCache* c = new StreamCache();  // never destroyed: outlives static engines
  return *c;
}

// Process-wide cache of pinned host blocks (cudaHostAlloc / cudaFreeHost
// synchronise the device; engines borrow and return blocks instead).
class PinnedCache {
 public:
  void* get(size_t bytes) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      // best fit, but only among blocks at most 2x the request: a 16-byte
      // report must not pin down a 32 MB block
      auto it = free_.lower_bound(bytes);
      if (it != free_.end() && it->first <= 2 * std::max<size_t>(bytes, 4096)) {
        void* p = it->second;
        sizes_[p] = it->first;
        cached_ -= it->first;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    // portable + mapped: finish_kernel writes its report here from any
    // device of the process (blocks are shared by engines on all devices)
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped) !=
        cudaSuccess)
      return nullptr;
    std::lock_guard<std::mutex> lock(mu_);
    sizes_[p] = bytes;
    return p;
  }
  // Returns a block.  Cached page-locked memory is capped: beyond kCap the
  // block is freed (cudaFreeHost synchronises, so only large, rare blocks
  // take that path; small report blocks stay cached).
  void put(void* p) {
    if (!p) return;
    size_t bytes;
    {
      std::lock_guard<std::mutex> lock(mu_);
      bytes = sizes_[p];
      if (cached_ + bytes <= kCap) {
        free_.emplace(bytes, p);
        cached_ += bytes;
        return;
      }
      sizes_.erase(p);
    }
    cudaFreeHost(p);
  }

 private:
  std::mutex mu_;
  static constexpr size_t kCap = size_t(256) << 20;
  std::multimap<size_t, void*> free_;
  std::map<void*, size_t> sizes_;
  size_t cached_ = 0;
};
PinnedCache& pinned() {
  static PinnedCache* c = new PinnedCache();  // never destroyed: outlives engines
  return *c;
}

}  // namespace

namespace hanf_host_detail {
void set_error(const std::string& s) { g_last_error = s; }
}  // namespace hanf_host_detail

namespace l2win {
std::mutex mu;
std::map<int, int> users;
}  // namespace l2win

struct hanf_engine {
  hanf_config cfg{};
  hanf_sketch_params params{};
  uint64_t n = 0;
  uint64_t lo = 0, hi = 0;   // node shard [lo, hi)
  uint64_t blocks = 0;       // ceil(n / 64)
  uint64_t words = 0;        // W
  uint64_t pitch = 0;        // row pitch in words (hanf::row_pitch)
  bool bytes = false;        // byte-layout counter store (hanf_device.cuh ByteLayout)
  int device = 0;
  cudaStream_t stream = nullptr;

  uint64_t* cnt[2] = {nullptr, nullptr};  // (n + 1) * pitch words + 8 (window loads)
  uint64_t* mod[2] = {nullptr, nullptr};  // blocks words
  double* est = nullptr;                  // n, in original id order
  double* block_sums = nullptr;           // blocks
  double* log_table = nullptr;            // m + 1
  uint64_t* partials = nullptr;           // hub chunks * pitch
  hanf::TaskBuild tasks;
  // shard CSR (kept for the worklist step) and its lazily built transpose
  uint64_t* csr_off = nullptr;
  uint32_t* csr_succ = nullptr;
  uint64_t succ_base = 0;
  unsigned long long* tr_off = nullptr;
  uint32_t* tr_succ = nullptr;
  uint64_t shard_arcs = 0;
  uint64_t* sig = nullptr;
  unsigned long long* mod_list = nullptr;
  uint32_t* work = nullptr;
  uint32_t* hub_tasks = nullptr;
  uint32_t* hub_index = nullptr;
  unsigned int* lens = nullptr;
  bool sparse_ok = false;     // worklist step allowed (layout, graph size, HANF_SPARSE)
  uint32_t sparse_after = 8;  // eligible steps before the transpose is built
  bool force_sparse = false;  // HANF_SPARSE=1 (tests)
  uint32_t sparse_wanted_steps = 0;
  hanf::ReduceOut* reduce = nullptr;
  double* reduce_sums = nullptr;
  unsigned long long* reduce_counts = nullptr;
  // locality relabelling (hanf_relabel.cu): the device works on rows;
  // order[row] = original id, perm[id] = row; dirty[g] = original-id
  // bitmaps of changed counters for the block sums (mod[g] is in rows)
  // batched runs (hanf_batch.cu): `batch` runs over the lifted graph, n =
  // n_real * batch rows; run k's seed mix and per-run sums
  uint32_t batch = 1;
  uint64_t n_real = 0;
  uint64_t blocks_real = 0;
  std::vector<uint64_t> batch_seeds;
  uint64_t* batch_mix = nullptr;                  // device [batch]
  double* batch_sums = nullptr;                   // device [batch][blocks_real]
  unsigned long long* batch_counts = nullptr;     // device [batch]
  unsigned long long* h_batch_counts = nullptr;   // pinned [batch]
  double* h_batch_sums[2] = {nullptr, nullptr};   // pinned [batch][blocks_real] per parity
  std::vector<double> batch_last;                 // N(t) of every run
  bool relabel = false;
  // csr_succ holds rows already (mapped through perm chunk by chunk under the
  // upload), still grouped by the caller's node order
  bool succ_rows = false;
  // relabelled shard of a peer-push run: rows interleaved across the
  // shards by degree; estimates are pushed to the peers and every commit
  // recomputes all original-id blocks from the full estimate array
  bool shard_relabel = false;
  // relabelled shards' commit after a step with few changes: the
  // original-id blocks of the changed rows (derived from the published row
  // bitmap) instead of every block; all_dirty_commit = recompute them all
  uint64_t* dirty_derived = nullptr;
  bool all_dirty_commit = true;
  // unsharded relabelled engines, dense sweeps: no original-id dirty bits
  // (one random atomic per changed row); the commit re-sums every block
  bool skip_dirty = false;
  // Relabelled engines: the hot row prefix of the generation a dense sweep
  // gathers is an L2 access-policy window of persisting lines (0: none)
  size_t l2_window = 0;
  size_t l2_setaside = 0;  // the device's maximum persisting set-aside
  bool l2_active = false;  // this engine holds the raised set-aside
  // hanf_shard_reduce ran for this step: the ranks re-summed one slice of
  // the original-id blocks each and published them; commit sums the inbox
  bool reduced = false;
  bool ever_reduced = false;  // (then the local block sums are only current in the slice)
  // relabelled engines keep estimates in row order (writes follow the task
  // order); finish_kernel gathers them through perm for the original-id
  // block sums (scattering them to the original slots instead measured
  // 1.36x slower per R-MAT 26 shard step)
  bool est_rows = false;
  uint32_t* order = nullptr;
  uint32_t* perm = nullptr;
  uint64_t* rl_off = nullptr;  // relabelled offsets until the worklist needs the CSR
  uint64_t* dirty[2] = {nullptr, nullptr};

  hanf::ReduceOut* h_reduce = nullptr;  // pinned (cache): total + count
  double* h_log_stage = nullptr;        // pinned (cache): the log table's upload source
  // pinned (cache), exact_sum mode: one per generation parity, so a step
  // can be launched while the previous step's block sums are summed
  double* h_block_sums[2] = {nullptr, nullptr};

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
  // CUDA graphs of the single-GPU step: [cur][step_mode][stale_valid]
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    uint64_t kernels = 0;
    uint32_t uses = 0;  // captured on the third use: capture + instantiate +
                        // destroy cost more than a one-shot run's few replays
  };
  StepGraph graphs[2][5][2];
  uint64_t* summ = nullptr;   // mode 3 summary bitmap (see create)
  unsigned long long* pack_count = nullptr;  // hanf_shard_pack scratch
  uint32_t summ_shift = 6;
  bool force_summary = false;  // HANF_SUMMARY=1 (tests): every skip sweep is mode 3
  // task-scan step (mode 4): flat TOS scan lists the tasks to sweep
  int task_scan = -1;             // HANF_TASKSCAN: -1 by size, 0 off, 1 forced
  unsigned int* scan_flags = nullptr;
  uint32_t* scan_list = nullptr;
  unsigned int* scan_count = nullptr;
  bool step_pending = false;   // hanf_step_launch done, hanf_step_complete not yet
  uint64_t summ_bits = 0;
  bool use_graphs = true;
  uint32_t* seg_live = nullptr;  // skip sweeps over segmented tasks (TaskBuild::seg_shift)
  // Source-blocked dense sweeps (hanf_block.cu; unsharded relabelled engines
  // with the packed store).  block_mode: 1 = built at create (HANF_BLOCK=1),
  // 2 = at the first re-seed, 0 = never, -1 = by size and use: at create
  // when the caller announced a long multi-run (cfg.expected_runs >=
  // kBlockRuns), else at the re-seed after kBlockDenseSteps dense steps,
  // when the steps saved so far would have repaid the build (ski rental; a
  // one-shot run and a short multi-run never pay for it).  Item k is row
  // n + 1 + k of both counter generations.
  static constexpr uint32_t kBlockRuns = 20;
  static constexpr uint64_t kBlockDenseSteps = 96;  // build ~0.47 s / ~5 ms saved per step
  uint64_t dense_steps = 0;
  int block_mode = -1;
  bool block_ready = false;
  bool block_tried = false;
  uint64_t block_items = 0;
  uint64_t block_arcs = 0;
  hanf::TaskBuild item_tasks;     // first sweep of a dense step: the items
  hanf::TaskBuild block_tasks;    // main sweep: the sources' lists name item rows
  uint64_t* item_partials = nullptr;
  uint64_t* block_partials = nullptr;
  uint64_t* item_bits = nullptr;  // the item sweep's changed-row bitmap (never read)
  // mod[1 - cur] is known to be all zero (seeding, or the last commit's
  // finish_kernel cleared it): the step's memset is skipped
  bool next_bits_clear = false;
  // Sharded engines keep cnt[2], mod[2] and two block-sum inboxes in one
  // IPC-exportable arena (cudaMalloc, not the pool), laid out identically
  // on every rank; attached peers' arenas receive this shard's rows, bitmap
  // words and block sums (peer-push exchange, hanf_shard_attach).
  void* arena = nullptr;
  uint64_t arena_bytes = 0;
  uint64_t arena_off[9] = {};  // cnt0 cnt1 mod0 mod1 inbox0 inbox1 est0 est1 need
  // peer-push needed-rows filter: arena region 8 is this shard's needed-rows
  // bitmap (n bits, from its TOS); need_of holds, peer after peer, the
  // peers' bits over this shard's range (need_words words each), copied at
  // attach.  HANF_PEER_NEED=0 pushes every written row instead.
  uint64_t* need = nullptr;
  uint64_t* need_of = nullptr;
  uint64_t need_words = 0;
  bool need_filter = true;
  uint64_t peer_lo[hanf::kMaxPeers] = {};
  uint64_t peer_hi[hanf::kMaxPeers] = {};
  // relabelled shards: estimates per generation (a fast peer's step t+1
  // must not overwrite what this rank's commit t re-sums); est = est_gen[cur]
  double* est_gen[2] = {nullptr, nullptr};
  double* inbox[2] = {nullptr, nullptr};     // block sums of all shards, per generation
  bool attached = false;
  // hanf_create_multi: this handle owns one attached shard engine per
  // device entry and drives them from one host thread (no kernels of its own)
  std::vector<hanf_engine*> parts;
  std::vector<cudaEvent_t> part_ev;  // per part: its compute (then reduce) is done
  uint32_t npeers = 0;
  uint8_t* peer_base[hanf::kMaxPeers] = {};
  bool peer_ipc[hanf::kMaxPeers] = {};       // opened with cudaIpcOpenMemHandle

  // the persisting set-aside goes with the last windowed engine of the device
  void release_l2() {
    if (!l2_active) return;
    std::lock_guard<std::mutex> lock(l2win::mu);
    if (--l2win::users[device] == 0) {
      cudaCtxResetPersistingL2Cache();
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    }
    l2_active = false;
  }

  void detach_peers() {
    for (uint32_t p = 0; p < npeers; ++p) {
      if (peer_ipc[p] && peer_base[p]) cudaIpcCloseMemHandle(peer_base[p]);
      peer_base[p] = nullptr;
      peer_ipc[p] = false;
    }
    if (need_of) cudaFree(need_of);
    need_of = nullptr;
    npeers = 0;
    attached = false;
  }

  ~hanf_engine() {
    static const bool prof = [] {
      const char* p = std::getenv("HANF_PROFILE");
      return p && p[0] == '1';
    }();
    auto t0 = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
      if (!prof) return;
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[hanf] destroy %-10s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - t0).count());
      t0 = now;
    };
    if (!parts.empty()) {
      // unmap every peer arena before any part frees its own
      for (hanf_engine* p : parts) {
        cudaSetDevice(p->device);
        cudaStreamSynchronize(p->stream);
        p->detach_peers();
      }
      for (size_t i = 0; i < parts.size(); ++i) {
        cudaSetDevice(parts[i]->device);
        if (part_ev[i]) cudaEventDestroy(part_ev[i]);
        delete parts[i];
      }
      parts.clear();
      return;
    }
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    phase("sync");
    if (l2_active) {
      release_l2();
      phase("l2");
    }
    for (auto& a : graphs)
      for (auto& b : a)
        for (auto& c : b)
          if (c.exec) cudaGraphExecDestroy(c.exec);
    phase("graphs");
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
    if (stream) cudaStreamSynchronize(stream);
    detach_peers();
    if (arena) {  // (peers that mapped it were detached by their owners' ranks first)
      cudaFree(arena);
      arena = nullptr;
      cnt[0] = cnt[1] = nullptr;
      mod[0] = mod[1] = nullptr;
      inbox[0] = inbox[1] = nullptr;
      est = nullptr;
      est_gen[0] = est_gen[1] = nullptr;
    }
    if (stream) {
      for (int i = 0; i < 2; ++i) {
        pfree(cnt[i], stream);
        pfree(mod[i], stream);
      }
      pfree(est, stream);
      pfree(block_sums, stream);
      pfree(log_table, stream);
      pfree(partials, stream);
      pfree(reduce, stream);
      pfree(reduce_sums, stream);
      pfree(reduce_counts, stream);
      pfree(csr_off, stream);
      pfree(csr_succ, stream);
      pfree(tr_off, stream);
      pfree(tr_succ, stream);
      pfree(sig, stream);
      pfree(mod_list, stream);
      pfree(work, stream);
      pfree(hub_tasks, stream);
      pfree(scan_flags, stream);
      pfree(scan_list, stream);
      pfree(scan_count, stream);
      pfree(hub_index, stream);
      pfree(batch_mix, stream);
      pfree(batch_sums, stream);
      pfree(batch_counts, stream);
      pfree(summ, stream);
      pfree(pack_count, stream);
      pfree(order, stream);
      pfree(perm, stream);
      pfree(rl_off, stream);
      pfree(dirty[0], stream);
      pfree(dirty[1], stream);
      pfree(lens, stream);
      pfree(seg_live, stream);
      pfree(dirty_derived, stream);
      pfree(item_partials, stream);
      pfree(block_partials, stream);
      pfree(item_bits, stream);
      hanf::free_tasks_device(&item_tasks, stream);
      hanf::free_tasks_device(&block_tasks, stream);
      hanf::free_tasks_device(&tasks, stream);
      if (cudaStreamSynchronize(stream) == cudaSuccess)
        streams().put(device, stream);
      else
        cudaStreamDestroy(stream);
      phase("free");
    }
    pinned().put(h_reduce);
    pinned().put(h_log_stage);
    pinned().put(h_block_sums[0]);
    pinned().put(h_block_sums[1]);
    pinned().put(h_batch_counts);
    pinned().put(h_batch_sums[0]);
    pinned().put(h_batch_sums[1]);
  }
};

namespace {

// Do the graph's ids carry locality?  Median |u - w| over the middle
// successor of up to 4096 evenly spaced nodes, against n/64: the copying
// model's windows (+-2^12 of 2^24) pass, permuted R-MAT / BA ids do not.
bool ids_local(const hanf_graph_view* g) {
  const uint64_t n = g->n;
  std::vector<uint64_t> d;
  d.reserve(4096);
  const uint64_t step = n > 4096 ? n / 4096 : 1;
  for (uint64_t u = 0; u < n && d.size() < 4096; u += step) {
    const uint64_t a = g->offsets[u], b = g->offsets[u + 1];
    if (b <= a || b > g->num_arcs) continue;  // (malformed rows are rejected later)
    const uint64_t w = g->arcs[a + (b - a) / 2];
    d.push_back(w > u ? w - u : u - w);
  }
  if (d.empty()) return true;
  std::nth_element(d.begin(), d.begin() + d.size() / 2, d.end());
  return d[d.size() / 2] < n / 64;
}

// Bitmap of the counters changed into generation g, in original ids (what
// the block sums and the modified count read).
// (relabelled shard engines keep no original-id bitmap: their commit
// recomputes every block, hanf_engine::shard_relabel)
uint64_t* dirty_of(const hanf_engine* e, int g) { return e->dirty[g] ? e->dirty[g] : e->mod[g]; }

// Recomputes estimates of the counters flagged in `dirty` (all when null)
// for blocks [b0, b1) of generation g.
hanf_status run_estimates(hanf_engine* e, int g, const uint64_t* dirty, uint64_t b0, uint64_t b1) {
  hanf::EstimateArgs a{};
  a.counters = e->cnt[g];
  a.bytes = e->bytes ? 1 : 0;
  a.dirty = dirty;
  a.est = e->est;
  a.block_sums = e->block_sums;
  a.n = e->n;
  a.block_begin = b0;
  a.block_end = b1;
  a.alpha = e->params.alpha;
  a.m = static_cast<double>(e->params.registers);
  a.registers = e->params.registers;
  a.register_bits = e->params.register_bits;
  a.pitch = static_cast<uint32_t>(e->pitch);
  a.log_table = e->log_table;
  if (e->est_rows) {  // row order: plain row blocks, no block sums here
    a.row_of = nullptr;
    a.block_sums = nullptr;
  } else {
    a.row_of = e->perm;  // blocks are original ids; counters are read from their rows
  }
  HANF_CUDA(hanf::launch_estimate(a, e->stream, &e->launches));
  return HANF_OK;
}

// Block sums of [b0, b1) from the cached estimates (when `recompute`), then
// the total of all block sums and the popcount of `bits`; waits for the
// stream.  exact_sum: the total is redone on the host in the reference's
// order (engine.hpp:115-117).
hanf_status finish_enqueue(hanf_engine* e, const uint64_t* bits, bool recompute, uint64_t b0,
                           uint64_t b1, bool in_step, bool from_inbox = false) {
  hanf::FinishArgs f{};
  f.est = recompute ? (in_step && e->shard_relabel ? e->est_gen[1 - e->cur] : e->est) : nullptr;
  f.bits = bits;
  // peer-push shards total the inbox the peers published into
  double* sums = in_step && e->attached && (!e->shard_relabel || from_inbox)
                     ? e->inbox[1 - e->cur]
                     : e->block_sums;
  f.block_sums = sums;
  f.out = e->reduce;
  f.n = e->n;
  f.blocks = e->blocks;
  f.b0 = b0;
  f.b1 = b1;
  f.perm = e->est_rows ? e->perm : nullptr;
  // relabelled shards: every block from the (peer-pushed) estimates, or
  // the derived dirty blocks (commit_enqueue)
  f.all_dirty = in_step && ((e->shard_relabel && e->all_dirty_commit) || e->skip_dirty) ? 1 : 0;
  // the last CTA writes total + count into the page-locked report itself
  // (no read-back copy node after the kernel)
  f.host_out = e->h_reduce;
  // exact_sum: every block sum also goes straight to this parity's
  // page-locked copy (the host sums them in the reference's order)
  if (e->cfg.exact_sum) f.host_sums = e->h_block_sums[e->cur];
  // single-GPU steps: the bitmap the next step writes (this step's mod_cur,
  // dead once the sweep has run) is cleared in the same pass.  Shards keep
  // their memset: peers publish into those words during their next step.
  const bool sharded = e->lo != 0 || e->hi != e->n;
  if (in_step && !sharded && e->batch == 1) f.clear = e->mod[e->cur];
  if (in_step && e->timing) HANF_CUDA(cudaEventRecord(e->ev[2], e->stream));
  HANF_CUDA(hanf::launch_finish(f, e->stream, &e->launches));
  if (in_step && e->timing) HANF_CUDA(cudaEventRecord(e->ev[3], e->stream));
  return HANF_OK;
}

// The reference's summation order of the block sums (engine.hpp:115-117),
// from the host copy made by the step launched at generation `parity`.
double host_block_total(const hanf_engine* e, int parity) {
  double s = 0.0;
  const double* b = e->h_block_sums[parity];
  for (uint64_t i = 0; i < e->blocks; ++i) s += b[i];
  return s;
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
    *total = host_block_total(e, e->cur);
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
// Batched runs: per-run dirty flags, counts and block sums of the generation
// `bits` describes, read back into the pinned buffers of parity e->cur.
hanf_status batch_enqueue(hanf_engine* e, const uint64_t* bits) {
  HANF_CUDA(hanf::launch_finish_batch(e->est, bits, e->n_real, e->batch, true, e->batch_sums,
                                      e->batch_counts, e->stream, &e->launches));
  HANF_CUDA(cudaMemcpyAsync(e->h_batch_counts, e->batch_counts,
                            sizeof(unsigned long long) * e->batch, cudaMemcpyDeviceToHost,
                            e->stream));
  HANF_CUDA(cudaMemcpyAsync(e->h_batch_sums[e->cur], e->batch_sums,
                            sizeof(double) * e->batch * e->blocks_real, cudaMemcpyDeviceToHost,
                            e->stream));
  return HANF_OK;
}
// N(t) of every run from the block sums read back at `parity`, summed in
// the reference's order (engine.hpp:115-117); counts[k] when non-null.
void batch_totals(hanf_engine* e, int parity, uint64_t* counts) {
  e->batch_last.assign(e->batch, 0.0);
  for (uint32_t k = 0; k < e->batch; ++k) {
    const double* b = e->h_batch_sums[parity] + static_cast<uint64_t>(k) * e->blocks_real;
    double s = 0.0;
    for (uint64_t i = 0; i < e->blocks_real; ++i) s += b[i];
    e->batch_last[k] = s;
    if (counts) counts[k] = e->h_batch_counts[k];
  }
}

// L2 access-policy window of the dense sweeps (UnionArgs::l2_window_bytes)
// for relabelled (DRAM-resident) engines: the hot row prefix, about 1.5x
// the persisting set-aside (config 5: 54.5 -> 53.7 ms; windows near 128 MiB
// fall off a cliff, 64 ms at 134 MB, so at most 120 MiB).  The set-aside
// itself shrinks the L2 left to everything else (config 2's byte rows in
// the same process: 0.135 -> 0.154 ms), so it is raised while a windowed
// engine lives and dropped with the last one (refcounted per device, at
// create before any upload and at destroy after the final sync, when the
// device is idle).  HANF_L2_WINDOW_MB sets the size, 0 turns windows off.
void choose_l2_window(hanf_engine* e) {
  int maxp = 0, maxw = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, e->device);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, e->device);
  if (maxp <= 0 || maxw <= 0 || !e->relabel || e->bytes) return;
  size_t cap = std::min<size_t>({static_cast<size_t>(maxp) * 3 / 2, static_cast<size_t>(maxw),
                                 120ull << 20});
  if (const char* w = std::getenv("HANF_L2_WINDOW_MB"))
    cap = std::min<size_t>(std::strtoull(w, nullptr, 10) << 20, static_cast<size_t>(maxw));
  e->l2_window = std::min<size_t>(cap, sizeof(uint64_t) * (e->n + 1) * e->pitch);
  e->l2_setaside = static_cast<size_t>(maxp);
}

// Raises the set-aside before the engine's first dense sweep, once its
// create work has drained (the build's random perm lookups lose L2 to the
// set-aside: +65 ms of config 5's create when raised there).  Outside any
// graph capture.
hanf_status activate_l2_window(hanf_engine* e) {
  if (!e->l2_window || e->l2_active) return HANF_OK;
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  std::lock_guard<std::mutex> lock(l2win::mu);
  if (l2win::users[e->device]++ == 0)
    HANF_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, e->l2_setaside));
  e->l2_active = true;
  return HANF_OK;
}

// Item rows (source-blocked dense sweeps) hold maxima of the running
// counters: a new run, or restored counters, start them from zero.
hanf_status clear_item_rows(hanf_engine* e) {
  if (!e->block_ready) return HANF_OK;
  for (int i = 0; i < 2; ++i)
    HANF_CUDA(cudaMemsetAsync(e->cnt[i] + (e->n + 1) * e->pitch, 0,
                              sizeof(uint64_t) * (e->block_items * e->pitch + 8), e->stream));
  return HANF_OK;
}

hanf_status seed_all(hanf_engine* e) {
  // a run starts with no persisting lines from an earlier one (the L2
  // window of §5.1 marks lines of the generation a dense sweep gathers)
  if (e->l2_active) HANF_CUDA(cudaCtxResetPersistingL2Cache());
  e->cur = 0;
  e->t = 0;
  e->stale_valid = false;
  e->systolic = false;
  {
    const hanf_status bs = clear_item_rows(e);
    if (bs != HANF_OK) return bs;
  }
  HANF_CUDA(hanf::launch_seed(e->cnt[0], e->cnt[1], e->mod[0], e->n, 0, e->n,
                              e->params.bucket_bits, e->params.register_bits,
                              e->params.words_per_counter, static_cast<uint32_t>(e->pitch),
                              e->params.seed, e->order, e->batch, e->batch_mix, e->bytes,
                              e->stream, &e->launches));
  HANF_CUDA(cudaMemsetAsync(e->mod[1], 0, sizeof(uint64_t) * e->blocks, e->stream));
  e->next_bits_clear = true;
  if (e->dirty[0]) {  // every counter was seeded: all ones in both id spaces
    HANF_CUDA(cudaMemcpyAsync(e->dirty[0], e->mod[0], sizeof(uint64_t) * e->blocks,
                              cudaMemcpyDeviceToDevice, e->stream));
    HANF_CUDA(cudaMemsetAsync(e->dirty[1], 0, sizeof(uint64_t) * e->blocks, e->stream));
  }
  if (e->shard_relabel) e->est = e->est_gen[0];
  hanf_status st = run_estimates(e, 0, nullptr, 0, e->blocks);
  if (st != HANF_OK) return st;
  if (e->shard_relabel)  // both generations hold the seeded estimates
    HANF_CUDA(cudaMemcpyAsync(e->est_gen[1], e->est_gen[0], sizeof(double) * e->n,
                              cudaMemcpyDeviceToDevice, e->stream));
  uint64_t count = 0;
  e->last_count = e->n;
  if (e->batch > 1) {  // N(0) of every run, in the reference's order
    st = batch_enqueue(e, e->mod[0]);
    if (st != HANF_OK) return st;
    HANF_CUDA(cudaStreamSynchronize(e->stream));
    batch_totals(e, e->cur, nullptr);
    e->last_sum = e->batch_last[0];
    return HANF_OK;
  }
  return finish(e, dirty_of(e, 0), e->est_rows, 0, e->est_rows ? e->blocks : 0, &e->last_sum,
                &count);
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

// Step kind for the current state: 0 dense sweep, 1 dense sweep skipping
// unmodified successors, 2 worklist step (engine.hpp:210-224), 3 skip sweep
// probing the modified-bitmap summary first, 4 task-scan step (the skip
// sweep over the tasks a flat TOS scan lists).  All produce the same bits;
// only the time differs.
bool sparse_wanted(const hanf_engine* e) {
  // segmented engines' skip sweeps visit only the segments in reach of a
  // changed counter: they beat the worklist down to ~n/4096 changed
  // (config 3: 0.43 against 0.65 ms per step between n/4096 and n/128)
  const uint64_t ratio = e->seg_live && !e->force_sparse ? 4096 : 128;
  return e->cfg.track_modified && e->t != 0 && e->sparse_ok && e->stale_valid &&
         ratio * e->last_count < e->n;
}
bool task_scan_wanted(const hanf_engine* e) {
  if (e->task_scan == 0 || e->lo != 0 || e->hi != e->n || e->batch != 1 || e->seg_live ||
      !hanf::fused_estimates(e->params.register_bits, e->params.registers))
    return false;
  if (e->task_scan == 1) return true;
  return e->tasks.tos_words >= (1ull << 28) && 64 * e->last_count < e->n;
}
// Eligible steps before the worklist's transpose is built (ski rental).  It
// costs about as much as 8 skip sweeps of the same arcs
// (profiles/r01_sparse.md) - but where the task-scan step (mode 4) serves
// the tail, an eligible step costs a fraction of a sweep: config 5's three
// tail steps take 20 ms per run by task scan against a 1.03 s transpose
// (profiles/r02_block.md), so such engines wait for 192 eligible steps
// (a 4-seed multirun went from 0.69 to ~0.43 s per run).
uint32_t sparse_after(const hanf_engine* e) {
  if (e->force_sparse || e->sparse_after != 8) return e->sparse_after;
  const bool scan = e->task_scan != 0 && e->lo == 0 && e->hi == e->n && e->batch == 1 &&
                    !e->seg_live && e->tasks.tos_words >= (1ull << 28) &&
                    hanf::fused_estimates(e->params.register_bits, e->params.registers);
  return scan ? 192 : e->sparse_after;
}
int step_mode(const hanf_engine* e) {
  if (!e->cfg.track_modified || e->t == 0) return 0;
  // build the transpose only once that many steps would have used it, so
  // short runs never pay for it
  if (sparse_wanted(e) && (e->tr_off || e->sparse_wanted_steps >= sparse_after(e))) return 2;
  // dense while at least half of the nodes that can change did (nodes of
  // out-degree 0 never do: 60% of config 5's, whose steps 2-4 change 99% of
  // the rest and ran 20% slower as skip sweeps)
  const uint64_t span = e->hi - e->lo;
  const uint64_t active = span ? e->tasks.active_nodes * (e->n / span) : e->n;
  if (2 * e->last_count >= active) return 0;
  // few changed counters on a large unsegmented single engine: list the
  // tasks in reach of a change with one flat TOS scan (mode 4); skip sweeps
  // otherwise walk every task (config 5's tail: ~10 ms for one counter)
  if (task_scan_wanted(e)) return 4;
  // few changed counters: filter the per-arc bitmap probes through the
  // L1-resident summary first (most probes then never reach L2)
  return e->force_summary || 16 * e->last_count < e->summ_bits ? 3 : 1;
}
// Called once at the start of every step, before step_mode.
void note_step(hanf_engine* e) {
  if (sparse_wanted(e) && !e->tr_off) ++e->sparse_wanted_steps;
}

// Builds the transpose and worklist scratch on first use (outside any
// graph capture).
hanf_status ensure_worklist_scratch(hanf_engine* e);

hanf_status ensure_sparse(hanf_engine* e) {
  if (e->tr_off) return HANF_OK;
  cudaStream_t s = e->stream;
  if (e->relabel && e->rl_off) {
    // the transpose is built from the relabelled CSR; the caller-order
    // copy is not needed after that
    uint32_t* succ = nullptr;
    int bad = 0;
    const hanf::RelabelOut r{e->order, e->succ_rows ? nullptr : e->perm, e->rl_off};
    HANF_CUDA(hanf::relabel_arcs_device(e->csr_off, e->csr_succ, e->n, e->shard_arcs, r, s, &succ,
                                        &bad, &e->launches));
    pfree(e->csr_off, s);
    pfree(e->csr_succ, s);
    e->csr_off = e->rl_off;
    e->csr_succ = succ;
    e->rl_off = nullptr;
  }
  HANF_CUDA(hanf::build_transpose_device(e->csr_off, e->csr_succ, e->lo, e->hi, e->succ_base, e->n,
                                         s, &e->tr_off, &e->tr_succ, &e->launches));
  // one signal task per kSignalChunk predecessors of a modified node
  HANF_CUDA(palloc(&e->mod_list, e->n + e->shard_arcs / hanf::kSignalChunk + 64, s));
  return ensure_worklist_scratch(e);
}

// The worklist stages' scratch (step mode 2).
hanf_status ensure_worklist_scratch(hanf_engine* e) {
  cudaStream_t s = e->stream;
  if (!e->sig) {
    HANF_CUDA(palloc(&e->sig, e->blocks, s));
    HANF_CUDA(palloc(&e->work, e->hi - e->lo + 1, s));
    HANF_CUDA(palloc(&e->hub_tasks, e->tasks.num_chunks + 1ull, s));
    HANF_CUDA(hanf::build_hub_index(e->tasks.hub_nodes, e->tasks.num_hubs, e->n, s, &e->hub_index,
                                    &e->launches));
    HANF_CUDA(palloc(&e->lens, 3, s));
  }
  HANF_CUDA(cudaStreamSynchronize(s));
  return HANF_OK;
}

// Peer-push exchange: generation ng of every attached peer.
hanf::PeerRows peer_rows(const hanf_engine* e, int ng) {
  hanf::PeerRows p{};
  p.count = e->attached ? e->npeers : 0;
  p.push_est = e->shard_relabel ? 1u : 0u;
  for (uint32_t i = 0; i < p.count; ++i) {
    p.next[i] = reinterpret_cast<uint64_t*>(e->peer_base[i] + e->arena_off[ng]);
    p.est[i] = reinterpret_cast<double*>(e->peer_base[i] + e->arena_off[6 + ng]);
    p.need[i] = e->need_of ? e->need_of + i * e->need_words : nullptr;
  }
  p.need_base = static_cast<uint32_t>(e->lo >> 6);
  return p;
}

// The sweep's work arrays from another task build (source-blocked sweeps).
void use_tasks(hanf::UnionArgs* a, const hanf::TaskBuild& t, uint64_t* partials) {
  a->tos = t.tos;
  a->wtasks = t.wtasks;
  a->num_wtasks = t.num_wtasks;
  a->order = t.order;
  a->hub_node = t.chunk_node;
  a->partials = partials;
  a->chunk_hub = t.chunk_hub;
  a->hub_nodes = t.hub_nodes;
  a->hub_first = t.hub_first;
  a->hub_count = t.hub_count;
  a->hub_ticket = t.hub_ticket;
}

hanf::UnionArgs union_args(const hanf_engine* e, int g, int ng) {
  hanf::UnionArgs a{};
  a.tos = e->tasks.tos;
  a.wtasks = e->tasks.wtasks;
  a.num_wtasks = e->tasks.num_wtasks;
  a.zero_row = static_cast<uint32_t>(e->n);
  a.row_limit = static_cast<uint32_t>(e->n + 1 + e->block_items);
  const bool fused = hanf::fused_estimates(e->params.register_bits, e->params.registers);
  a.est = fused ? (e->shard_relabel ? e->est_gen[ng] : e->est) : nullptr;
  a.ep = hanf::EstimateParams{e->params.alpha, static_cast<double>(e->params.registers),
                              e->params.registers, e->params.register_bits,
                              e->params.words_per_counter, e->log_table};
  a.cur = e->cnt[g];
  a.next = e->cnt[ng];
  a.mod_cur = e->mod[g];
  a.mod_next = e->mod[ng];
  a.order = e->tasks.order;
  a.hub_node = e->tasks.chunk_node;
  a.partials = e->partials;
  a.chunk_hub = e->tasks.chunk_hub;
  a.hub_nodes = e->tasks.hub_nodes;
  a.hub_first = e->tasks.hub_first;
  a.hub_count = e->tasks.hub_count;
  a.hub_ticket = e->tasks.hub_ticket;
  a.pitch = static_cast<uint32_t>(e->pitch);
  a.stale_valid = e->stale_valid ? 1 : 0;
  a.orig_of = e->order;
  a.est_index = e->est_rows ? nullptr : e->order;
  a.dirty_next = e->skip_dirty ? nullptr : e->dirty[ng];
  a.l2_window_bytes = 0;
  a.peers = peer_rows(e, ng);
  a.bytes = e->bytes ? 1 : 0;
  return a;
}

hanf_status compute_sparse(hanf_engine* e) {
  const int g = e->cur, ng = 1 - e->cur;
  const uint64_t w0 = e->lo >> 6, w1 = (e->hi + 63) >> 6;
  hanf::SparseArgs a{};
  a.off = e->csr_off;
  a.succ = e->csr_succ;
  a.succ_base = e->succ_base;
  a.node_base = e->lo;
  a.cur = e->cnt[g];
  a.next = e->cnt[ng];
  a.mod_cur = e->mod[g];
  a.mod_next = e->mod[ng];
  a.est = e->est;
  a.ep = hanf::EstimateParams{e->params.alpha, static_cast<double>(e->params.registers),
                              e->params.registers, e->params.register_bits,
                              e->params.words_per_counter, e->log_table};
  a.pitch = static_cast<uint32_t>(e->pitch);
  a.tr_off = e->tr_off;
  a.tr_succ = e->tr_succ;
  a.sig = e->sig;
  a.mod_list = e->mod_list;
  a.work = e->work;
  a.hub_tasks = e->hub_tasks;
  a.lens = e->lens;
  a.hub_index = e->hub_index;
  a.orig_of = e->order;
  a.est_index = e->est_rows ? nullptr : e->order;
  a.dirty_next = e->dirty[ng];
  a.hub_first = e->tasks.hub_first;
  a.hub_count = e->tasks.hub_count;
  a.n = e->n;
  a.blocks = e->blocks;
  a.hi = e->hi;
  a.peers = peer_rows(e, ng);
  a.bytes = e->bytes ? 1 : 0;
  HANF_CUDA(hanf::launch_sparse_step(a, w0, w1, e->params.register_bits, e->params.registers,
                                     e->stream, &e->launches));
  if (e->tasks.num_chunks) {
    // worklist hubs: their chunk tasks through the dense kernel (skipping
    // unmodified successors), chunk partials folded by the usual ticket
    hanf::UnionArgs u = union_args(e, g, ng);
    u.check_mod = 1;
    u.task_list = e->hub_tasks;
    u.task_count = e->lens + 2;
    u.num_wtasks = e->tasks.num_chunks;
    HANF_CUDA(hanf::launch_union(u, e->params.register_bits, e->params.registers, e->stream,
                                 &e->launches));
  }
  return HANF_OK;
}

hanf_status compute_shard(hanf_engine* e);

// A sharded compute, then (peer-push exchange) the shard's bitmap words and
// block sums into every peer's arena and the local inbox.
hanf_status compute_local(hanf_engine* e) {
  const hanf_status st = compute_shard(e);
  if (st != HANF_OK || !e->attached) return st;
  const int ng = 1 - e->cur;
  hanf::PublishArgs p{};
  p.mod_next = e->mod[ng];
  p.block_sums = e->shard_relabel ? nullptr : e->block_sums;  // (commit redoes all blocks)
  p.w0 = e->lo >> 6;
  p.w1 = (e->hi + 63) >> 6;
  p.count = e->npeers;
  for (uint32_t i = 0; i < e->npeers; ++i) {
    p.peer_mod[i] = reinterpret_cast<uint64_t*>(e->peer_base[i] + e->arena_off[2 + ng]);
    p.peer_sums[i] = reinterpret_cast<double*>(e->peer_base[i] + e->arena_off[4 + ng]);
  }
  p.peer_sums[e->npeers] = e->inbox[ng];
  HANF_CUDA(hanf::launch_publish(p, e->stream, &e->launches));
  return HANF_OK;
}

hanf_status compute_shard(hanf_engine* e) {
  const int g = e->cur, ng = 1 - e->cur;
  if (e->shard_relabel && !e->attached)
    return fail(HANF_INVALID_ARGUMENT,
                "relabelled shard engines exchange through hanf_shard_attach (peer-push)");
  const uint64_t w0 = e->lo >> 6, w1 = (e->hi + 63) >> 6;
  // the next bitmap is zero already where the previous commit cleared it
  // (single-GPU engines, finish_kernel `clear`); shards clear their words
  if (!e->next_bits_clear)
    HANF_CUDA(cudaMemsetAsync(e->mod[ng] + w0, 0, sizeof(uint64_t) * (w1 - w0), e->stream));
  e->next_bits_clear = false;
  // Dense sweeps of unsharded relabelled engines change nearly every block:
  // rather than an original-id dirty bit per changed row (a random atomic
  // each), the commit re-sums every block through perm (same sums, same
  // order).  The count comes from the row bitmap (popcount is permutation-
  // invariant).
  e->skip_dirty = e->dirty[ng] && e->est_rows && e->lo == 0 && e->hi == e->n && step_mode(e) == 0;
  if (e->dirty[ng] && !e->skip_dirty)  // unsharded relabelling: the whole original-id bitmap
    HANF_CUDA(cudaMemsetAsync(e->dirty[ng], 0, sizeof(uint64_t) * e->blocks, e->stream));
  if (e->timing) HANF_CUDA(cudaEventRecord(e->ev[0], e->stream));
  if (step_mode(e) == 2 && e->tr_off) {
    const hanf_status st = compute_sparse(e);
    if (st != HANF_OK) return st;
    if (e->timing) HANF_CUDA(cudaEventRecord(e->ev[1], e->stream));
    if (e->lo != 0 || e->hi != e->n) {
      hanf::FinishArgs f{e->est, e->mod[ng], e->block_sums, e->reduce, e->n, e->blocks, w0, w1};
      HANF_CUDA(hanf::launch_finish(f, e->stream, &e->launches));
    }
    return HANF_OK;
  }
  hanf::UnionArgs a = union_args(e, g, ng);
  // skipping unmodified successors costs a bitmap probe per arc and saves
  // a counter gather per skipped arc: worth it once most counters settled
  const int mode = step_mode(e);
  a.check_mod = mode != 0 ? 1 : 0;
  if (mode != 4 && e->l2_active) a.l2_window_bytes = e->l2_window;  // (skip sweeps too: -2%)
  if (mode != 0 && e->seg_live) {
    HANF_CUDA(hanf::launch_segment_live(e->mod[g], e->tasks.seg_min, e->tasks.seg_max,
                                        e->tasks.num_segs, e->seg_live, e->stream, &e->launches));
    a.seg_live = e->seg_live;
    a.seg_shift = e->tasks.seg_shift;
  }
  if (mode == 3 || mode == 4) {
    HANF_CUDA(hanf::launch_summary(e->mod[g], e->blocks + 1, e->summ_shift, e->summ_bits, e->summ,
                                   e->stream, &e->launches));
    a.summ = e->summ;
    a.summ_shift = e->summ_shift;
    a.summ_words = static_cast<uint32_t>((e->summ_bits + 63) / 64);
  }
  if (mode == 4) {
    // the tasks in reach of a change, from one pass over the TOS
    HANF_CUDA(cudaMemsetAsync(e->scan_flags, 0, sizeof(unsigned int) * e->tasks.num_wtasks, e->stream));
    HANF_CUDA(cudaMemsetAsync(e->scan_count, 0, sizeof(unsigned int), e->stream));
    hanf::TaskScanArgs ts{};
    ts.tos = e->tasks.tos;
    ts.tos_words = e->tasks.tos_words;
    ts.wtasks = e->tasks.wtasks;
    ts.num_wtasks = e->tasks.num_wtasks;
    ts.zero_row = static_cast<uint32_t>(e->n);
    ts.mod_cur = e->mod[g];
    ts.summ = e->summ;
    ts.summ_shift = e->summ_shift;
    ts.summ_words = a.summ_words;
    ts.chunk_hub = e->tasks.chunk_hub;
    ts.hub_first = e->tasks.hub_first;
    ts.hub_count = e->tasks.hub_count;
    ts.flags = e->scan_flags;
    ts.list = e->scan_list;
    ts.count = e->scan_count;
    HANF_CUDA(hanf::launch_task_scan(ts, e->stream, &e->launches));
    a.task_list = e->scan_list;
    a.task_count = e->scan_count;
  }
  const bool fused = a.est != nullptr;
  if (mode == 0 && e->block_ready) {
    // Source-blocked dense sweep (hanf_block.cu).  First the items: their
    // rows n + 1 + k of the current generation take the maximum of the
    // item's cold successors (counters only grow, so the row's value of two
    // steps ago folds in harmlessly: the sweep's own-row rule applies to it
    // unchanged).  Then the main sweep over the lists that name the items.
    hanf::UnionArgs v = a;
    use_tasks(&v, e->item_tasks, e->item_partials);
    v.next = e->cnt[g];
    v.mod_next = e->item_bits;
    v.est = nullptr;
    v.dirty_next = nullptr;
    v.orig_of = nullptr;
    v.est_index = nullptr;
    v.stale_valid = 0;
    v.l2_window_bytes = 0;
    HANF_CUDA(hanf::launch_union(v, e->params.register_bits, e->params.registers, e->stream,
                                 &e->launches));
    use_tasks(&a, e->block_tasks, e->block_partials);
  }
  HANF_CUDA(hanf::launch_union(a, e->params.register_bits, e->params.registers, e->stream,
                               &e->launches));
  if (mode == 4)  // rows changed last step that no listed task rewrote
    HANF_CUDA(hanf::launch_stale_fixup(e->mod[g], e->mod[ng], e->n, static_cast<uint32_t>(e->pitch),
                                       e->cnt[g], e->cnt[ng], e->stream, &e->launches));
  if (e->timing) HANF_CUDA(cudaEventRecord(e->ev[1], e->stream));
  const bool sharded = e->lo != 0 || e->hi != e->n;
  if (!fused) {
    // (row-order estimates: the row bitmap says which rows to redo)
    const hanf_status st = run_estimates(e, ng, e->est_rows ? e->mod[ng] : dirty_of(e, ng), w0, w1);
    if (st != HANF_OK) return st;
  } else if (sharded && !e->shard_relabel) {
    // block sums of this shard now: they are exchanged before commit
    hanf::FinishArgs f{e->est, e->mod[ng], e->block_sums, e->reduce, e->n, e->blocks, w0, w1};
    HANF_CUDA(hanf::launch_finish(f, e->stream, &e->launches));
  }
  return HANF_OK;
}

// Source-blocked dense sweeps (hanf_block.cu): which engines, and with
// which shape.  Config 5 (measured, profiles/r02_block.md): the 2^21 rows of
// highest out-degree as sources, rows past the first 2^21 (84 MB, what L2
// keeps anyway) as cold, segments of 2^21 rows, item tasks grouped 2^18
// items at a time (a flat optimum: 48.7 ms; 49.2-50.2 with 2^20 sources or
// 2^20-row segments, 52 with 2^19- or 2^23-row segments).  HANF_BLOCK_S /
// _T / _SEG / _GROUP give the log2 of each (tests force small ones).
bool block_eligible(const hanf_engine* e) {
  return e->relabel && !e->shard_relabel && e->lo == 0 && e->hi == e->n && e->batch == 1 &&
         !e->bytes && !e->seg_live && !e->arena && e->parts.empty() && e->n >= 64 &&
         e->csr_off && e->csr_succ &&
         hanf::fused_estimates(e->params.register_bits, e->params.registers);
}
bool block_wanted_by_size(const hanf_engine* e) {
  // counters far beyond L2 and enough arcs that the hot sources' lists
  // split into items of several arcs (config 5; config 4's BA graph has no
  // such sources)
  return e->tasks.tos_words >= (1ull << 31) && (e->n + 1) * e->pitch * 8 >= (4ull << 30);
}

hanf_status build_block(hanf_engine* e) {
  e->block_tried = true;
  if (!block_eligible(e)) return HANF_OK;
  cudaStream_t s = e->stream;
  const uint64_t n = e->n;
  auto env_log2 = [](const char* name, uint32_t dflt) {
    const char* v = std::getenv(name);
    return v && v[0] ? static_cast<uint32_t>(std::atoi(v)) : dflt;
  };
  // rows of ~84 MB stay in L2 on their own; as many per segment
  uint32_t cold_log2 = 0;
  while ((2ull << cold_log2) * e->pitch * 8 <= (84ull << 20)) ++cold_log2;
  cold_log2 = env_log2("HANF_BLOCK_T", cold_log2);
  const uint32_t src_log2 = env_log2("HANF_BLOCK_S", cold_log2);
  const uint32_t seg_log2 = env_log2("HANF_BLOCK_SEG", cold_log2);
  const uint32_t group_log2 = env_log2("HANF_BLOCK_GROUP", 18);
  if (cold_log2 > 31 || src_log2 > 31 || seg_log2 > 31 || group_log2 < 6 || group_log2 > 31)
    return fail(HANF_INVALID_ARGUMENT, "HANF_BLOCK_* out of range");
  const uint64_t cold = std::min<uint64_t>(1ull << cold_log2, n);
  const uint64_t sources = std::min<uint64_t>(1ull << src_log2, n);
  if (cold >= n || ((n - cold - 1) >> seg_log2) + 1 > 4096) return HANF_OK;  // nothing to block
  HANF_CUDA(cudaStreamSynchronize(s));
  // the engine's CSR: the caller's arcs through perm, or (once the worklist
  // step relabelled them) rows already
  const bool caller_ids = e->rl_off != nullptr;
  const hanf::CsrView base{e->csr_off, 0, e->csr_succ, e->succ_base,
                           caller_ids ? e->order : nullptr,
                           caller_ids && !e->succ_rows ? e->perm : nullptr, n};
  hanf::BlockSplit b;
  cudaError_t ce = hanf::build_block_split(base, n, sources, cold, seg_log2, s, &b, &e->launches);
  // (too many rows for 32-bit ids, or no room for the build's scratch: the
  // plain sweep stays)
  auto soft = [](cudaError_t x) {
    if (x != cudaErrorInvalidValue && x != cudaErrorMemoryAllocation) return false;
    cudaGetLastError();
    return true;
  };
  if (soft(ce)) return HANF_OK;
  HANF_CUDA(ce);
  // items of one arc save nothing (forced modes keep them: tests)
  if (b.items == 0 || (e->block_mode == -1 && b.blocked_arcs < 2 * b.items)) {
    hanf::free_block_split(&b, s);
    return HANF_OK;
  }
  auto drop = [&](hanf_status st) {
    hanf::free_block_split(&b, s);
    hanf::free_tasks_device(&e->item_tasks, s);
    hanf::free_tasks_device(&e->block_tasks, s);
    pfree(e->item_partials, s);
    pfree(e->block_partials, s);
    pfree(e->item_bits, s);
    return st;
  };
  int bad = 0;
  const hanf::CsrView items{b.item_off, n + 1, b.item_succ, 0, nullptr, nullptr, n};
  ce = hanf::build_tasks_device(items, n + 1, n + 1 + b.items, n, group_log2, s, nullptr,
                                &e->item_tasks, &bad, &e->launches, false, false);
  if (ce != cudaSuccess || bad)
    return drop(ce == cudaSuccess || soft(ce) ? HANF_OK : cuda_fail(ce, "item task build"));
  hanf::CsrView main = base;
  main.ovr_off = b.src_off;
  main.ovr_succ = b.src_succ;
  main.ovr_rows = sources;
  ce = hanf::build_tasks_device(main, 0, n, n, 32, s, nullptr, &e->block_tasks, &bad, &e->launches,
                                false, true, n + 1 + b.items);
  if (ce != cudaSuccess || bad)
    return drop(ce == cudaSuccess || soft(ce) ? HANF_OK : cuda_fail(ce, "blocked task build"));
  const uint64_t items_n = b.items;
  e->block_arcs = b.blocked_arcs;
  hanf::free_block_split(&b, s);
  cudaError_t ae = palloc(&e->item_partials, static_cast<size_t>(e->item_tasks.num_chunks) * e->pitch, s);
  if (ae == cudaSuccess)
    ae = palloc(&e->block_partials, static_cast<size_t>(e->block_tasks.num_chunks) * e->pitch, s);
  if (ae == cudaSuccess) ae = palloc(&e->item_bits, (n + 1 + items_n + 63) / 64 + 1, s);
  if (ae == cudaSuccess)
    ae = cudaMemsetAsync(e->item_bits, 0, sizeof(uint64_t) * ((n + 1 + items_n + 63) / 64 + 1), s);
  if (ae != cudaSuccess) return drop(soft(ae) ? HANF_OK : cuda_fail(ae, "blocked sweep scratch"));
  // both generations grow by the item rows (the caller re-seeds next)
  uint64_t* grown[2] = {nullptr, nullptr};
  const uint64_t nw = (n + 1 + items_n) * e->pitch + 8;
  HANF_CUDA(cudaStreamSynchronize(s));
  {
    size_t free_b = 0, total_b = 0;  // room for both grown generations once the old ones are freed?
    HANF_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t extra = 2 * 8 * items_n * e->pitch;
    if (free_b < extra + (1ull << 30)) return drop(HANF_OK);
  }
  for (int i = 0; i < 2 && ae == cudaSuccess; ++i) {
    pfree(e->cnt[i], s);  // (freed first: two grown generations may not fit beside the old ones)
    ae = palloc(&grown[i], nw, s);
    if (ae == cudaSuccess) {
      e->cnt[i] = grown[i];
      ae = cudaMemsetAsync(e->cnt[i] + n * e->pitch, 0,
                           sizeof(uint64_t) * ((1 + items_n) * e->pitch + 8), s);
    }
  }
  if (ae != cudaSuccess) {
    // without counter arrays the engine cannot go on
    drop(HANF_OK);
    return cuda_fail(ae, "source-blocked sweep allocation");
  }
  for (auto& x : e->graphs)  // captured steps hold the old arrays
    for (auto& y : x)
      for (auto& z : y) {
        if (z.exec) cudaGraphExecDestroy(z.exec);
        z = hanf_engine::StepGraph{};
      }
  // the item sweep wants the whole L2 for its segment: no persisting
  // set-aside for the hot prefix (config 5: 49.2 ms without, 50.4 with)
  e->release_l2();
  e->l2_window = 0;
  e->block_items = items_n;
  e->block_ready = true;
  HANF_CUDA(cudaStreamSynchronize(s));
  return HANF_OK;
}

bool commit_recomputes(const hanf_engine* e) {
  // single GPU with fused estimates: the block sums are recomputed in the
  // same launch as the totals
  const bool sharded = e->lo != 0 || e->hi != e->n;
  return e->est_rows || e->shard_relabel ||
         (!sharded && hanf::fused_estimates(e->params.register_bits, e->params.registers));
}

// Relabelled shards: the bitmap of original-id blocks to re-sum for the
// step being committed.  Few changes in the previous step (the tail): the
// blocks of this step's changed rows (a scatter over the row bitmap);
// dense steps: every block (all_dirty_commit; n estimate gathers anyway).
hanf_status relabel_dirty(hanf_engine* e, const uint64_t** bits) {
  const int ng = 1 - e->cur;
  e->all_dirty_commit = 64 * e->last_count >= e->n || (e->ever_reduced && !e->reduced);
  *bits = e->mod[ng];  // (all_dirty: only the count is read from it)
  if (!e->all_dirty_commit) {
    if (!e->dirty_derived) HANF_CUDA(palloc(&e->dirty_derived, e->blocks, e->stream));
    HANF_CUDA(cudaMemsetAsync(e->dirty_derived, 0, sizeof(uint64_t) * e->blocks, e->stream));
    HANF_CUDA(hanf::launch_derive_dirty(e->mod[ng], e->order, e->blocks, e->n, e->dirty_derived,
                                        e->stream, &e->launches));
    *bits = e->dirty_derived;
  }
  return HANF_OK;
}

hanf_status commit_enqueue(hanf_engine* e) {
  const int ng = 1 - e->cur;
  if (e->batch > 1) return batch_enqueue(e, e->mod[ng]);
  if (e->shard_relabel && e->reduced) {
    // the block sums are in the inbox (hanf_shard_reduce): totals only
    e->reduced = false;
    e->all_dirty_commit = false;
    return finish_enqueue(e, e->mod[ng], false, 0, e->blocks, true, true);
  }
  if (e->shard_relabel) {
    const uint64_t* bits = nullptr;
    const hanf_status rs = relabel_dirty(e, &bits);
    if (rs != HANF_OK) return rs;
    return finish_enqueue(e, bits, true, 0, e->blocks, true);
  }
  const hanf_status st = finish_enqueue(e, e->skip_dirty ? e->mod[ng] : dirty_of(e, ng),
                                        commit_recomputes(e), 0, e->blocks, true);
  // (finish_kernel cleared mod[cur], the next step's mod_next)
  if (st == HANF_OK && e->lo == 0 && e->hi == e->n) e->next_bits_clear = true;
  return st;
}

// Generation swap and the per-step state after a step's modified count is
// known (engine.hpp:198-216); N(t) is set by the caller.
void advance_state(hanf_engine* e, uint64_t count) {
  e->cur = 1 - e->cur;                             // std::swap, engine.hpp:198-200
  if (e->shard_relabel) e->est = e->est_gen[e->cur];
  e->stale_valid = true;
  if (e->cfg.use_systolic && !e->systolic && count > 0 &&
      static_cast<double>(count) < e->cfg.systolic_threshold * static_cast<double>(e->n))
    e->systolic = true;                            // engine.hpp:211-216
  ++e->t;
  e->last_count = count;
}

hanf_status commit_complete(hanf_engine* e, hanf_iteration_report* rep) {
  double total = 0.0;
  uint64_t count = 0;
  const hanf_status st = finish_complete(e, &total, &count, true);
  if (st != HANF_OK) return st;
  e->cur = 1 - e->cur;                             // std::swap, engine.hpp:198-200
  if (e->shard_relabel) e->est = e->est_gen[e->cur];
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
// Enqueues one whole single-GPU step (compute + finish + read-backs) on the
// engine stream, graphed when allowed; the caller completes it.
hanf_status step_enqueue(hanf_engine* e) {
  note_step(e);
  const int mode = step_mode(e);
  if (mode == 2) {
    const hanf_status st = ensure_sparse(e);
    if (st != HANF_OK) return st;
  }
  if (mode == 0) {
    ++e->dense_steps;
    const hanf_status st = activate_l2_window(e);
    if (st != HANF_OK) return st;
  }
  if (mode == 4 && !e->scan_list) {  // (allocated outside any graph capture)
    HANF_CUDA(palloc(&e->scan_flags, e->tasks.num_wtasks, e->stream));
    HANF_CUDA(palloc(&e->scan_list, e->tasks.num_wtasks, e->stream));
    HANF_CUDA(palloc(&e->scan_count, 1, e->stream));
  }
  if (!e->use_graphs || e->timing) {
    const hanf_status st = compute_local(e);
    if (st != HANF_OK) return st;
    return commit_enqueue(e);
  }
  hanf_engine::StepGraph& G = e->graphs[e->cur][mode][e->stale_valid ? 1 : 0];
  if (!G.exec && ++G.uses < 3) {
    hanf_status st = compute_local(e);
    if (st != HANF_OK) return st;
    return commit_enqueue(e);
  }
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
  return HANF_OK;
}

}  // namespace

namespace {  // hanf_create_multi's step (defined with it, below)
hanf_status multi_step_enqueue(hanf_engine* e);
hanf_status multi_step_complete(hanf_engine* e, hanf_iteration_report* rep);
hanf_status multi_reset(hanf_engine* e, const uint64_t* seed);
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
  cfg->shard_count = 0;
  cfg->expected_runs = 0;
  return HANF_OK;
}

hanf_status hanf_sketch_params_make(uint32_t b, uint64_t seed, uint32_t r, hanf_sketch_params* out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null output");
  return make_params(b, seed, r, out);
}

// One engine; K > 1 = K batched runs over the lifted graph (hanf_batch.cu).
static hanf_status create_engine(const hanf_graph_view* g, const hanf_config* cfg_in,
                                 const uint64_t* seeds, uint32_t K, hanf_engine** out) {
  if (!g || !cfg_in || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  const auto t_create0 = std::chrono::steady_clock::now();
  hanf_status st = validate_config(cfg_in);
  if (st != HANF_OK) return st;
  const uint64_t n_real = g->n;
  if (n_real > (1ull << 32) - 1)
    return fail(HANF_INVALID_ARGUMENT, "graph too large for 32-bit node ids");
  if (n_real > 0 && !g->offsets) return fail(HANF_INVALID_ARGUMENT, "null offsets");
  if (n_real > 0 && (g->offsets[0] != 0 || g->offsets[n_real] != g->num_arcs))
    return fail(HANF_INVALID_ARGUMENT, "offsets must run from 0 to the arc count");
  if (g->num_arcs > 0 && !g->arcs) return fail(HANF_INVALID_ARGUMENT, "null arcs");
  if (K > 1) {
    if (K != 2 && K != 4 && K != 8)
      return fail(HANF_INVALID_ARGUMENT, "batched runs: runs must be 2, 4 or 8");
    if (n_real * K > (1ull << 32) - 1)
      return fail(HANF_INVALID_ARGUMENT, "batched runs: n * runs must stay below 2^32");
    if (cfg_in->shard_begin != 0 || cfg_in->shard_end != 0)
      return fail(HANF_INVALID_ARGUMENT, "batched runs cannot be sharded");
  }
  const uint64_t n = n_real * K;  // rows (= nodes unless batched)

  hanf_config cfg = *cfg_in;
  if (cfg.max_iterations == 0) cfg.max_iterations = n_real + 1;  // engine.hpp:78
  uint32_t r = cfg.register_bits;
  if (r == 0) r = n_real < (1ull << 32) ? 5 : 6;                 // engine.hpp:79-80
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
  e->batch = K;
  e->n_real = n_real;
  e->blocks_real = (n_real + 63) / 64;
  if (K > 1) e->batch_seeds.assign(seeds, seeds + K);
  e->lo = lo;
  e->hi = hi;
  e->blocks = (n + 63) / 64;
  e->words = params.words_per_counter;
  // Counter store.  Byte registers (hanf_device.cuh ByteLayout: one coalesced
  // access and 3 instructions per 4 registers per gathered counter) when a
  // generation of byte rows stays L2-resident; DRAM-resident arrays keep
  // the reference packing, whose 1.6x smaller footprint wins there (config
  // 2: 0.139 vs 0.177 ms per union sweep; configs 3/4/5: 7.08/13.5/66.5 vs
  // 5.92/12.97/58.8 ms, profiles/r02_byte_layout.md).  HANF_LAYOUT=bytes or
  // packed forces either; both give the same bits.
  const bool bytes_ok = hanf::byte_layout_supported(params.register_bits, params.registers);
  e->bytes = bytes_ok && (n + 1) * params.registers <= (96ull << 20);
  if (const char* ly = std::getenv("HANF_LAYOUT")) {
    if (std::strcmp(ly, "packed") == 0) e->bytes = false;
    if (std::strcmp(ly, "bytes") == 0) e->bytes = bytes_ok;
  }
  e->pitch = hanf::row_pitch(params.register_bits, params.registers, params.words_per_counter,
                             e->bytes);
  if (const char* fs = std::getenv("HANF_SUMMARY")) e->force_summary = fs[0] == '1';
  if (const char* bl = std::getenv("HANF_BLOCK"))
    e->block_mode = bl[0] == '1' ? 1 : (bl[0] == '0' ? 0 : (bl[0] == '2' ? 2 : -1));
  if (const char* pn = std::getenv("HANF_PEER_NEED")) e->need_filter = pn[0] != '0';
  if (const char* ts = std::getenv("HANF_TASKSCAN")) e->task_scan = ts[0] == '1' ? 1 : (ts[0] == '0' ? 0 : -1);
  if (const char* ng = std::getenv("HANF_NO_GRAPHS")) e->use_graphs = std::atoi(ng) == 0;
  if (lo != 0 || hi != n) e->use_graphs = false;  // sharded steps are split around the exchange
  // Worklist step (HANF_SPARSE=0 disables): taken once fewer than n/128
  // counters changed (the measured crossover on the long-diameter copying
  // graph) on graphs with >= 2^22 arcs (below that one dense launch costs
  // less than the worklist's launches); profiles/r01_sparse.md.
  e->sparse_ok = hanf::sparse_supported(params.register_bits, params.registers) &&
                 hanf::fused_estimates(params.register_bits, params.registers) &&
                 n > 0 && (K > 1 ? g->num_arcs * K : g->offsets[hi] - g->offsets[lo]) >= (1ull << 22);
  {
    const char* sp = std::getenv("HANF_SPARSE");
    if (sp && sp[0] == '0') e->sparse_ok = false;
    if (sp && sp[0] == '1') {  // tests: force it on every supported graph, at once
      e->sparse_ok = hanf::sparse_supported(params.register_bits, params.registers) &&
                     hanf::fused_estimates(params.register_bits, params.registers);
      e->sparse_after = 1;
      e->force_sparse = true;
    }
  }

  // Locality relabelling (hanf_relabel.cu), unsharded engines only:
  // HANF_RELABEL=1/0 forces it; by default graphs whose counters do not fit
  // in L2 (one generation > 64 MB) and whose ids show no locality (sampled
  // successors far from their source) are renumbered by degree.
  // Shards relabel only for the peer-push exchange (cfg.shard_count), with
  // equal shards and fused estimates: rows are interleaved across the
  // shards in degree order (relabel_order_device `ways`).
  const bool shard_cfg = lo != 0 || hi != n;
  const bool shard_may_relabel =
      shard_cfg && cfg.shard_count > 1 && n > 0 && n % (64ull * cfg.shard_count) == 0 &&
      hi - lo == n / cfg.shard_count && lo % (n / cfg.shard_count) == 0 &&
      hanf::fused_estimates(params.register_bits, params.registers);
  if ((!shard_cfg || shard_may_relabel) && n > 0 && K == 1) {
    const char* rl = std::getenv("HANF_RELABEL");
    if (rl && (rl[0] == '0' || rl[0] == '1'))
      e->relabel = rl[0] == '1';
    else
      e->relabel = (n + 1) * e->words * 8 > (64ull << 20) && !ids_local(g);
    e->est_rows = e->relabel;
    if (shard_cfg && e->relabel) {
      // estimates stay in row order and are pushed to the peers with their
      // rows; the commit gathers them through perm for every block
      e->shard_relabel = true;
      e->sparse_ok = false;  // (the worklist needs a row-space CSR of the shard)
    }
  }
  cudaStream_t helper = nullptr;  // upload stream: idle before any buffer is freed
  auto bail = [&](hanf_status s) {
    const std::string msg = g_last_error;
    if (helper) cudaStreamSynchronize(helper);
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
  configure_pool(cfg.device);
  if (!(lo != 0 || hi != n) && K == 1) choose_l2_window(e);
  HANF_TRY(streams().get(cfg.device, &e->stream));
  cudaStream_t s = e->stream;
  // row n is an all-zero counter (the union kernels' padding target); 8
  // extra words keep the 256-bit window loads of the last rows in bounds
  const uint64_t nw = (n + 1) * e->pitch + 8;
  const bool sharded = lo != 0 || hi != n;
  if (sharded) {
    // the exchange arena (see hanf_engine::arena): same offsets on every rank
    auto al = [](uint64_t bytes) { return (bytes + 255) & ~255ull; };
    const uint64_t sizes[9] = {nw * 8, nw * 8, (e->blocks + 1) * 8, (e->blocks + 1) * 8,
                               e->blocks * 8, e->blocks * 8, n * 8,
                               e->shard_relabel ? n * 8 : 8, (e->blocks + 1) * 8};
    uint64_t off = 0;
    for (int i = 0; i < 9; ++i) {
      e->arena_off[i] = off;
      off += al(sizes[i] ? sizes[i] : 8);
    }
    e->arena_bytes = off;
    HANF_TRY(cudaMalloc(&e->arena, off));
    uint8_t* base = static_cast<uint8_t*>(e->arena);
    for (int i = 0; i < 2; ++i) {
      e->cnt[i] = reinterpret_cast<uint64_t*>(base + e->arena_off[i]);
      e->mod[i] = reinterpret_cast<uint64_t*>(base + e->arena_off[2 + i]);
      e->inbox[i] = reinterpret_cast<double*>(base + e->arena_off[4 + i]);
    }
    e->est = reinterpret_cast<double*>(base + e->arena_off[6]);
    e->need = reinterpret_cast<uint64_t*>(base + e->arena_off[8]);
    if (e->shard_relabel) {
      e->est_gen[0] = e->est;
      e->est_gen[1] = reinterpret_cast<double*>(base + e->arena_off[7]);
    }
  } else {
    HANF_TRY(palloc(&e->cnt[0], nw, s));
    HANF_TRY(palloc(&e->cnt[1], nw, s));
  }
  HANF_TRY(cudaMemsetAsync(e->cnt[0] + n * e->pitch, 0, sizeof(uint64_t) * (e->pitch + 8), s));
  HANF_TRY(cudaMemsetAsync(e->cnt[1] + n * e->pitch, 0, sizeof(uint64_t) * (e->pitch + 8), s));
  // one extra word: the padding row n (TOS padding, skipped arcs) is probed
  // like any successor and must read as unmodified
  if (!sharded) {
    HANF_TRY(palloc(&e->mod[0], e->blocks + 1, s));
    HANF_TRY(palloc(&e->mod[1], e->blocks + 1, s));
  }
  HANF_TRY(cudaMemsetAsync(e->mod[0] + e->blocks, 0, sizeof(uint64_t), s));
  HANF_TRY(cudaMemsetAsync(e->mod[1] + e->blocks, 0, sizeof(uint64_t), s));
  // summary of the modified bitmap for the skip sweep's tail (mode 3): one
  // bit per 2^summ_shift rows, at most 32 KB; the mode-3 sweep runs as a
  // persistent grid whose CTAs stage it in shared memory once (a random
  // probe then costs a bank, not an L1 line)
  e->summ_shift = 6;
  while (((n + 1) >> e->summ_shift) >= (1ull << 18)) ++e->summ_shift;
  e->summ_bits = ((n + 1) >> e->summ_shift) + 1;
  HANF_TRY(palloc(&e->summ, (e->summ_bits + 63) / 64, s));
  if (!sharded) HANF_TRY(palloc(&e->est, n, s));
  HANF_TRY(palloc(&e->block_sums, e->blocks, s));
  {
    const uint64_t ctas = (e->blocks + hanf::kFinishBlocks - 1) / hanf::kFinishBlocks;
    HANF_TRY(palloc(&e->reduce, 1, s));
    HANF_TRY(palloc(&e->reduce_sums, ctas, s));
    HANF_TRY(palloc(&e->reduce_counts, ctas, s));
    // staged in the engine's page-locked report block: an async copy, no
    // synchronisation (the first finish_kernel writes that block afterwards)
    e->h_reduce = static_cast<hanf::ReduceOut*>(pinned().get(sizeof(hanf::ReduceOut)));
    if (!e->h_reduce) return bail(fail(HANF_OUT_OF_MEMORY, "pinned host allocation failed"));
    hanf::ReduceOut init{};
    init.partial_sum = e->reduce_sums;
    init.partial_count = e->reduce_counts;
    *e->h_reduce = init;
    HANF_TRY(cudaMemcpyAsync(e->reduce, e->h_reduce, sizeof(init), cudaMemcpyHostToDevice, s));
  }
  if (cfg.exact_sum) {
    for (auto& hb : e->h_block_sums) {
      hb = static_cast<double*>(pinned().get(sizeof(double) * (e->blocks ? e->blocks : 1)));
      if (!hb) return bail(fail(HANF_OUT_OF_MEMORY, "pinned host allocation failed"));
    }
  }
  // linear-counting table m*log(m/z), same expression as hll.hpp:139
  {
    const double m = static_cast<double>(params.registers);
    const size_t entries = params.registers + 1;
    e->h_log_stage = static_cast<double*>(pinned().get(sizeof(double) * entries));
    if (!e->h_log_stage) return bail(fail(HANF_OUT_OF_MEMORY, "pinned host allocation failed"));
    e->h_log_stage[0] = 0.0;
    for (uint32_t z = 1; z <= params.registers; ++z)
      e->h_log_stage[z] = m * std::log(m / static_cast<double>(z));
    HANF_TRY(palloc(&e->log_table, entries, s));
    HANF_TRY(cudaMemcpyAsync(e->log_table, e->h_log_stage, sizeof(double) * entries,
                             cudaMemcpyHostToDevice, s));  // (staging kept while the engine lives)
  }
  // HANF_PROFILE=1: print the create phases (synchronising between them)
  static const bool prof = [] {
    const char* p = std::getenv("HANF_PROFILE");
    return p && p[0] == '1';
  }();
  auto t_prev = t_create0;
  auto phase = [&](const char* what) {
    if (!prof) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hanf] create %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_prev).count());
    t_prev = now;
  };
  phase("alloc");
  if (n > 0) {
    // the shard's CSR goes to the device to build the tasks (it is laid
    // out again in task order there) and stays for the worklist step
    // (batched runs upload the caller's graph and lift it on the device)
    // (relabelled shards: the whole graph - their rows are spread over it)
    const bool whole = K > 1 || e->shard_relabel;
    const uint64_t up_lo = whole ? 0 : lo, up_hi = whole ? n_real : hi;
    // Segments (HANF_SEGMENTS=0/1 forces): graphs whose ids carry locality
    // (the copying model's windows) group their tasks by node segment, so
    // a warp's nodes are id-neighbours and late skip sweeps visit only the
    // segments near the changed counters (profiles/r01_segments.md).
    // (Two ways to hide step 1 or the TOS fill under the arcs upload were
    // measured and removed: profiles/r01_pipeline.md.)
    uint32_t seg_shift = 32;
    bool seg_skip = false;
    {
      uint32_t bits = 0;
      while ((1ull << bits) < n) ++bits;
      const char* sg = std::getenv("HANF_SEGMENTS");
      const bool want = sg && (sg[0] == '0' || sg[0] == '1')
                            ? sg[0] == '1'
                            : K == 1 && !e->relabel && n >= (1ull << 20) && ids_local(g);
      if (want && K == 1 && !e->relabel && n > 1) {
        // 4096 segments (config 3: 2^12 nodes each; the +-2^12 windows make
        // finer ones no better)
        seg_shift = bits > 18 ? bits - 12 : 6;
        if (const char* sh = std::getenv("HANF_SEG_SHIFT")) seg_shift = std::atoi(sh);
        if (seg_shift < 6) seg_shift = 6;
        seg_skip = true;
      }
    }
    uint64_t a0 = g->offsets[up_lo], a1 = g->offsets[up_hi];
    uint64_t* d_off = nullptr;
    uint32_t* d_succ = nullptr;
    HANF_TRY(palloc(&d_off, up_hi - up_lo + 1, s));
    e->csr_off = d_off;  // owned by the engine at once: error paths free them
    HANF_TRY(palloc(&d_succ, a1 - a0, s));
    e->csr_succ = d_succ;
    // offsets first on the engine stream; the arcs follow on a helper
    // stream while the engine stream seeds and sorts by degree (only the
    // TOS fill waits for them)
    cudaStream_t s2 = nullptr;
    HANF_TRY(streams().get(cfg.device, &s2));
    helper = s2;
    cudaEvent_t ev_off = nullptr, ev_arcs = nullptr;
    struct UploadGuard {  // the helper streams are idle again before anything is freed
      int dev;
      cudaStream_t st;
      cudaEvent_t a, b;
      std::vector<cudaEvent_t> chunks;
      cudaStream_t st3 = nullptr;  // maps uploaded arc chunks to rows (relabelled engines)
      ~UploadGuard() {
        for (cudaStream_t x : {st, st3}) {
          if (!x) continue;
          if (cudaStreamSynchronize(x) == cudaSuccess)
            streams().put(dev, x);
          else
            cudaStreamDestroy(x);
        }
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
        for (cudaEvent_t c : chunks) cudaEventDestroy(c);
      }
    } guard{cfg.device, s2, nullptr, nullptr, {}};
    HANF_TRY(cudaEventCreateWithFlags(&ev_off, cudaEventDisableTiming));
    guard.a = ev_off;
    HANF_TRY(cudaEventCreateWithFlags(&ev_arcs, cudaEventDisableTiming));
    guard.b = ev_arcs;
    HANF_TRY(cudaMemcpyAsync(d_off, g->offsets + up_lo, sizeof(uint64_t) * (up_hi - up_lo + 1),
                             cudaMemcpyHostToDevice, s));
    HANF_TRY(cudaEventRecord(ev_off, s));
    HANF_TRY(cudaStreamWaitEvent(s2, ev_off, 0));
    // Large relabelled engines upload the arcs in chunks: each chunk's ids
    // are mapped to rows through perm as soon as it has landed (on a third
    // stream, under the rest of the upload), so the TOS fill that follows the
    // upload streams row ids instead of gathering perm for every arc
    // (config 5: ~4.3 G random 4-byte gathers off the critical path).
    const uint64_t up_arcs = a1 - a0;
    // (HANF_MAP_CHUNK=arcs forces it with that chunk size, 0 turns it off: tests)
    bool map_chunks = e->relabel && K == 1 && up_arcs >= (1ull << 26);
    uint64_t chunk_arcs = std::max<uint64_t>(up_arcs / 32 + 1, 1ull << 24);
    if (const char* mc = std::getenv("HANF_MAP_CHUNK")) {
      const uint64_t forced = std::strtoull(mc, nullptr, 10);
      map_chunks = e->relabel && K == 1 && forced > 0 && up_arcs > 0;
      chunk_arcs = std::max<uint64_t>(forced, up_arcs / 1024 + 1);
    }
    if (!map_chunks) chunk_arcs = up_arcs;
    for (uint64_t c0 = 0; c0 < up_arcs; c0 += chunk_arcs) {
      const uint64_t len = std::min(chunk_arcs, up_arcs - c0);
      HANF_TRY(cudaMemcpyAsync(d_succ + c0, g->arcs + a0 + c0, sizeof(uint32_t) * len,
                               cudaMemcpyHostToDevice, s2));
      if (map_chunks) {
        cudaEvent_t ce = nullptr;
        HANF_TRY(cudaEventCreateWithFlags(&ce, cudaEventDisableTiming));
        guard.chunks.push_back(ce);
        HANF_TRY(cudaEventRecord(ce, s2));
      }
    }
    HANF_TRY(cudaEventRecord(ev_arcs, s2));
    phase("offsets");
    if (K > 1) {
      HANF_TRY(cudaStreamWaitEvent(s, ev_arcs, 0));
      uint64_t* voff = nullptr;
      uint32_t* vsucc = nullptr;
      const cudaError_t le = hanf::lift_graph_device(d_off, d_succ, n_real, a1 - a0, K, s, &voff,
                                                     &vsucc, &e->launches);
      cudaFreeAsync(d_off, s);
      cudaFreeAsync(d_succ, s);
      d_off = voff;
      d_succ = vsucc;
      e->csr_off = d_off;  // owned by the engine from here on
      e->csr_succ = d_succ;
      HANF_TRY(le);
      a1 = (a1 - a0) * K;
      a0 = 0;
      // run k's seed mix (item_hash, hash.hpp:20-22) and the per-run sums
      std::vector<uint64_t> mix(K);
      for (uint32_t k = 0; k < K; ++k) mix[k] = hanf_rng::mix64(seeds[k] ^ 0x9e3779b97f4a7c15ULL);
      HANF_TRY(palloc(&e->batch_mix, K, s));
      HANF_TRY(cudaMemcpyAsync(e->batch_mix, mix.data(), sizeof(uint64_t) * K,
                               cudaMemcpyHostToDevice, s));
      HANF_TRY(palloc(&e->batch_sums, static_cast<uint64_t>(K) * e->blocks_real, s));
      HANF_TRY(palloc(&e->batch_counts, K, s));
      HANF_TRY(cudaStreamSynchronize(s));  // `mix` is a stack object
      e->h_batch_counts = static_cast<unsigned long long*>(
          pinned().get(sizeof(unsigned long long) * K));
      for (auto& hb : e->h_batch_sums)
        hb = static_cast<double*>(pinned().get(sizeof(double) * K * (e->blocks_real + 1)));
      if (!e->h_batch_counts || !e->h_batch_sums[0] || !e->h_batch_sums[1])
        return bail(fail(HANF_OUT_OF_MEMORY, "pinned host allocation failed"));
      phase("lift");
    }
    if (e->relabel) {
      // renumber rows by out-degree (offsets only: overlaps the arcs upload)
      hanf::RelabelOut r;
      const cudaError_t re = hanf::relabel_order_device(
          d_off, n, e->shard_relabel ? cfg.shard_count : 1, static_cast<uint32_t>(e->pitch), s, &r,
          &e->launches);
      e->order = r.order;
      e->perm = r.perm;
      e->rl_off = r.off;
      HANF_TRY(re);
      if (e->shard_relabel) pfree(e->rl_off, s);  // (no worklist step: no relabelled CSR)
      if (!e->shard_relabel) {
        HANF_TRY(palloc(&e->dirty[0], e->blocks, s));
        HANF_TRY(palloc(&e->dirty[1], e->blocks, s));
      }
      phase("relabel");
    }
    cudaEvent_t succ_ready = ev_arcs;
    if (map_chunks) {
      // perm is complete on `s` here; chunk c is mapped once it has landed
      cudaStream_t s3 = nullptr;
      HANF_TRY(streams().get(cfg.device, &s3));
      guard.st3 = s3;
      cudaEvent_t ev_perm = nullptr, ev_mapped = nullptr;
      HANF_TRY(cudaEventCreateWithFlags(&ev_perm, cudaEventDisableTiming));
      guard.chunks.push_back(ev_perm);
      HANF_TRY(cudaEventCreateWithFlags(&ev_mapped, cudaEventDisableTiming));
      guard.chunks.push_back(ev_mapped);
      const size_t nchunks = guard.chunks.size() - 2;
      HANF_TRY(cudaEventRecord(ev_perm, s));
      HANF_TRY(cudaStreamWaitEvent(s3, ev_perm, 0));
      for (size_t c = 0; c < nchunks; ++c) {
        const uint64_t c0 = c * chunk_arcs;
        HANF_TRY(cudaStreamWaitEvent(s3, guard.chunks[c], 0));
        HANF_TRY(hanf::launch_map_ids(d_succ + c0, std::min(chunk_arcs, up_arcs - c0), e->perm, n,
                                      s3, &e->launches));
      }
      HANF_TRY(cudaEventRecord(ev_mapped, s3));
      succ_ready = ev_mapped;
      e->succ_rows = true;
    }
    st = seed_all(e);
    if (st != HANF_OK) return bail(st);
    phase("seed");
    int bad = 0;
    // relabelled: row v's successors are the caller's arcs of order[v],
    // through perm unless the upload mapped them already
    const hanf::CsrView view{d_off, up_lo, d_succ, a0, e->order, e->succ_rows ? nullptr : e->perm, n};
    const cudaError_t be = hanf::build_tasks_device(view, lo, hi, n, seg_shift, s, succ_ready,
                                                    &e->tasks, &bad, &e->launches, seg_skip,
                                                    !seg_skip);
    // (also on the build's error paths) frees on `s` come after the upload
    HANF_TRY(cudaStreamWaitEvent(s, ev_arcs, 0));
    HANF_TRY(cudaStreamWaitEvent(s, succ_ready, 0));
    e->csr_off = d_off;
    e->csr_succ = d_succ;
    e->succ_base = a0;
    e->shard_arcs = a1 - a0;
    if (be == cudaErrorInvalidValue)
      return bail(fail(HANF_INVALID_ARGUMENT, "too many nodes or tasks in one engine shard"));
    HANF_TRY(be);
    if (bad)
      return bail(fail(HANF_INVALID_ARGUMENT,
                       "arc endpoint out of range or offsets not non-decreasing"));
    if (e->shard_relabel) {  // the TOS holds the shard's rows; no worklist CSR is kept
      pfree(e->csr_off, s);
      pfree(e->csr_succ, s);
    }
    if (seg_skip && e->tasks.seg_shift < 32)
      HANF_TRY(palloc(&e->seg_live, e->tasks.num_segs, s));
    phase("build");
    HANF_TRY(palloc(&e->partials, static_cast<size_t>(e->tasks.num_chunks) * e->pitch, s));
    if (e->need)  // peer-push filter: the rows this shard gathers (read at the peers' attach)
      HANF_TRY(hanf::launch_need_rows(e->tasks.tos, e->tasks.tos_words, n, e->need, s,
                                      &e->launches));
    // HANF_BLOCK=1, or a long multi-run announced on a large engine: blocked
    // dense sweeps from the first run on
    if (e->block_mode == 1 || (e->block_mode == -1 && cfg.expected_runs >= hanf_engine::kBlockRuns &&
                               block_wanted_by_size(e))) {
      st = build_block(e);
      if (st == HANF_OK && e->block_ready) st = seed_all(e);  // (the counter arrays moved)
      if (st != HANF_OK) return bail(st);
    }
  }
#undef HANF_TRY
  *out = e;
  return HANF_OK;
}

hanf_status hanf_create(const hanf_graph_view* g, const hanf_config* cfg, hanf_engine** out) {
  return create_engine(g, cfg, nullptr, 1, out);
}

hanf_status hanf_create_batch(const hanf_graph_view* g, const hanf_config* cfg,
                              const uint64_t* seeds, uint32_t runs, hanf_engine** out) {
  if (!seeds) return fail(HANF_INVALID_ARGUMENT, "null seeds");
  if (runs == 1) {
    if (!cfg) return fail(HANF_INVALID_ARGUMENT, "null argument");
    hanf_config c = *cfg;
    c.seed = seeds[0];
    return create_engine(g, &c, nullptr, 1, out);
  }
  return create_engine(g, cfg, seeds, runs, out);
}

// run_to_stabilisation of every batched run (engine.hpp:233-275 per run):
// pipelined like the single run; run k's series ends at its own
// stabilisation (a run whose counters stopped changing never changes again).
hanf_status hanf_run_batch(hanf_engine* e, double* values, uint64_t* modified, uint64_t cap,
                           uint64_t* lengths) {
  if (!e || !lengths) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->batch < 2) return fail(HANF_INVALID_ARGUMENT, "not a batched engine (hanf_create_batch)");
  const uint32_t K = e->batch;
  std::vector<std::vector<double>> vals(K);
  std::vector<std::vector<uint64_t>> mods(K);
  for (uint32_t k = 0; k < K; ++k) {
    vals[k].push_back(e->batch_last.empty() ? 0.0 : e->batch_last[k]);
    mods[k].push_back(e->n_real);
  }
  if (e->n > 0) {
    HANF_CUDA(cudaSetDevice(e->device));
    hanf_status st = step_enqueue(e);
    if (st != HANF_OK) return st;
    std::vector<uint64_t> counts(K);
    uint64_t steps = 0;
    for (;;) {
      const int parity = e->cur;
      HANF_CUDA(cudaStreamSynchronize(e->stream));
      uint64_t total = 0;
      for (uint32_t k = 0; k < K; ++k) total += (counts[k] = e->h_batch_counts[k]);
      advance_state(e, total);
      ++steps;
      if (total == 0) break;
      const bool capped = steps >= e->cfg.max_iterations;
      if (!capped) {
        st = step_enqueue(e);
        if (st != HANF_OK) return st;
      }
      batch_totals(e, parity, nullptr);
      for (uint32_t k = 0; k < K; ++k)
        if (counts[k]) {
          vals[k].push_back(e->batch_last[k]);
          mods[k].push_back(counts[k]);
        }
      if (capped)
        return fail(HANF_GUARD, "engine: iteration cap " + std::to_string(e->cfg.max_iterations) +
                                    " exceeded; pathological input or bug");
    }
  }
  bool fits = true;
  for (uint32_t k = 0; k < K; ++k) {
    auto& v = vals[k];
    for (size_t t = 1; t < v.size(); ++t) v[t] = std::max(v[t], v[t - 1]);
    lengths[k] = v.size();
    fits = fits && v.size() <= cap;
  }
  if (!fits) return fail(HANF_CAPACITY, "output capacity too small for a batched run");
  for (uint32_t k = 0; k < K; ++k) {
    if (values) std::copy(vals[k].begin(), vals[k].end(), values + static_cast<uint64_t>(k) * cap);
    if (modified) std::copy(mods[k].begin(), mods[k].end(), modified + static_cast<uint64_t>(k) * cap);
  }
  return HANF_OK;
}

void hanf_destroy(hanf_engine* e) { delete e; }


hanf_status hanf_reset(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (!e->parts.empty()) return multi_reset(e, nullptr);
  if (e->n == 0) {
    e->t = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  if (!e->block_tried &&
      (e->block_mode == 2 || (e->block_mode == -1 && block_wanted_by_size(e) &&
                              e->dense_steps >= hanf_engine::kBlockDenseSteps))) {
    // a long-lived engine: the blocked dense sweeps pay for their build from here on
    const hanf_status bs = build_block(e);
    if (bs != HANF_OK) return bs;
  }
  return seed_all(e);
}

namespace {
void put_le(std::string& out, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>(v >> (8 * i)));
}
uint64_t get_le(const unsigned char* p, int bytes) {
  uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}
}  // namespace

// hll.hpp:275-286: "HCA1", u32 b, u32 r, u64 n, u64 seed, n*W words (LE).
hanf_status hanf_save_counters(hanf_engine* e, const char* path) {
  if (!e || !path) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "batched engine: no single counter array");
  std::vector<uint64_t> words(e->n * e->words);
  if (e->n) {
    const hanf_status st = hanf_read_counters(e, 0, e->n, words.data());
    if (st != HANF_OK) return st;
  }
  std::string head("HCA1");
  put_le(head, e->params.bucket_bits, 4);
  put_le(head, e->params.register_bits, 4);
  put_le(head, e->n, 8);
  put_le(head, e->params.seed, 8);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return fail(HANF_IO_ERROR, std::string("cannot open for writing: ") + path);
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  if (ok && !words.empty())  // little-endian host: raw words are the LE encoding
    ok = std::fwrite(words.data(), sizeof(uint64_t), words.size(), f) == words.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(HANF_IO_ERROR, std::string("write failed: ") + path);
  return HANF_OK;
}

// hll.hpp:288-303 load_counters, into a running engine (resume).
hanf_status hanf_restore_counters(hanf_engine* e, const char* path, uint64_t iteration) {
  if (!e || !path) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (!e->parts.empty())
    return fail(HANF_INVALID_ARGUMENT, "restore into a multi-device engine is not supported");
  if (e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "batched engine: no single counter array");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail(HANF_IO_ERROR, std::string("cannot open: ") + path);
  unsigned char h[28];
  const size_t got = std::fread(h, 1, sizeof h, f);
  if (got < 4 || std::memcmp(h, "HCA1", 4) != 0) {
    std::fclose(f);
    return fail(HANF_PARSE_ERROR, std::string(path) + ": bad counter snapshot magic");
  }
  if (got < sizeof h) {
    std::fclose(f);
    return fail(HANF_PARSE_ERROR, std::string(path) + ": truncated header");
  }
  const uint64_t b = get_le(h + 4, 4), r = get_le(h + 8, 4), n = get_le(h + 12, 8),
                 seed = get_le(h + 20, 8);
  if (b != e->params.bucket_bits || r != e->params.register_bits || n != e->n) {
    std::fclose(f);
    return fail(HANF_INVALID_ARGUMENT, "snapshot (b, r, n) does not match the engine");
  }
  std::vector<uint64_t> words(n * e->words);
  const size_t rd = words.empty() ? 0 : std::fread(words.data(), sizeof(uint64_t), words.size(), f);
  std::fclose(f);
  if (rd != words.size())
    return fail(HANF_PARSE_ERROR, std::string(path) + ": truncated counter data");
  if (n == 0) {
    e->t = iteration;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  cudaStream_t s = e->stream;
  uint64_t* tmp = nullptr;
  HANF_CUDA(palloc(&tmp, words.size(), s));
  cudaError_t ce = cudaMemcpyAsync(tmp, words.data(), sizeof(uint64_t) * words.size(),
                                   cudaMemcpyHostToDevice, s);
  for (int g = 0; g < 2 && ce == cudaSuccess; ++g)  // both generations (next == cur)
    ce = hanf::launch_scatter_rows(tmp, e->perm, n, static_cast<uint32_t>(e->pitch),
                                   static_cast<uint32_t>(e->words), e->cnt[g], e->bytes,
                                   e->params.registers, s, &e->launches);
  cudaFreeAsync(tmp, s);
  HANF_CUDA(ce);
  {
    const hanf_status bs = clear_item_rows(e);
    if (bs != HANF_OK) return bs;
  }
  // every counter counts as modified: the next step recomputes every node
  HANF_CUDA(hanf::launch_seed_bitmap(e->mod[0], e->n, s));
  HANF_CUDA(cudaMemsetAsync(e->mod[1], 0, sizeof(uint64_t) * e->blocks, s));
  if (e->dirty[0]) {
    HANF_CUDA(cudaMemcpyAsync(e->dirty[0], e->mod[0], sizeof(uint64_t) * e->blocks,
                              cudaMemcpyDeviceToDevice, s));
    HANF_CUDA(cudaMemsetAsync(e->dirty[1], 0, sizeof(uint64_t) * e->blocks, s));
  }
  e->cfg.seed = seed;
  e->params.seed = seed;
  e->cur = 0;
  e->stale_valid = false;
  e->systolic = false;
  if (e->shard_relabel) e->est = e->est_gen[0];
  hanf_status st = run_estimates(e, 0, nullptr, 0, e->blocks);
  if (st != HANF_OK) return st;
  if (e->shard_relabel)
    HANF_CUDA(cudaMemcpyAsync(e->est_gen[1], e->est_gen[0], sizeof(double) * e->n,
                              cudaMemcpyDeviceToDevice, s));
  uint64_t count = 0;
  st = finish(e, dirty_of(e, 0), e->est_rows, 0, e->est_rows ? e->blocks : 0, &e->last_sum,
              &count);
  if (st != HANF_OK) return st;
  e->last_count = e->n;
  e->t = iteration;
  return HANF_OK;
}

hanf_status hanf_reseed(hanf_engine* e, uint64_t seed) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (!e->parts.empty()) {
    if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
    return multi_reset(e, &seed);
  }
  if (e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "batched engine: seeds are fixed at creation");
  e->cfg.seed = seed;
  e->params.seed = seed;  // only the seeding hash reads it (engine.hpp:84-85)
  return hanf_reset(e);
}

hanf_status hanf_sum_estimates(hanf_engine* e, double* sum) {
  if (!e || !sum) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *sum = e->n == 0 ? 0.0 : e->last_sum;
  return HANF_OK;
}

// hanf_step split at the device boundary: launch enqueues the whole step on
// the engine stream and returns; complete waits and reports.
hanf_status hanf_step_launch(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "batched engine: use hanf_run_batch");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (!e->parts.empty()) {
    const hanf_status st = multi_step_enqueue(e);
    if (st == HANF_OK) e->step_pending = true;
    return st;
  }
  if (e->n == 0) {
    e->step_pending = true;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  const hanf_status st = step_enqueue(e);
  if (st == HANF_OK) e->step_pending = true;
  return st;
}

hanf_status hanf_step_complete(hanf_engine* e, hanf_iteration_report* rep) {
  if (!e || !rep) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (!e->step_pending) return fail(HANF_INVALID_ARGUMENT, "no launched step");
  e->step_pending = false;
  if (!e->parts.empty()) return multi_step_complete(e, rep);
  if (e->n == 0) {
    rep->sum = 0.0;
    rep->modified = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  return commit_complete(e, rep);
}

hanf_status hanf_step(hanf_engine* e, hanf_iteration_report* rep) {
  if (!e || !rep) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (!e->parts.empty()) {
    hanf_status st = multi_step_enqueue(e);
    if (st != HANF_OK) return st;
    return multi_step_complete(e, rep);
  }
  if (e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "batched engine: use hanf_run_batch");
  if (e->n == 0) {                       // engine.hpp:124
    rep->sum = 0.0;
    rep->modified = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  // (phase timing needs events between the kernels: step_enqueue runs
  // ungraphed then)
  const hanf_status st = step_enqueue(e);
  if (st != HANF_OK) return st;
  return commit_complete(e, rep);
}

hanf_status hanf_shard_compute(hanf_engine* e) {
  if (e && !e->parts.empty()) return fail(HANF_INVALID_ARGUMENT, "not a shard engine");
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (e->n == 0) return HANF_OK;
  HANF_CUDA(cudaSetDevice(e->device));
  note_step(e);
  if (step_mode(e) == 2) {
    const hanf_status sst = ensure_sparse(e);
    if (sst != HANF_OK) return sst;
  }
  return compute_local(e);
}

// Changed-rows exchange: the rows this shard's step wrote (changed now or
// stale) - exactly the rows in which every peer's copy of the next
// generation differs (peers hold generation t-1 there: the same stale-slot
// invariant as the single engine).  ids/rows are device buffers.
hanf_status hanf_shard_pack(hanf_engine* e, uint32_t* ids, uint64_t* rows, uint64_t cap,
                            uint64_t* count) {
  if (!e || !count || (cap && (!ids || !rows))) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *count = 0;
  if (e->n == 0) return HANF_OK;
  if (e->relabel || e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "not a shard engine");
  HANF_CUDA(cudaSetDevice(e->device));
  const int ng = 1 - e->cur;
  if (!e->pack_count) HANF_CUDA(palloc(&e->pack_count, 1, e->stream));
  HANF_CUDA(hanf::launch_pack_rows(e->mod[ng], e->stale_valid ? e->mod[e->cur] : e->mod[ng], e->lo,
                                   e->hi, e->cnt[ng], static_cast<uint32_t>(e->pitch), ids, rows,
                                   cap, e->pack_count, count, e->stream, &e->launches));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  if (*count > cap) return HANF_CAPACITY;  // (no error message: the caller falls back)
  return HANF_OK;
}

hanf_status hanf_shard_unpack(hanf_engine* e, const uint32_t* ids, const uint64_t* rows,
                              uint64_t count) {
  if (!e || (count && (!ids || !rows))) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->n == 0 || count == 0) return HANF_OK;
  HANF_CUDA(cudaSetDevice(e->device));
  HANF_CUDA(hanf::launch_unpack_rows(ids, rows, count, e->n, static_cast<uint32_t>(e->pitch),
                                     e->cnt[1 - e->cur], e->stream, &e->launches));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  return HANF_OK;
}

hanf_status hanf_shard_commit(hanf_engine* e, hanf_iteration_report* rep) {
  if (!e || !rep) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (e->n == 0) {
    rep->sum = 0.0;
    rep->modified = 0;
    return HANF_OK;
  }
  HANF_CUDA(cudaSetDevice(e->device));
  return commit(e, rep);
}

// ---- peer-push exchange ----------------------------------------------------
hanf_status hanf_shard_export(hanf_engine* e, hanf_shard_peer* out) {
  if (e && !e->parts.empty()) return fail(HANF_INVALID_ARGUMENT, "not a shard engine");
  if (!e || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  std::memset(out, 0, sizeof(*out));
  out->n = e->n;
  out->row_pitch = e->pitch;
  out->shard_begin = e->lo;
  out->shard_end = e->hi;
  out->device = e->device;
  out->relabelled = (e->shard_relabel ? 1 : 0) | (e->bytes ? 2 : 0);
  out->arena_bytes = e->arena_bytes;
  if (!e->arena) return HANF_OK;  // a one-shard engine (all nodes): nothing to map
  HANF_CUDA(cudaSetDevice(e->device));
  // the needed-rows bitmap the peers copy at attach is complete
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  cudaIpcMemHandle_t h;
  HANF_CUDA(cudaIpcGetMemHandle(&h, e->arena));
  static_assert(sizeof(h) == sizeof(out->ipc_handle), "cudaIpcMemHandle_t size");
  std::memcpy(out->ipc_handle, &h, sizeof(h));
  return HANF_OK;
}

namespace {

// The shards must tile [0, n) with identical arenas; `self` describes e.
hanf_status check_peers(const hanf_engine* e, const hanf_shard_peer* peers, uint32_t count,
                        uint32_t self) {
  if (count == 0 || self >= count) return fail(HANF_INVALID_ARGUMENT, "self outside the peer list");
  if (count > hanf::kMaxPeers + 1)
    return fail(HANF_INVALID_ARGUMENT, "peer-push exchange: at most 8 shards");
  const hanf_shard_peer& me = peers[self];
  if (me.n != e->n || me.shard_begin != e->lo || me.shard_end != e->hi ||
      me.arena_bytes != e->arena_bytes ||
      me.relabelled != ((e->shard_relabel ? 1 : 0) | (e->bytes ? 2 : 0)))
    return fail(HANF_INVALID_ARGUMENT, "peers[self] does not describe this engine");
  std::vector<std::pair<uint64_t, uint64_t>> ranges;
  for (uint32_t p = 0; p < count; ++p) {
    if (peers[p].n != e->n || peers[p].row_pitch != e->pitch ||
        peers[p].arena_bytes != e->arena_bytes || peers[p].relabelled != me.relabelled)
      return fail(HANF_INVALID_ARGUMENT, "peer engines differ in graph or counter layout");
    if (peers[p].shard_end > peers[p].shard_begin)
      ranges.emplace_back(peers[p].shard_begin, peers[p].shard_end);
  }
  std::sort(ranges.begin(), ranges.end());
  uint64_t at = 0;
  for (const auto& r : ranges) {
    if (r.first != at) return fail(HANF_INVALID_ARGUMENT, "shard ranges do not tile [0, n)");
    at = r.second;
  }
  if (at != e->n) return fail(HANF_INVALID_ARGUMENT, "shard ranges do not tile [0, n)");
  return HANF_OK;
}

}  // namespace

namespace {

// Peer-push filter, at attach: copies every peer's needed-rows bits over
// this shard's range (words [lo/64, ceil(hi/64)) of the peer's arena
// region 8) into need_of.  The peers' bitmaps are complete: export and
// attach_local synchronise the peer's stream first.
hanf_status load_peer_need(hanf_engine* e) {
  if (!e->need_filter || e->npeers == 0 || e->hi <= e->lo) return HANF_OK;
  const uint64_t w0 = e->lo >> 6, w1 = (e->hi + 63) >> 6;
  e->need_words = w1 - w0;
  HANF_CUDA(cudaMalloc(&e->need_of, sizeof(uint64_t) * e->npeers * e->need_words));
  for (uint32_t i = 0; i < e->npeers; ++i)
    HANF_CUDA(cudaMemcpyAsync(e->need_of + i * e->need_words,
                              e->peer_base[i] + e->arena_off[8] + sizeof(uint64_t) * w0,
                              sizeof(uint64_t) * e->need_words, cudaMemcpyDefault, e->stream));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  return HANF_OK;
}

}  // namespace

// Filtered peer-push leaves this shard's copies of peer rows it never
// gathers stale; a read-back first copies every peer's own range of the
// current generation from the peer's arena (peer memory, stream-ordered).
// Rows this shard gathers are equal on both sides already.
static hanf_status pull_peer_rows(hanf_engine* e) {
  if (!e->attached || !e->need_of) return HANF_OK;
  const int g = e->cur;
  for (uint32_t i = 0; i < e->npeers; ++i) {
    const uint64_t lo = e->peer_lo[i], hi = e->peer_hi[i];
    if (hi <= lo) continue;
    HANF_CUDA(cudaMemcpyAsync(e->cnt[g] + lo * e->pitch,
                              e->peer_base[i] + e->arena_off[g] + sizeof(uint64_t) * lo * e->pitch,
                              sizeof(uint64_t) * (hi - lo) * e->pitch, cudaMemcpyDefault,
                              e->stream));
  }
  return HANF_OK;
}

hanf_status hanf_shard_attach(hanf_engine* e, const hanf_shard_peer* peers, uint32_t count,
                              uint32_t self) {
  if (!e || !peers) return fail(HANF_INVALID_ARGUMENT, "null argument");
  hanf_status st = check_peers(e, peers, count, self);
  if (st != HANF_OK) return st;
  HANF_CUDA(cudaSetDevice(e->device));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  e->detach_peers();
  if (!e->arena) return HANF_OK;  // one shard: nothing to exchange
  for (uint32_t p = 0; p < count; ++p) {
    if (p == self) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, peers[p].ipc_handle, sizeof(h));
    void* ptr = nullptr;
    const cudaError_t err = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (err != cudaSuccess) {
      e->detach_peers();
      return cuda_fail(err, "cudaIpcOpenMemHandle (peer shard arena)");
    }
    e->peer_base[e->npeers] = static_cast<uint8_t*>(ptr);
    e->peer_ipc[e->npeers] = true;
    e->peer_lo[e->npeers] = peers[p].shard_begin;
    e->peer_hi[e->npeers] = peers[p].shard_end;
    ++e->npeers;
  }
  st = load_peer_need(e);
  if (st != HANF_OK) {
    e->detach_peers();
    return st;
  }
  e->attached = true;
  return HANF_OK;
}

hanf_status hanf_shard_attach_local(hanf_engine* e, hanf_engine* const* peers, uint32_t count,
                                    uint32_t self) {
  if (!e || !peers) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (self >= count || peers[self] != e)
    return fail(HANF_INVALID_ARGUMENT, "peers[self] must be this engine");
  std::vector<hanf_shard_peer> desc(count);
  for (uint32_t p = 0; p < count; ++p) {
    if (!peers[p]) return fail(HANF_INVALID_ARGUMENT, "null peer engine");
    desc[p] = hanf_shard_peer{};
    desc[p].n = peers[p]->n;
    desc[p].row_pitch = peers[p]->pitch;
    desc[p].shard_begin = peers[p]->lo;
    desc[p].shard_end = peers[p]->hi;
    desc[p].arena_bytes = peers[p]->arena_bytes;
    desc[p].device = peers[p]->device;
    desc[p].relabelled = (peers[p]->shard_relabel ? 1 : 0) | (peers[p]->bytes ? 2 : 0);
  }
  hanf_status st = check_peers(e, desc.data(), count, self);
  if (st != HANF_OK) return st;
  HANF_CUDA(cudaSetDevice(e->device));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  e->detach_peers();
  if (!e->arena) return HANF_OK;
  for (uint32_t p = 0; p < count; ++p) {
    if (p == self) continue;
    if (peers[p]->device != e->device) {
      int ok = 0;
      HANF_CUDA(cudaDeviceCanAccessPeer(&ok, e->device, peers[p]->device));
      if (!ok) return fail(HANF_INVALID_ARGUMENT, "no peer access between the shard devices");
      const cudaError_t pe = cudaDeviceEnablePeerAccess(peers[p]->device, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (pe != cudaSuccess)
        return cuda_fail(pe, "cudaDeviceEnablePeerAccess");
    }
    e->peer_base[e->npeers] = static_cast<uint8_t*>(peers[p]->arena);
    e->peer_ipc[e->npeers] = false;
    e->peer_lo[e->npeers] = peers[p]->lo;
    e->peer_hi[e->npeers] = peers[p]->hi;
    ++e->npeers;
    // the needed-rows bitmap load_peer_need copies is complete
    HANF_CUDA(cudaSetDevice(peers[p]->device));
    HANF_CUDA(cudaStreamSynchronize(peers[p]->stream));
    HANF_CUDA(cudaSetDevice(e->device));
  }
  st = load_peer_need(e);
  if (st != HANF_OK) {
    e->detach_peers();
    return st;
  }
  e->attached = true;
  return HANF_OK;
}

hanf_status hanf_shard_reduce(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  if (!e->shard_relabel || !e->attached || e->n == 0) return HANF_OK;  // nothing to share
  HANF_CUDA(cudaSetDevice(e->device));
  const int ng = 1 - e->cur;
  const uint32_t G = e->cfg.shard_count;
  const uint64_t per = e->blocks / G;                   // (n is a multiple of 64 G)
  const uint64_t k = e->lo / (e->n / G);                // this shard's index
  const uint64_t b0 = k * per, b1 = b0 + per;
  const uint64_t* bits = nullptr;
  e->reduced = true;  // (relabel_dirty: the slice protocol is in use)
  e->ever_reduced = true;
  hanf_status st = relabel_dirty(e, &bits);
  if (st != HANF_OK) return st;
  // this rank's slice of the block sums (the totals this launch also makes
  // are discarded: the commit redoes them from the inbox)
  hanf::FinishArgs f{};
  f.est = e->est_gen[ng];
  f.bits = bits;
  f.block_sums = e->block_sums;
  f.out = e->reduce;
  f.n = e->n;
  f.blocks = e->blocks;
  f.b0 = b0;
  f.b1 = b1;
  f.perm = e->est_rows ? e->perm : nullptr;
  f.all_dirty = e->all_dirty_commit ? 1 : 0;
  HANF_CUDA(hanf::launch_finish(f, e->stream, &e->launches));
  hanf::PublishArgs p{};
  p.mod_next = nullptr;  // (bitmap words went with the compute)
  p.block_sums = e->block_sums;
  p.w0 = b0;
  p.w1 = b1;
  p.count = e->npeers;
  for (uint32_t i = 0; i < e->npeers; ++i) {
    p.peer_mod[i] = nullptr;
    p.peer_sums[i] = reinterpret_cast<double*>(e->peer_base[i] + e->arena_off[4 + ng]);
  }
  p.peer_sums[e->npeers] = e->inbox[ng];
  HANF_CUDA(hanf::launch_publish(p, e->stream, &e->launches));
  return HANF_OK;
}

hanf_status hanf_shard_push_stats(hanf_engine* e, uint64_t* changed, uint64_t* pushed) {
  if (!e || !changed || !pushed) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (!e->parts.empty()) return fail(HANF_INVALID_ARGUMENT, "not a shard engine");
  *changed = *pushed = 0;
  if (e->hi <= e->lo) return HANF_OK;
  HANF_CUDA(cudaSetDevice(e->device));
  const uint64_t w0 = e->lo >> 6, words = ((e->hi + 63) >> 6) - w0;
  const uint64_t* rows = e->mod[e->cur] + w0;  // the last step's modified bits
  uint64_t* d = nullptr;  // [0] pushed, [1] changed
  uint64_t* d_ones = nullptr;
  HANF_CUDA(palloc(&d, 2, e->stream));
  cudaError_t ce = palloc(&d_ones, words, e->stream);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(d_ones, 0xff, sizeof(uint64_t) * words, e->stream);
  if (ce == cudaSuccess)  // changed rows: popcount against one all-ones "peer"
    ce = hanf::launch_count_pushes(rows, d_ones, words, 1, d + 1, e->stream, &e->launches);
  if (ce == cudaSuccess && e->need_of)
    ce = hanf::launch_count_pushes(rows, e->need_of, words, e->npeers, d, e->stream, &e->launches);
  uint64_t h[2] = {0, 0};
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, e->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->stream);
  pfree(d, e->stream);
  if (d_ones) pfree(d_ones, e->stream);
  HANF_CUDA(ce);
  *changed = h[1];
  *pushed = e->need_of ? h[0] : h[1] * (e->attached ? e->npeers : 0);
  return HANF_OK;
}

hanf_status hanf_shard_wait(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  HANF_CUDA(cudaSetDevice(e->device));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  return HANF_OK;
}

hanf_status hanf_shard_detach(hanf_engine* e) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  HANF_CUDA(cudaSetDevice(e->device));
  HANF_CUDA(cudaStreamSynchronize(e->stream));
  e->detach_peers();
  return HANF_OK;
}

// ---- one handle over several GPUs (hanf_create_multi) ---------------------
}  // extern "C"
namespace {
hanf_status multi_cross_wait(hanf_engine* e) {
  const size_t G = e->parts.size();
  for (size_t k = 0; k < G; ++k) {
    HANF_CUDA(cudaSetDevice(e->parts[k]->device));
    for (size_t j = 0; j < G; ++j)
      if (j != k) HANF_CUDA(cudaStreamWaitEvent(e->parts[k]->stream, e->part_ev[j], 0));
  }
  return HANF_OK;
}

// Every part computes its node range on its own stream (its union kernels
// push the rows they write into the peers' arenas over NVLink peer memory,
// then publish bitmap words and block sums); each stream then waits on the
// other parts' compute events - a device-side barrier, no host round trip -
// relabelled parts re-sum their slice of the blocks behind a second such
// barrier, and every part enqueues its commit.
hanf_status multi_step_enqueue(hanf_engine* e) {
  const size_t G = e->parts.size();
  for (size_t k = 0; k < G; ++k) {
    hanf_status st = hanf_shard_compute(e->parts[k]);
    if (st != HANF_OK) return st;
    HANF_CUDA(cudaSetDevice(e->parts[k]->device));
    HANF_CUDA(cudaEventRecord(e->part_ev[k], e->parts[k]->stream));
  }
  hanf_status st = multi_cross_wait(e);
  if (st != HANF_OK) return st;
  if (e->parts[0]->shard_relabel) {
    for (size_t k = 0; k < G; ++k) {
      st = hanf_shard_reduce(e->parts[k]);
      if (st != HANF_OK) return st;
      HANF_CUDA(cudaSetDevice(e->parts[k]->device));
      HANF_CUDA(cudaEventRecord(e->part_ev[k], e->parts[k]->stream));
    }
    st = multi_cross_wait(e);
    if (st != HANF_OK) return st;
  }
  for (size_t k = 0; k < G; ++k) {
    HANF_CUDA(cudaSetDevice(e->parts[k]->device));
    st = commit_enqueue(e->parts[k]);
    if (st != HANF_OK) return st;
  }
  return HANF_OK;
}

// Every part's commit reduces the same full arrays: the reports agree.
hanf_status multi_step_complete(hanf_engine* e, hanf_iteration_report* rep) {
  hanf_iteration_report first{};
  for (size_t k = 0; k < e->parts.size(); ++k) {
    HANF_CUDA(cudaSetDevice(e->parts[k]->device));
    hanf_iteration_report r{};
    const hanf_status st = commit_complete(e->parts[k], &r);
    if (st != HANF_OK) return st;
    if (k == 0)
      first = r;
    else if (r.modified != first.modified)
      return fail(HANF_CUDA_ERROR, "shard engines disagree on the modified count");
  }
  e->t = e->parts[0]->t;
  e->last_sum = e->parts[0]->last_sum;
  e->last_count = e->parts[0]->last_count;
  *rep = first;
  return HANF_OK;
}

hanf_status multi_sync(hanf_engine* e) {
  for (hanf_engine* p : e->parts) {
    HANF_CUDA(cudaSetDevice(p->device));
    HANF_CUDA(cudaStreamSynchronize(p->stream));
  }
  return HANF_OK;
}

hanf_status multi_reset(hanf_engine* e, const uint64_t* seed) {
  hanf_status st = multi_sync(e);  // no part may still push into a peer being re-seeded
  if (st != HANF_OK) return st;
  for (hanf_engine* p : e->parts) {
    st = seed ? hanf_reseed(p, *seed) : hanf_reset(p);
    if (st != HANF_OK) return st;
  }
  st = multi_sync(e);
  if (st != HANF_OK) return st;
  if (seed) {
    e->cfg.seed = *seed;
    e->params.seed = *seed;
  }
  e->t = 0;
  e->last_sum = e->parts[0]->last_sum;
  e->last_count = e->n;
  return HANF_OK;
}
}  // namespace
extern "C" {

hanf_status hanf_create_multi(const hanf_graph_view* g, const hanf_config* cfg,
                              const int32_t* devices, uint32_t count, hanf_engine** out) {
  if (!g || !cfg || !devices || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (count < 1 || count > HANF_MAX_PEERS + 1)
    return fail(HANF_INVALID_ARGUMENT, "hanf_create_multi takes 1.." +
                                           std::to_string(HANF_MAX_PEERS + 1) + " devices");
  if (cfg->shard_begin || cfg->shard_end)
    return fail(HANF_INVALID_ARGUMENT, "hanf_create_multi makes the shards itself");
  const uint64_t n = g->n;
  if (count == 1 || n < 64ull * count) {  // one shard (tiny graphs: no empty shards)
    hanf_config c = *cfg;
    c.device = devices[0];
    return hanf_create(g, &c, out);
  }
  // contiguous ranges of ceil(n / count) nodes rounded up to 64 (whole
  // bitmap words and blocks); n % (64 count) == 0 gives equal shards, which
  // may relabel (interleaved by degree)
  uint64_t per = (n + count - 1) / count;
  per = (per + 63) / 64 * 64;
  std::unique_ptr<hanf_engine> m(new (std::nothrow) hanf_engine());
  if (!m) return fail(HANF_OUT_OF_MEMORY, "engine allocation failed");
  m->device = -1;
  for (uint32_t k = 0; k < count; ++k) {
    hanf_config c = *cfg;
    c.device = devices[k];
    c.shard_begin = std::min<uint64_t>(n, k * per);
    c.shard_end = std::min<uint64_t>(n, (k + 1) * per);
    c.shard_count = count;
    hanf_engine* part = nullptr;
    hanf_status st = hanf_create(g, &c, &part);
    if (st != HANF_OK) return st;  // (m's destructor frees the parts made so far)
    m->parts.push_back(part);
    m->part_ev.push_back(nullptr);
    HANF_CUDA(cudaSetDevice(devices[k]));
    HANF_CUDA(cudaEventCreateWithFlags(&m->part_ev.back(), cudaEventDisableTiming));
  }
  for (uint32_t k = 1; k < count; ++k)
    if (m->parts[k]->shard_relabel != m->parts[0]->shard_relabel)
      return fail(HANF_INVALID_ARGUMENT, "shards disagree on relabelling");
  for (uint32_t k = 0; k < count; ++k) {
    const hanf_status st = hanf_shard_attach_local(m->parts[k], m->parts.data(), count, k);
    if (st != HANF_OK) return st;
  }
  m->cfg = m->parts[0]->cfg;  // (normalised: max_iterations 0 -> n + 1, ...)
  m->cfg.device = devices[0];
  m->cfg.shard_begin = m->cfg.shard_end = 0;
  m->cfg.shard_count = 0;
  m->params = m->parts[0]->params;
  m->n = n;
  m->lo = 0;
  m->hi = n;
  m->blocks = m->parts[0]->blocks;
  m->words = m->parts[0]->words;
  m->pitch = m->parts[0]->pitch;
  m->last_sum = m->parts[0]->last_sum;
  m->last_count = n;
  *out = m.release();
  return HANF_OK;
}

hanf_status hanf_run_to_stabilisation(hanf_engine* e, double* values, uint64_t* modified,
                                      uint64_t capacity, uint64_t* length, double* wall) {
  if (!e || !length) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (e->batch > 1) return fail(HANF_INVALID_ARGUMENT, "batched engine: use hanf_run_batch");
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
  const bool sharded = e->lo != 0 || e->hi != e->n || !e->parts.empty();
  if (e->cfg.termination == 0 && !e->timing && !sharded) {
    // Pipelined: once a step's modified count is known, the next step is
    // launched before the host sums this step's block sums (exact_sum) -
    // the next step reads only the count.  Same steps, same bits.
    HANF_CUDA(cudaSetDevice(e->device));
    hanf_status st = step_enqueue(e);
    if (st != HANF_OK) return st;
    for (;;) {
      const int parity = e->cur;
      HANF_CUDA(cudaStreamSynchronize(e->stream));
      const uint64_t count = e->h_reduce->count;
      const double dev_total = e->h_reduce->total;
      advance_state(e, count);
      if (count == 0) break;  // the stabilising step is not recorded
      const bool capped = vals.size() >= e->cfg.max_iterations;  // no further step allowed
      if (!capped) {
        st = step_enqueue(e);
        if (st != HANF_OK) return st;
      }
      const double total = e->cfg.exact_sum ? host_block_total(e, parity) : dev_total;
      e->last_sum = total;
      vals.push_back(total);
      mods.push_back(count);
      if (capped)
        return fail(HANF_GUARD, "engine: iteration cap " + std::to_string(e->cfg.max_iterations) +
                                    " exceeded; pathological input or bug");
    }
  } else for (;;) {
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
  if (e->step_pending) return fail(HANF_INVALID_ARGUMENT, "a launched step is not complete");
  if (!e->parts.empty()) return hanf_read_counters(e->parts[0], first, count, dst);
  if (first > e->n || count > e->n - first)
    return fail(HANF_OUT_OF_RANGE, "counter index out of range");
  if (count == 0) return HANF_OK;
  if (!dst) return fail(HANF_INVALID_ARGUMENT, "null destination");
  HANF_CUDA(cudaSetDevice(e->device));
  {
    const hanf_status ps = pull_peer_rows(e);
    if (ps != HANF_OK) return ps;
  }
  if (e->relabel || e->bytes) {
    // counter of original id first + i lives in row perm[first + i]; byte
    // rows are packed into the reference layout on the way
    uint64_t* tmp = nullptr;
    HANF_CUDA(palloc(&tmp, count * e->words, e->stream));
    cudaError_t ce = hanf::launch_gather_rows(e->cnt[e->cur], e->perm, first, count,
                                              static_cast<uint32_t>(e->pitch),
                                              static_cast<uint32_t>(e->words), tmp, e->bytes,
                                              e->params.registers, e->stream, &e->launches);
    if (ce == cudaSuccess)
      ce = cudaMemcpyAsync(dst, tmp, sizeof(uint64_t) * count * e->words, cudaMemcpyDeviceToHost,
                           e->stream);
    cudaFreeAsync(tmp, e->stream);
    HANF_CUDA(ce);
    HANF_CUDA(cudaStreamSynchronize(e->stream));
    return HANF_OK;
  }
  // rows are `pitch` words apart on the device, W apart in the reference
  // packing the caller expects
  HANF_CUDA(cudaMemcpy2DAsync(dst, sizeof(uint64_t) * e->words, e->cnt[e->cur] + first * e->pitch,
                              sizeof(uint64_t) * e->pitch, sizeof(uint64_t) * e->words, count,
                              cudaMemcpyDeviceToHost, e->stream));
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
  *active = (e->parts.empty() ? e : e->parts[0])->systolic ? 1 : 0;
  return HANF_OK;
}

hanf_status hanf_num_nodes(const hanf_engine* e, uint64_t* n) {
  if (!e || !n) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *n = e->n;
  return HANF_OK;
}

hanf_status hanf_stream(const hanf_engine* e, void** stream) {
  if (!e || !stream) return fail(HANF_INVALID_ARGUMENT, "null argument");
  // (multi-device handles: the first part's stream)
  *stream = static_cast<void*>(e->parts.empty() ? e->stream : e->parts[0]->stream);
  return HANF_OK;
}

hanf_status hanf_launch_count(const hanf_engine* e, uint64_t* launches) {
  if (!e || !launches) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *launches = e->launches;
  for (const hanf_engine* p : e->parts) *launches += p->launches;
  return HANF_OK;
}

hanf_status hanf_block_stats(const hanf_engine* e, uint64_t* items, uint64_t* arcs) {
  if (!e || !items || !arcs) return fail(HANF_INVALID_ARGUMENT, "null argument");
  *items = e->block_ready ? e->block_items : 0;
  *arcs = e->block_ready ? e->block_arcs : 0;
  return HANF_OK;
}

hanf_status hanf_set_timing(hanf_engine* e, int32_t enable) {
  if (!e) return fail(HANF_INVALID_ARGUMENT, "null engine");
  for (hanf_engine* p : e->parts) {  // multi-device: per part (hanf_timing reports the first)
    const hanf_status st = hanf_set_timing(p, enable);
    if (st != HANF_OK) return st;
  }
  if (!e->parts.empty()) return HANF_OK;
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
  if (!e->parts.empty()) e = e->parts[0];
  if (union_ms) *union_ms = e->union_ms;
  if (estimate_ms) *estimate_ms = e->estimate_ms;
  if (reduce_ms) *reduce_ms = e->reduce_ms;
  if (steps) *steps = e->timed_steps;
  return HANF_OK;
}

hanf_status hanf_pin_host(const void* p, uint64_t bytes) {
  if (!p || bytes == 0) return fail(HANF_INVALID_ARGUMENT, "null or empty host range");
  HANF_CUDA(cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterPortable));
  return HANF_OK;
}

hanf_status hanf_unpin_host(const void* p) {
  if (!p) return fail(HANF_INVALID_ARGUMENT, "null host pointer");
  HANF_CUDA(cudaHostUnregister(const_cast<void*>(p)));
  return HANF_OK;
}

hanf_status hanf_device_buffers(hanf_engine* e, hanf_buffers* out) {
  if (!e || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (!e->parts.empty()) return fail(HANF_INVALID_ARGUMENT, "multi-device engine: no single buffer set");
  const int ng = 1 - e->cur;
  out->next_counters = e->cnt[ng];
  out->next_modified = e->mod[ng];
  out->block_sums = e->block_sums;
  out->words_per_counter = e->words;
  out->row_pitch = e->pitch;
  out->blocks = e->blocks;
  out->shard_begin = e->lo;
  out->shard_end = e->hi;
  out->relabelled = e->relabel ? 1u : 0u;
  out->reserved = 0;
  return HANF_OK;
}

}  // extern "C"
