// hanf_internal.h -- host-side declarations shared by the engine and the
// kernel launchers (not part of the public ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "hanf_device.cuh"

namespace hanf {

// Union sweep work decomposition (see hanf_kernels.cu and build_tasks):
// nodes with out-degree > kHubDegree are split into chunks of kHubChunk arcs.
constexpr uint32_t kHubDegree = 1024;
constexpr uint32_t kHubChunk = 1024;

struct WarpTask {      // 16 bytes, one per warp of the union launch
  uint64_t tos;        // first id of this warp in the task-ordered successor array
  uint32_t item;       // light: first index into order[]; hub: chunk index
  uint16_t trips;      // id rows of 32 (= max successors per lane)
  uint8_t lg;          // log2(lanes per node)
  uint8_t nodes;       // light: nodes in this warp (<= 32 >> lg); 0 = hub chunk
};

// Device-built work of the union sweep (hanf_build.cu); pool allocations.
struct TaskBuild {
  uint32_t* order = nullptr;       // light nodes, descending degree
  WarpTask* wtasks = nullptr;      // hub chunks first, then light warps (heavy first)
  uint32_t* tos = nullptr;         // task-ordered successor ids
  uint64_t tos_words = 0;
  uint32_t num_wtasks = 0;
  uint32_t* chunk_node = nullptr;  // per hub chunk: node, hub index
  uint32_t* chunk_hub = nullptr;
  uint32_t num_chunks = 0;
  uint32_t* hub_nodes = nullptr;   // per hub: node, first chunk, chunks, ticket
  uint32_t* hub_first = nullptr;
  uint32_t* hub_count = nullptr;
  uint32_t* hub_ticket = nullptr;
  uint32_t num_hubs = 0;
  uint64_t active_nodes = 0;       // nodes of the range with out-degree >= 1
  // Segments (graphs whose ids carry locality): light tasks are grouped by
  // node segment v >> seg_shift (degree order within a segment), and
  // [seg_min[s], seg_max[s]] bounds the successors and nodes of segment s,
  // so a skip sweep drops every task of a segment with no modified row in
  // that range (hanf_kernels.cu segment_live_kernel).  seg_shift = 32: one
  // segment, no bounds.
  uint32_t seg_shift = 32;
  uint32_t num_segs = 1;
  uint32_t* seg_min = nullptr;
  uint32_t* seg_max = nullptr;
  // light tasks in groups of one (segment, class) pair, segment-major (the
  // locality order) or class-major (pipelined create: the heaviest tasks of
  // every segment first); group k = task slots [group_task_begin[k],
  // group_task_begin[k+1]) of segment group_seg[k] (hub chunk tasks are
  // slots [0, num_chunks))
  std::vector<uint64_t> group_task_begin;
  std::vector<uint32_t> group_seg;
  uint64_t* chunk_begin = nullptr;  // (build scratch)
  int* fill_bad = nullptr;
};
// The CSR as the task build reads it: node (row) v's successors are arcs
// [begin(v), end(v)) of `succ` (from index succ_base), each mapped through
// `perm` when the graph is relabelled (row v = original id orig_of[v];
// `off` is then indexed by original id, lo = 0).
struct CsrView {
  const uint64_t* off;
  uint64_t lo;
  const uint32_t* succ;
  uint64_t succ_base;
  const uint32_t* orig_of;  // nullptr: identity labels (off indexed by v - lo)
  const uint32_t* perm;
  uint64_t n;
  // Source-blocked dense sweeps (hanf_block.cu): rows [0, ovr_rows) take
  // their successor lists from a second CSR already in row space (arc
  // indices of that CSR carry kOvr, so begin/end/id stay the whole
  // interface and end - begin is still the degree).
  const uint64_t* ovr_off = nullptr;
  const uint32_t* ovr_succ = nullptr;
  uint64_t ovr_rows = 0;
  static constexpr uint64_t kOvr = 1ull << 63;
  __device__ __forceinline__ uint64_t begin(uint64_t v) const {
    if (v < ovr_rows) return kOvr | ovr_off[v];
    return orig_of ? off[orig_of[v]] : off[v - lo];
  }
  __device__ __forceinline__ uint64_t end(uint64_t v) const {
    if (v < ovr_rows) return kOvr | ovr_off[v + 1];
    return orig_of ? off[orig_of[v] + 1] : off[v - lo + 1];
  }
  __device__ __forceinline__ uint32_t id(uint64_t k) const {
    if (k & kOvr) return ovr_succ[k & ~kOvr];
    const uint32_t w = succ[k - succ_base];
    return perm && w < n ? perm[w] : w;  // out-of-range ids stay out of range (flagged)
  }
};
// Builds the tasks of nodes [lo, hi) from the shard's CSR on the device.
// Sets *bad_input when offsets decrease or an arc endpoint is >= n.  Only
// the final TOS fill reads the arcs: it waits for `succ_ready` (when
// non-null), so the arcs upload overlaps the degree sort and task layout.
// Successor ids must be < id_limit (0: n); TOS padding is always row n.
cudaError_t build_tasks_device(const CsrView& g, uint64_t lo, uint64_t hi, uint64_t n,
                               uint32_t seg_shift, cudaStream_t s, cudaEvent_t succ_ready,
                               TaskBuild* out, int* bad_input, uint64_t* launches,
                               bool seg_bounds = true, bool class_major = false,
                               uint64_t id_limit = 0);
// Source-blocked dense sweeps (hanf_block.cu).  The arcs from the `sources`
// first rows (the highest out-degrees of a relabelled engine) to rows >=
// `cold` are cut out of those rows' lists and regrouped into items: one per
// (segment of 2^seg_shift successor rows, source) pair with at least one
// such arc, numbered segment-major.  Item k becomes row n + 1 + k of the
// counter arrays: a first sweep over the items (successors = the cold rows,
// all tasks of a segment together, so the segment stays in L2) leaves the
// item's maximum in that row, and the main sweep gathers it through the
// one id that replaced the item's arcs in its source's list.
struct BlockSplit {
  uint64_t* item_off = nullptr;  // [items + 1] into item_succ
  uint32_t* item_succ = nullptr; // cold successor rows, item after item
  uint64_t items = 0;
  uint64_t blocked_arcs = 0;
  uint64_t* src_off = nullptr;   // [sources + 1] into src_succ
  uint32_t* src_succ = nullptr;  // per source: its rows < cold, then n + 1 + k per item
  uint64_t src_arcs = 0;
};
cudaError_t build_block_split(const CsrView& g, uint64_t n, uint64_t sources, uint64_t cold,
                              uint32_t seg_shift, cudaStream_t s, BlockSplit* out,
                              uint64_t* launches);
void free_block_split(BlockSplit* b, cudaStream_t s);
void free_tasks_device(TaskBuild* t, cudaStream_t s);

// Locality relabelling (hanf_relabel.cu): rows renumbered by descending
// out-degree, from the offsets alone; order[row] = original id, perm[id] =
// row, off = the relabelled offsets (pool allocations, caller frees).
struct RelabelOut {
  uint32_t* order = nullptr;
  uint32_t* perm = nullptr;
  uint64_t* off = nullptr;
};
// ways > 1 (relabelled shards, n a multiple of 64 * ways): degree rank i
// goes to row (i mod ways) * n/ways + i / ways, so every shard's rows get
// the same degree profile with its hot rows first.  Rows of an odd pitch
// (< 16 words) past a hot prefix are assigned line-aligned slots first
// (the coldest ranks take the rows that straddle a 128-byte line).
cudaError_t relabel_order_device(const uint64_t* d_off, uint64_t n, uint32_t ways, uint32_t pitch,
                                 cudaStream_t s, RelabelOut* out, uint64_t* launches);
// The relabelled arcs (only the worklist step's transpose needs them; the
// union sweep's TOS is filled through CsrView).  *bad = arc endpoint >= n.
// ids[i] = perm[ids[i]] in place for ids < n (arc chunks mapped to rows as
// they land, under the rest of the upload).
cudaError_t launch_map_ids(uint32_t* ids, uint64_t count, const uint32_t* perm, uint64_t n,
                           cudaStream_t s, uint64_t* launches);
cudaError_t relabel_arcs_device(const uint64_t* d_off, const uint32_t* d_succ, uint64_t n,
                                uint64_t arcs, const RelabelOut& r, cudaStream_t s,
                                uint32_t** succ_out, int* bad, uint64_t* launches);
// rows perm[first + i] (or first + i) of `counters`, W words each, packed
// densely into dst (device)
cudaError_t launch_seed_bitmap(uint64_t* bits, uint64_t n, cudaStream_t s);
cudaError_t launch_summary(const uint64_t* bits, uint64_t words, uint32_t shift, uint64_t summ_bits,
                           uint64_t* summ, cudaStream_t s, uint64_t* launches);
// (bytes: the device rows are byte registers, `registers` of them; the
// dense rows on the other side keep the reference packing, r = 5)
cudaError_t launch_scatter_rows(const uint64_t* src, const uint32_t* perm, uint64_t count,
                                uint32_t pitch, uint32_t words, uint64_t* counters, bool bytes,
                                uint32_t registers, cudaStream_t s, uint64_t* launches);
cudaError_t launch_gather_rows(const uint64_t* counters, const uint32_t* perm, uint64_t first,
                               uint64_t count, uint32_t pitch, uint32_t words, uint64_t* dst,
                               bool bytes, uint32_t registers, cudaStream_t s, uint64_t* launches);

// Worklist ("systolic") step, hanf_sparse.cu.
struct SparseArgs {
  const uint64_t* off;        // shard CSR offsets (index v - node_base)
  const uint32_t* succ;       // shard CSR arcs (index arc - succ_base)
  uint64_t succ_base;
  uint64_t node_base;
  const uint64_t* cur;
  uint64_t* next;
  const uint64_t* mod_cur;
  uint64_t* mod_next;
  double* est;
  EstimateParams ep;
  uint32_t pitch;             // row pitch (u64 words between counters)
  const unsigned long long* tr_off;  // transpose of the shard's arcs: preds of every node
  const uint32_t* tr_succ;
  uint64_t* sig;              // scratch bitmap (signalled nodes)
  unsigned long long* mod_list;  // scratch: (modified node << 32 | predecessor chunk)
  uint32_t* work;             // scratch: worklist (nodes of out-degree <= kHubDegree)
  uint32_t* hub_tasks;        // scratch: chunk tasks of worklist hubs (dense kernel)
  unsigned int* lens;         // [0] modified chunks, [1] worklist, [2] hub tasks
  const unsigned int* work_len;
  const uint32_t* orig_of;    // row -> original id (for dirty_next)
  const uint32_t* est_index;  // est slot of a row (nullptr: the row itself)
  uint64_t* dirty_next;       // original-id bitmap of changed counters (nullptr: = mod_next)
  const uint32_t* hub_index;  // node -> hub (UINT32_MAX: not a hub)
  const uint32_t* hub_first;  // per hub: first chunk task, chunk count
  const uint32_t* hub_count;
  uint64_t n, blocks, hi;
  PeerRows peers;             // sharded peer-push: also store written rows there
  uint32_t bytes;             // byte-layout counter store
};
// Changed-rows exchange of sharded steps (hanf_sparse.cu): the rows of
// [lo, hi) the step wrote (mod_next | mod_cur) packed as (ids, rows), and
// rows scattered back into a counter array (ids >= n are padding).
cudaError_t launch_pack_rows(const uint64_t* mod_next, const uint64_t* mod_cur, uint64_t lo,
                             uint64_t hi, const uint64_t* counters, uint32_t pitch, uint32_t* ids,
                             uint64_t* rows, uint64_t cap, unsigned long long* d_count,
                             uint64_t* count, cudaStream_t s, uint64_t* launches);
cudaError_t launch_unpack_rows(const uint32_t* ids, const uint64_t* rows, uint64_t count, uint64_t n,
                               uint32_t pitch, uint64_t* counters, cudaStream_t s,
                               uint64_t* launches);
// predecessors signalled per warp task of the signal kernel
constexpr uint32_t kSignalChunk = 256;
// node -> hub index map for the worklist step (UINT32_MAX elsewhere)
cudaError_t build_hub_index(const uint32_t* hub_nodes, uint32_t hubs, uint64_t n, cudaStream_t s,
                            uint32_t** out, uint64_t* launches);
cudaError_t build_transpose_device(const uint64_t* d_off, const uint32_t* d_succ, uint64_t lo,
                                   uint64_t hi, uint64_t succ_base, uint64_t n, cudaStream_t s,
                                   unsigned long long** tr_off, uint32_t** tr_succ,
                                   uint64_t* launches);
cudaError_t launch_sparse_step(const SparseArgs& a, uint64_t w0, uint64_t w1, uint32_t register_bits,
                               uint32_t registers, cudaStream_t s, uint64_t* launches);
bool sparse_supported(uint32_t register_bits, uint32_t registers);

struct UnionArgs {
  const uint32_t* tos;       // task-ordered successor ids
  const WarpTask* wtasks;
  uint32_t num_wtasks;
  const uint64_t* cur;       // generation t (read only)
  uint64_t* next;            // generation t+1
  const uint64_t* mod_cur;   // bitmap: counters changed by the previous step
  uint64_t* mod_next;        // bitmap: counters changed by this step (pre-zeroed)
  const uint32_t* order;     // node ids of light tasks
  const uint32_t* hub_node;  // per hub chunk: node
  uint64_t* partials;        // per hub chunk: partial counter (pitch words)
  const uint32_t* chunk_hub; // per hub chunk: hub index
  const uint32_t* hub_nodes; // per hub: node, first chunk, chunk count
  const uint32_t* hub_first;
  const uint32_t* hub_count;
  uint32_t* hub_ticket;      // per hub: chunks finished this step (self-resetting)
  uint32_t pitch;            // row pitch in u64 words (>= W, see row_pitch)
  uint32_t chunks;           // chunks per counter
  uint32_t zero_row;         // index of the all-zero counter row (= n)
  uint32_t row_limit;        // rows of cur / next (n + 1, or more with item rows: hanf_block.cu)
  int32_t check_mod;         // skip successors whose bit is clear in mod_cur
  int32_t stale_valid;       // next[v] may be stale where mod_cur[v] is set
  double* est;               // per-counter estimates (nullptr: not fused)
  EstimateParams ep;
  const uint32_t* orig_of;         // row -> original id (for dirty_next)
  const uint32_t* est_index;       // est slot of a row (nullptr: the row itself)
  uint64_t* dirty_next;            // original-id bitmap of changed counters (nullptr: = mod_next)
  const uint64_t* summ;            // mode 3: summary of mod_cur (nullptr: probe mod_cur only)
  uint32_t summ_shift;             // one summary bit per 2^summ_shift rows
  uint32_t summ_words;             // summary length (staged in shared memory)
  const uint32_t* task_list;       // non-null: run only these task indices
  const unsigned int* task_count;  // (device) length of task_list
  PeerRows peers;                  // sharded peer-push: also store written rows there
  const uint32_t* seg_live;        // skip sweeps over segmented tasks: segment s has work
  uint32_t seg_shift;              // (TaskBuild::seg_shift)
  uint32_t bytes;                  // byte-layout counter store (ByteLayout)
  size_t l2_window_bytes;          // dense sweeps: hot prefix of cur kept in persisting L2
};

struct EstimateArgs {
  const uint64_t* counters;  // generation to estimate
  const uint64_t* dirty;     // bitmap: counters to re-estimate (nullptr = all)
  double* est;               // cached per-counter estimates
  double* block_sums;        // per 64-counter block
  unsigned long long* count; // += popcount of dirty over the range
  uint64_t n;
  uint64_t block_begin;      // blocks [block_begin, block_end)
  uint64_t block_end;
  double alpha;
  double m;
  uint32_t registers;
  uint32_t register_bits;
  uint32_t pitch;            // row pitch in u64 words
  const double* log_table;
  const uint32_t* row_of;    // original id -> row (nullptr: identity labels)
  uint32_t bytes;            // byte-layout counter store
};

// Task-scan step (hanf_kernels.cu, step mode 4): tasks with a successor
// modified by the previous step, listed from one flat pass over the TOS.
struct TaskScanArgs {
  const uint32_t* tos;
  uint64_t tos_words;
  const WarpTask* wtasks;
  uint32_t num_wtasks;
  uint32_t zero_row;
  const uint64_t* mod_cur;
  const uint64_t* summ;     // summary of mod_cur (one bit per 2^summ_shift rows)
  uint32_t summ_shift;
  uint32_t summ_words;
  const uint32_t* chunk_hub;
  const uint32_t* hub_first;
  const uint32_t* hub_count;
  unsigned int* flags;      // per task, zeroed before the scan
  uint32_t* list;           // listed task indices
  unsigned int* count;      // (device) list length, zeroed before the scan
};
cudaError_t launch_task_scan(const TaskScanArgs& a, cudaStream_t s, uint64_t* launches);
cudaError_t launch_stale_fixup(const uint64_t* mod_cur, const uint64_t* mod_next, uint64_t n,
                               uint32_t pitch, const uint64_t* cur, uint64_t* next, cudaStream_t s,
                               uint64_t* launches);
// Peer-push needed-rows filter: the shard's needed-rows bitmap from its TOS
// (zeroed first), and sum over peers of popcount(rows & need[p]).
cudaError_t launch_need_rows(const uint32_t* tos, uint64_t count, uint64_t n, uint64_t* need,
                             cudaStream_t s, uint64_t* launches);
cudaError_t launch_count_pushes(const uint64_t* rows, const uint64_t* need, uint64_t words,
                                uint32_t peers, uint64_t* out, cudaStream_t s, uint64_t* launches);

// Launchers (hanf_kernels.cu).  All are stream-ordered and asynchronous.
cudaError_t launch_seed(uint64_t* a, uint64_t* b, uint64_t* mod, uint64_t n,
                        uint64_t node_begin, uint64_t node_end, uint32_t bucket_bits,
                        uint32_t register_bits, uint32_t words, uint32_t pitch, uint64_t seed,
                        const uint32_t* orig_of, uint32_t batch, const uint64_t* batch_mix,
                        bool bytes, cudaStream_t s, uint64_t* launches);
// Batched runs (hanf_batch.cu): the K-fold lifted CSR (row v*K + k), and
// the per-run block sums / modified counts of a generation.
cudaError_t lift_graph_device(const uint64_t* d_off, const uint32_t* d_succ, uint64_t n, uint64_t arcs,
                              uint32_t K, cudaStream_t s, uint64_t** voff, uint32_t** vsucc,
                              uint64_t* launches);
cudaError_t launch_finish_batch(const double* est, const uint64_t* bits, uint64_t n_real, uint32_t K,
                                bool recompute, double* block_sums, unsigned long long* counts,
                                cudaStream_t s, uint64_t* launches);
cudaError_t launch_union(const UnionArgs& args, uint32_t register_bits,
                         uint32_t registers, cudaStream_t s, uint64_t* launches);
cudaError_t launch_estimate(const EstimateArgs& args, cudaStream_t s, uint64_t* launches);
// true when the union kernels compute estimates themselves (single-chunk layouts)
bool fused_estimates(uint32_t register_bits, uint32_t registers);
// Row pitch of the counter arrays (u64 words between counters): W, except
// W = 3 which is padded to one aligned 32-byte sector
// (profiles/r01_row_pitch.md); m / 8 in the byte layout.
uint32_t row_pitch(uint32_t register_bits, uint32_t registers, uint32_t words, bool bytes);
// The byte layout serves r = 5 with 16 <= m <= 128 (one to eight lanes per
// row); other layouts keep the reference packing on the device too.
bool byte_layout_supported(uint32_t register_bits, uint32_t registers);

// Step epilogue (block sums + totals), see finish_kernel.
constexpr int kFinishThreads = 256;  // threads per CTA
constexpr int kFinishBlocks = 64;    // 64-counter blocks per CTA
struct ReduceOut {
  double total;
  unsigned long long count;
  unsigned int ticket;
  double* partial_sum;              // [ceil(blocks / kFinishBlocks)]
  unsigned long long* partial_count;
};
struct FinishArgs {
  const double* est;      // per-counter estimates (nullptr: block sums are current)
  const uint64_t* bits;   // modified bitmap = dirty flags of the blocks
  double* block_sums;
  ReduceOut* out;
  uint64_t n;
  uint64_t blocks;        // totals over [0, blocks)
  uint64_t b0, b1;        // block sums recomputed over [b0, b1)
  const uint32_t* perm = nullptr;  // estimates in row order: original id o is est[perm[o]]
  int32_t all_dirty = 0;           // recompute every block of [b0, b1) (bits: count only)
  ReduceOut* host_out = nullptr;   // page-locked: total + count written there too (zero-copy
                                   // report, no read-back copy after the kernel)
  uint64_t* clear = nullptr;       // words [0, blocks) zeroed (the next step's mod_next)
  double* host_sums = nullptr;     // page-locked: every block sum [0, blocks) written there
                                   // too (exact_sum: the host redoes the total in order)
};
cudaError_t launch_finish(const FinishArgs& a, cudaStream_t s, uint64_t* launches);
// dirty[order[r] / 64] |= bit for every row r set in `rows` (pre-zeroed
// dirty; relabelled shards' commit of a step with few changes)
cudaError_t launch_derive_dirty(const uint64_t* rows, const uint32_t* order, uint64_t words,
                                uint64_t n, uint64_t* dirty, cudaStream_t s, uint64_t* launches);
// live[s] = some row of [seg_min[s], seg_max[s]] is set in mod_cur (a
// segment without one has no node that can change or is stale)
cudaError_t launch_segment_live(const uint64_t* mod_cur, const uint32_t* seg_min,
                                const uint32_t* seg_max, uint32_t segs, uint32_t* live,
                                cudaStream_t s, uint64_t* launches);
// Peer-push exchange: bitmap words and block sums [w0, w1) of this shard
// into every peer's arena (and the block sums into the local inbox).
struct PublishArgs {
  const uint64_t* mod_next;  // nullptr: block sums only
  const double* block_sums;  // nullptr: bitmap words only
  uint64_t w0, w1;
  uint64_t* peer_mod[kMaxPeers];
  double* peer_sums[kMaxPeers + 1];  // [count] = the local inbox
  uint32_t count;
};
cudaError_t launch_publish(const PublishArgs& a, cudaStream_t s, uint64_t* launches);

}  // namespace hanf
