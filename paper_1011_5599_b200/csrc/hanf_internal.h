// hanf_internal.h -- host-side declarations shared by the engine and the
// kernel launchers (not part of the public ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hanf {

// Warp-task classes of the union kernel.
// Class 0 holds hub chunks (one warp per <= kHubChunk arcs of a node with
// out-degree > kHubDegree, writing a partial counter); classes 1..6 hold
// nodes handled by G = 32, 16, 8, 4, 2, 1 lanes each, ordered by
// descending degree so the longest tasks start first.
constexpr int kNumClasses = 7;
constexpr uint32_t kHubDegree = 1024;
constexpr uint32_t kHubChunk = 1024;

struct TaskTable {
  uint32_t warp_begin[kNumClasses + 1];  // prefix of warp counts; [7] = total warps
  uint32_t item_begin[kNumClasses];      // first index into order[] / hub arrays
  uint32_t item_end[kNumClasses];
  uint32_t log2g[kNumClasses];           // lanes per node = 1 << log2g
};

struct UnionArgs {
  const uint64_t* offsets;   // CSR offsets (global node ids, absolute arc index)
  const uint32_t* succ;      // CSR successor ids
  const uint64_t* cur;       // generation t (read only)
  uint64_t* next;            // generation t+1
  const uint64_t* mod_cur;   // bitmap: counters changed by the previous step
  uint64_t* mod_next;        // bitmap: counters changed by this step (pre-zeroed)
  const uint32_t* order;     // node ids of classes 1..6
  const uint32_t* hub_node;  // per hub chunk: node
  const uint64_t* hub_begin; // per hub chunk: arc range
  const uint64_t* hub_end;
  uint64_t* partials;        // per hub chunk: partial counter (W words)
  uint64_t succ_base;        // arc index of succ[0] (shard-local CSR)
  uint32_t words;            // W
  uint32_t chunks;           // chunks per counter
  int32_t check_mod;         // skip successors whose bit is clear in mod_cur
  int32_t stale_valid;       // next[v] may be stale where mod_cur[v] is set
  TaskTable tasks;
};

struct HubArgs {
  const uint64_t* cur;
  uint64_t* next;
  const uint64_t* mod_cur;
  uint64_t* mod_next;
  const uint32_t* hub_nodes;      // distinct hub nodes
  const uint32_t* hub_first;      // first chunk of each hub
  const uint32_t* hub_count;      // chunks of each hub
  const uint64_t* partials;
  uint32_t num_hubs;
  uint32_t words;
  uint32_t chunks;
  int32_t stale_valid;
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
  uint32_t words;
  const double* log_table;
};

// Launchers (hanf_kernels.cu).  All are stream-ordered and asynchronous.
cudaError_t launch_seed(uint64_t* a, uint64_t* b, uint64_t* mod, uint64_t n,
                        uint64_t node_begin, uint64_t node_end, uint32_t bucket_bits,
                        uint32_t register_bits, uint32_t words, uint64_t seed,
                        cudaStream_t s, uint64_t* launches);
cudaError_t launch_union(const UnionArgs& args, uint32_t register_bits,
                         uint32_t registers, cudaStream_t s, uint64_t* launches);
cudaError_t launch_hub_finalize(const HubArgs& args, uint32_t register_bits,
                                uint32_t registers, cudaStream_t s, uint64_t* launches);
cudaError_t launch_estimate(const EstimateArgs& args, cudaStream_t s, uint64_t* launches);
constexpr int kReduceCtas = 296;
constexpr int kReduceThreads = 256;
struct ReduceOut {
  double total;
  unsigned long long count;
  double partial_sum[kReduceCtas];
  unsigned long long partial_count[kReduceCtas];
};
cudaError_t launch_reduce(const double* block_sums, const uint64_t* bits, uint64_t begin,
                          uint64_t end, ReduceOut* out, cudaStream_t s, uint64_t* launches);

}  // namespace hanf
