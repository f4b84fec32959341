// hanf_build.cu -- builds the union sweep's work on the device, once per
// graph (NfEngine construction, engine.hpp:70-90):
//
//   1. degrees of the shard's nodes; bad CSR input (decreasing offsets, arc
//      endpoint >= n) raises a flag instead of a host pass over the arcs;
//   2. nodes with out-degree >= 1 sorted by descending degree, stable in id
//      (CUB radix sort of (~deg, id));
//   3. nodes of out-degree > kHubDegree are split into kHubChunk-arc chunks
//      (one warp each); the others form "light" warps of 32/G nodes with
//      G = next_pow2(ceil(deg/32)) lanes per node;
//   4. the task-ordered successor array (TOS): warp w owns rows
//      [tos/32, tos/32 + trips) of 32 ids, lane (node slot j, sub) holding
//      successor i*G + sub of node j in row i, or the zero row n.
// All buffers come from the stream-ordered pool (cudaMallocAsync).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdint>
#include <cstring>
#include <vector>

#include "hanf_internal.h"

namespace hanf {
namespace {

__host__ __device__ __forceinline__ uint32_t log2g_of(uint64_t d) {
  uint32_t g = 0;
  while ((32ull << g) < d) ++g;  // G = 2^g lanes, each walks <= 32 arcs
  return g;
}

// keys = (group prefix << 32) | ~deg, vals = node: hubs (prefix 0) first
// in descending degree, then light nodes by group - one (segment, class)
// pair, prefix 1 + group_index(), see TaskBuild - and descending degree
// within it; degree-0 nodes get the largest key and sort to the tail.
// Counts hubs and degree-0 nodes.
__host__ __device__ __forceinline__ uint64_t group_index(uint32_t seg, uint32_t lg, uint32_t segs,
                                                         bool class_major) {
  return class_major ? static_cast<uint64_t>(5 - lg) * segs + seg
                     : static_cast<uint64_t>(seg) * 6 + (5 - lg);
}

__global__ void degree_keys_kernel(const CsrView g, uint64_t lo, uint64_t count, uint32_t seg_shift,
                                   uint32_t segs, bool class_major,
                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                   unsigned long long* __restrict__ counters, int* __restrict__ bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  unsigned long long hubs = 0, zeros = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += stride) {
    const uint64_t a = g.begin(lo + i), b = g.end(lo + i);
    if (b < a) {
      *bad = 1;
      keys[i] = ~0ull;
      vals[i] = static_cast<uint32_t>(lo + i);
      ++zeros;
      continue;
    }
    const uint64_t d = b - a;
    const uint64_t dk = ~static_cast<uint32_t>(d < 0xfffffffeull ? d : 0xfffffffeull);
    const uint32_t seg = seg_shift >= 32 ? 0u : static_cast<uint32_t>((lo + i) >> seg_shift);
    const uint64_t grp = 1 + group_index(seg, log2g_of(d), segs, class_major);
    keys[i] = d == 0 ? ~0ull : (d > kHubDegree ? dk : (grp << 32) | dk);
    vals[i] = static_cast<uint32_t>(lo + i);
    hubs += d > kHubDegree;
    zeros += d == 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    hubs += __shfl_down_sync(0xffffffffu, hubs, o);
    zeros += __shfl_down_sync(0xffffffffu, zeros, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hubs) atomicAdd(counters + 0, hubs);
    if (zeros) atomicAdd(counters + 1, zeros);
  }
}

// Group boundaries in the sorted light range [begin, end): bounds[i] =
// first index whose key prefix is > i (group i = [bounds[i-1], bounds[i])
// with bounds[-1] = begin), i < groups.
__global__ void group_bounds_kernel(const uint64_t* __restrict__ sorted_keys, uint64_t begin,
                                    uint64_t end, uint64_t groups,
                                    unsigned long long* __restrict__ bounds) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= groups) return;
  const uint64_t key = (i + 2) << 32;  // first key of group i + 1
  uint64_t a = begin, b = end;
  while (a < b) {
    const uint64_t mid = (a + b) / 2;
    if (sorted_keys[mid] < key) a = mid + 1; else b = mid;
  }
  bounds[i] = a;
}

// light warp tasks: slots [C, C + W).  Group k = one (segment, class)
// pair in task order (segments ascending, heavier classes first); groups
// are non-empty, warp_begin ascending.
struct LightGroup {
  uint64_t item_begin;  // index into order[] (light nodes only)
  uint64_t item_end;
  uint64_t warp_begin;  // task slots, relative to the first light slot
  uint32_t lg;          // lanes per node = 2^lg
  uint32_t pad;
};

// Group table from the boundaries (one CTA): group i = sorted positions
// [bounds[i-1], bounds[i]) (bounds[-1] = hubs), its class, and its first
// light warp = exclusive scan of the groups' warp counts; wbeg[ng] = total.
// Empty groups get warp_begin = the next group's (light_tasks_kernel's
// binary search then skips them).
__global__ void __launch_bounds__(1024)
groups_kernel(const unsigned long long* __restrict__ bounds, uint64_t ng, uint64_t hubs,
              uint32_t segs, bool class_major, LightGroup* __restrict__ groups,
              unsigned long long* __restrict__ wbeg) {
  __shared__ unsigned long long part[1024];
  unsigned long long carry = 0;
  for (uint64_t base = 0; base < ng; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    unsigned long long w = 0;
    uint32_t lg = 0;
    uint64_t a = 0, e = 0;
    if (i < ng) {
      a = i ? bounds[i - 1] : hubs;
      e = bounds[i];
      lg = class_major ? 5 - static_cast<uint32_t>(i / segs) : 5 - static_cast<uint32_t>(i % 6);
      const uint64_t per = 32u >> lg;
      w = e > a ? (e - a + per - 1) / per : 0;
    }
    part[threadIdx.x] = w;
    __syncthreads();
    for (uint32_t o = 1; o < 1024; o <<= 1) {  // inclusive scan (Hillis-Steele)
      const unsigned long long x = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += x;
      __syncthreads();
    }
    const unsigned long long incl = carry + part[threadIdx.x];
    if (i < ng) {
      groups[i] = LightGroup{a - hubs, (e > a ? e : a) - hubs, incl - w, lg, 0};
      wbeg[i] = incl - w;
    }
    carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) wbeg[ng] = carry;
}

// Segment bounds: [seg_min, seg_max] covers every node of the segment and
// every successor of those nodes (atomics, warp-reduced when a warp's nodes
// share a segment).
__global__ void segment_bounds_kernel(const CsrView g, uint64_t lo, uint64_t hi, uint32_t seg_shift,
                                      uint32_t* __restrict__ seg_min,
                                      uint32_t* __restrict__ seg_max) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t first = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (uint64_t base = first - (threadIdx.x & 31); base < hi - lo; base += stride) {
    const uint64_t i = base + (threadIdx.x & 31);
    uint32_t mn = 0xffffffffu, mx = 0;
    uint32_t seg = 0xffffffffu;
    if (i < hi - lo) {
      const uint32_t v = static_cast<uint32_t>(lo + i);
      seg = v >> seg_shift;
      mn = mx = v;
      const uint64_t a = g.begin(v), b = g.end(v);
      for (uint64_t k = a; k < b; ++k) {
        const uint32_t w = g.id(k);
        mn = w < mn ? w : mn;
        mx = w > mx ? w : mx;
      }
    }
    const uint32_t seg0 = __shfl_sync(0xffffffffu, seg, 0);
    if (__all_sync(0xffffffffu, seg == seg0 || seg == 0xffffffffu)) {
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t a = __shfl_down_sync(0xffffffffu, mn, o);
        const uint32_t b = __shfl_down_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
      }
      if ((threadIdx.x & 31) == 0 && seg0 != 0xffffffffu) {
        atomicMin(seg_min + seg0, mn);
        atomicMax(seg_max + seg0, mx);
      }
    } else if (seg != 0xffffffffu) {
      atomicMin(seg_min + seg, mn);
      atomicMax(seg_max + seg, mx);
    }
  }
}

// per-hub chunk counts
__global__ void hub_chunks_kernel(const CsrView g,
                                  const uint32_t* __restrict__ hub_nodes, uint32_t hubs,
                                  uint32_t* __restrict__ chunks) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= hubs) return;
  const uint32_t v = hub_nodes[h];
  const uint64_t d = g.end(v) - g.begin(v);
  chunks[h] = static_cast<uint32_t>((d + kHubChunk - 1) / kHubChunk);
}

// hub chunk tables + their warp tasks (trips) in task slots [0, C)
__global__ void hub_tasks_kernel(const CsrView g,
                                 const uint32_t* __restrict__ hub_nodes, uint32_t hubs,
                                 const uint32_t* __restrict__ hub_first,
                                 const uint32_t* __restrict__ hub_count,
                                 uint32_t* __restrict__ chunk_node, uint32_t* __restrict__ chunk_hub,
                                 uint64_t* __restrict__ chunk_begin, WarpTask* __restrict__ tasks,
                                 uint64_t* __restrict__ trips) {
  const uint32_t h = blockIdx.x;
  if (h >= hubs) return;
  const uint32_t v = hub_nodes[h];
  const uint64_t s = g.begin(v), e = g.end(v);
  for (uint32_t k = threadIdx.x; k < hub_count[h]; k += blockDim.x) {
    const uint32_t c = hub_first[h] + k;
    const uint64_t a = s + static_cast<uint64_t>(k) * kHubChunk;
    const uint64_t len = e - a < kHubChunk ? e - a : kHubChunk;
    chunk_node[c] = v;
    chunk_hub[c] = h;
    chunk_begin[c] = a;
    const uint16_t t = static_cast<uint16_t>((len + 31) / 32);
    tasks[c] = WarpTask{0, c, t, 5, 0};
    trips[c] = t;
  }
}

__global__ void light_tasks_kernel(const CsrView g,
                                   const uint32_t* __restrict__ order,
                                   const LightGroup* __restrict__ groups, uint32_t num_groups,
                                   uint64_t total, uint64_t first_slot,
                                   WarpTask* __restrict__ tasks, uint64_t* __restrict__ trips) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
       w += stride) {
    uint32_t a = 0, b = num_groups - 1;  // last group with warp_begin <= w
    while (a < b) {
      const uint32_t mid = (a + b + 1) / 2;
      if (groups[mid].warp_begin <= w) a = mid; else b = mid - 1;
    }
    const LightGroup gr = groups[a];
    const uint32_t lg = gr.lg;
    const uint32_t per = 32u >> lg;
    const uint64_t item = gr.item_begin + (w - gr.warp_begin) * per;
    const uint64_t rem = gr.item_end - item;
    const uint32_t nodes = static_cast<uint32_t>(rem < per ? rem : per);
    const uint32_t v = order[item];
    const uint64_t d = g.end(v) - g.begin(v);
    const uint32_t G = 1u << lg;
    const uint16_t t = static_cast<uint16_t>((d + G - 1) / G);
    tasks[first_slot + w] = WarpTask{0, static_cast<uint32_t>(item), t, static_cast<uint8_t>(lg),
                                     static_cast<uint8_t>(nodes)};
    trips[first_slot + w] = t;
  }
}

__global__ void set_tos_kernel(WarpTask* __restrict__ tasks, const uint64_t* __restrict__ scan,
                               uint64_t count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < count;
       w += stride)
    tasks[w].tos = scan[w] * 32;
}

// One warp per task writes its TOS rows (padding = zero row) and checks the
// successor ids it copies.
__global__ void __launch_bounds__(256)
fill_tos_kernel(const CsrView g, const uint32_t* __restrict__ order,
                const uint64_t* __restrict__ chunk_begin, const uint32_t* __restrict__ chunk_node,
                const WarpTask* __restrict__ tasks, uint64_t num_tasks, uint32_t n,
                uint32_t limit, uint32_t* __restrict__ tos, int* __restrict__ bad) {
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  bool out_of_range = false;
  for (uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
       w < num_tasks; w += warps) {
    // Row by row: lane l writes entry l of every row (coalesced 128-byte
    // stores, padding included), reading successor i G + sub of its node
    // (a node's G lanes read consecutive arcs; each lane walks its own list)
    const WarpTask t = tasks[w];
    uint32_t* dst = tos + t.tos;
    uint64_t s = 0, d = 0;  // this lane's arcs, and its stride / first index in them
    uint32_t step = 32, first = lane;
    if (t.nodes == 0) {
      s = chunk_begin[t.item];
      const uint64_t e = g.end(chunk_node[t.item]);
      d = e - s < kHubChunk ? e - s : kHubChunk;
    } else {
      const uint32_t j = lane >> t.lg;
      step = 1u << t.lg;
      first = lane & (step - 1);
      if (j < t.nodes) {
        const uint32_t v = order[t.item + j];
        s = g.begin(v);
        d = g.end(v) - s;
      }
    }
    for (uint32_t i = 0; i < t.trips; ++i) {
      const uint64_t k = static_cast<uint64_t>(i) * step + first;
      uint32_t id = n;
      if (k < d) {
        id = g.id(s + k);
        out_of_range |= id >= limit;
        if (id >= limit) id = n;  // (a pipelined sweep may run before the check)
      }
      dst[32 * i + lane] = id;
    }
  }
  if (__any_sync(0xffffffffu, out_of_range) && lane == 0) *bad = 1;
}

template <class T>
cudaError_t pool_alloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1), s);
}

// The build's small device->host reads go through page-locked memory: a
// pageable read queues behind the arcs upload running on the helper stream
// (measured: the whole build then waits for the upload), a pinned one uses
// the other copy engine.  Synchronises `s`.
cudaError_t read_back(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  thread_local void* buf = nullptr;  // (kept for the thread's lifetime)
  thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    const size_t want = bytes < 4096 ? 4096 : bytes;
    const cudaError_t e = cudaHostAlloc(&buf, want, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    cap = want;
  }
  cudaError_t e = cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) std::memcpy(dst, buf, bytes);
  return e;
}

// Host->device counterpart of read_back (a pageable copy would also wait
// for the arcs upload).  Synchronises `s`.
cudaError_t write_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  thread_local void* buf = nullptr;
  thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    const size_t want = bytes < 4096 ? 4096 : bytes;
    const cudaError_t e = cudaHostAlloc(&buf, want, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    cap = want;
  }
  std::memcpy(buf, src, bytes);
  cudaError_t e = cudaMemcpyAsync(dst, buf, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}

}  // namespace

#define HANF_BUILD_TRY(expr)                    \
  do {                                          \
    const cudaError_t _e = (expr);              \
    if (_e != cudaSuccess) return _e;           \
  } while (0)

cudaError_t build_tasks_device(const CsrView& g, uint64_t lo, uint64_t hi, uint64_t n,
                               uint32_t seg_shift, cudaStream_t s, cudaEvent_t succ_ready,
                               TaskBuild* out, int* bad_input, uint64_t* launches,
                               bool seg_bounds, bool class_major, uint64_t id_limit) {
  *out = TaskBuild{};
  if (id_limit == 0) id_limit = n;
  if (seg_shift < 32 && hi > lo) {
    out->seg_shift = seg_shift;
    out->num_segs = static_cast<uint32_t>(((hi - 1) >> seg_shift) + 1);
  }
  const uint32_t segs = out->num_segs;
  *bad_input = 0;
  const uint64_t count = hi - lo;
  const uint32_t threads = 256;
  auto grid = [&](uint64_t items) {
    uint64_t b = (items + threads - 1) / threads;
    if (b > 148ull * 32) b = 148ull * 32;
    return static_cast<uint32_t>(b ? b : 1);
  };
  uint64_t *keys = nullptr, *skeys = nullptr;
  uint32_t *vals = nullptr, *svals = nullptr;
  unsigned long long* counters = nullptr;
  int* d_bad = nullptr;
  HANF_BUILD_TRY(pool_alloc(&keys, count, s));
  HANF_BUILD_TRY(pool_alloc(&vals, count, s));
  HANF_BUILD_TRY(pool_alloc(&skeys, count, s));
  HANF_BUILD_TRY(pool_alloc(&svals, count, s));
  HANF_BUILD_TRY(pool_alloc(&counters, 8, s));
  HANF_BUILD_TRY(pool_alloc(&d_bad, 1, s));
  HANF_BUILD_TRY(cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned long long), s));
  HANF_BUILD_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
  degree_keys_kernel<<<grid(count), threads, 0, s>>>(g, lo, count, out->seg_shift, segs,
                                                     class_major, keys, vals, counters, d_bad);
  ++*launches;
  HANF_BUILD_TRY(cudaGetLastError());
  // key bits: 32 degree bits + the segment prefix (0 for hubs, 1..S for
  // light nodes; degree-0 nodes are all ones, the largest in any width)
  int prefix_bits = 1;
  while ((1ull << prefix_bits) <= 6ull * segs + 1) ++prefix_bits;
  const int end_bit = 32 + prefix_bits;
  size_t temp_bytes = 0;
  HANF_BUILD_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, skeys, vals, svals,
                                                 static_cast<int64_t>(count), 0, end_bit, s));
  void* temp = nullptr;
  HANF_BUILD_TRY(cudaMallocAsync(&temp, temp_bytes ? temp_bytes : 1, s));
  HANF_BUILD_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, skeys, vals, svals,
                                                 static_cast<int64_t>(count), 0, end_bit, s));
  ++*launches;
  HANF_BUILD_TRY(cudaFreeAsync(temp, s));
  unsigned long long h_counts[8] = {};
  HANF_BUILD_TRY(read_back(h_counts, counters, sizeof(h_counts), s));
  const uint64_t hubs = h_counts[0], zeros = h_counts[1];
  const uint64_t light = count - zeros - hubs;
  if (hubs > 0xffffffffull || light > 0xffffffffull) return cudaErrorInvalidValue;

  // group boundaries (sorted order: hubs, then light nodes by group,
  // descending degree within each)
  const uint64_t ng = 6ull * segs;
  unsigned long long* d_bounds = nullptr;
  HANF_BUILD_TRY(pool_alloc(&d_bounds, ng, s));
  group_bounds_kernel<<<static_cast<uint32_t>((ng + 255) / 256), 256, 0, s>>>(
      skeys, hubs, hubs + light, ng, d_bounds);
  ++*launches;
  HANF_BUILD_TRY(cudaGetLastError());
  // the group table is made on the device (a host->device copy would queue
  // behind the arcs upload on the copy engine); the host reads back the
  // warp offsets only
  LightGroup* d_groups = nullptr;
  HANF_BUILD_TRY(pool_alloc(&d_groups, ng, s));
  unsigned long long* d_wbeg = nullptr;
  HANF_BUILD_TRY(pool_alloc(&d_wbeg, ng + 1, s));
  groups_kernel<<<1, 1024, 0, s>>>(d_bounds, ng, hubs, segs, class_major, d_groups, d_wbeg);
  ++*launches;
  HANF_BUILD_TRY(cudaGetLastError());
  std::vector<unsigned long long> wbeg(ng + 1);
  HANF_BUILD_TRY(read_back(wbeg.data(), d_wbeg, sizeof(unsigned long long) * (ng + 1), s));
  HANF_BUILD_TRY(cudaFreeAsync(d_bounds, s));
  HANF_BUILD_TRY(cudaFreeAsync(d_wbeg, s));
  TaskBuild& o = *out;
  o.active_nodes = hubs + light;
  const uint64_t warps = wbeg[ng];
  for (uint64_t i = 0; i < ng; ++i) {
    if (wbeg[i + 1] == wbeg[i]) continue;  // empty group
    o.group_seg.push_back(class_major ? static_cast<uint32_t>(i % segs)
                                      : static_cast<uint32_t>(i / 6));
    o.group_task_begin.push_back(wbeg[i]);
  }
  o.group_task_begin.push_back(warps);

  // hub tables
  o.num_hubs = static_cast<uint32_t>(hubs);
  HANF_BUILD_TRY(pool_alloc(&o.hub_nodes, hubs, s));
  HANF_BUILD_TRY(pool_alloc(&o.hub_first, hubs, s));
  HANF_BUILD_TRY(pool_alloc(&o.hub_count, hubs, s));
  HANF_BUILD_TRY(pool_alloc(&o.hub_ticket, hubs, s));
  HANF_BUILD_TRY(cudaMemsetAsync(o.hub_ticket, 0, sizeof(uint32_t) * (hubs ? hubs : 1), s));
  if (hubs) {
    HANF_BUILD_TRY(cudaMemcpyAsync(o.hub_nodes, svals, sizeof(uint32_t) * hubs,
                                   cudaMemcpyDeviceToDevice, s));
    hub_chunks_kernel<<<static_cast<uint32_t>((hubs + 255) / 256), 256, 0, s>>>(
        g, o.hub_nodes, static_cast<uint32_t>(hubs), o.hub_count);
    ++*launches;
    HANF_BUILD_TRY(cudaGetLastError());
  }
  uint64_t chunks = 0;
  if (hubs) {
    size_t tb = 0;
    HANF_BUILD_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, o.hub_count, o.hub_first,
                                                 static_cast<int64_t>(hubs), s));
    void* t2 = nullptr;
    HANF_BUILD_TRY(cudaMallocAsync(&t2, tb ? tb : 1, s));
    HANF_BUILD_TRY(cub::DeviceScan::ExclusiveSum(t2, tb, o.hub_count, o.hub_first,
                                                 static_cast<int64_t>(hubs), s));
    ++*launches;
    HANF_BUILD_TRY(cudaFreeAsync(t2, s));
    uint32_t last_first = 0, last_count = 0;
    HANF_BUILD_TRY(read_back(&last_first, o.hub_first + hubs - 1, 4, s));
    HANF_BUILD_TRY(read_back(&last_count, o.hub_count + hubs - 1, 4, s));
    chunks = static_cast<uint64_t>(last_first) + last_count;
  }
  const uint64_t num_tasks = chunks + warps;
  if (num_tasks > 0x7fffffffull / 32) return cudaErrorInvalidValue;
  o.num_chunks = static_cast<uint32_t>(chunks);
  o.num_wtasks = static_cast<uint32_t>(num_tasks);
  for (auto& t : o.group_task_begin) t += chunks;  // absolute task slots
  HANF_BUILD_TRY(pool_alloc(&o.chunk_node, chunks, s));
  HANF_BUILD_TRY(pool_alloc(&o.chunk_hub, chunks, s));
  uint64_t* chunk_begin = nullptr;
  HANF_BUILD_TRY(pool_alloc(&chunk_begin, chunks, s));
  HANF_BUILD_TRY(pool_alloc(&o.wtasks, num_tasks, s));
  uint64_t *trips = nullptr, *scan = nullptr;
  HANF_BUILD_TRY(pool_alloc(&trips, num_tasks + 1, s));
  HANF_BUILD_TRY(pool_alloc(&scan, num_tasks + 1, s));
  HANF_BUILD_TRY(pool_alloc(&o.order, light, s));
  if (light)
    HANF_BUILD_TRY(cudaMemcpyAsync(o.order, svals + hubs, sizeof(uint32_t) * light,
                                   cudaMemcpyDeviceToDevice, s));
  if (hubs) {
    hub_tasks_kernel<<<static_cast<uint32_t>(hubs), 128, 0, s>>>(
        g, o.hub_nodes, static_cast<uint32_t>(hubs), o.hub_first, o.hub_count,
        o.chunk_node, o.chunk_hub, chunk_begin, o.wtasks, trips);
    ++*launches;
    HANF_BUILD_TRY(cudaGetLastError());
  }
  if (warps) {
    light_tasks_kernel<<<grid(warps), threads, 0, s>>>(g, o.order, d_groups,
                                                       static_cast<uint32_t>(ng), warps,
                                                       chunks, o.wtasks, trips);
    ++*launches;
    HANF_BUILD_TRY(cudaGetLastError());
  }
  HANF_BUILD_TRY(cudaMemsetAsync(trips + num_tasks, 0, sizeof(uint64_t), s));
  {
    size_t tb = 0;
    HANF_BUILD_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, trips, scan,
                                                 static_cast<int64_t>(num_tasks + 1), s));
    void* t3 = nullptr;
    HANF_BUILD_TRY(cudaMallocAsync(&t3, tb ? tb : 1, s));
    HANF_BUILD_TRY(cub::DeviceScan::ExclusiveSum(t3, tb, trips, scan,
                                                 static_cast<int64_t>(num_tasks + 1), s));
    ++*launches;
    HANF_BUILD_TRY(cudaFreeAsync(t3, s));
  }
  uint64_t rows = 0;
  HANF_BUILD_TRY(read_back(&rows, scan + num_tasks, 8, s));
  if (num_tasks) {
    set_tos_kernel<<<grid(num_tasks), threads, 0, s>>>(o.wtasks, scan, num_tasks);
    ++*launches;
    HANF_BUILD_TRY(cudaGetLastError());
  }
  o.tos_words = rows * 32;
  HANF_BUILD_TRY(pool_alloc(&o.tos, o.tos_words, s));
  if (succ_ready) HANF_BUILD_TRY(cudaStreamWaitEvent(s, succ_ready, 0));
  if (num_tasks) {
    fill_tos_kernel<<<grid(num_tasks * 32), threads, 0, s>>>(
        g, o.order, chunk_begin, o.chunk_node, o.wtasks, num_tasks,
        static_cast<uint32_t>(n), static_cast<uint32_t>(id_limit), o.tos, d_bad);
    ++*launches;
    HANF_BUILD_TRY(cudaGetLastError());
  }
  if (o.seg_shift < 32 && seg_bounds) {
    HANF_BUILD_TRY(pool_alloc(&o.seg_min, segs, s));
    HANF_BUILD_TRY(pool_alloc(&o.seg_max, segs, s));
    HANF_BUILD_TRY(cudaMemsetAsync(o.seg_min, 0xff, sizeof(uint32_t) * segs, s));
    HANF_BUILD_TRY(cudaMemsetAsync(o.seg_max, 0, sizeof(uint32_t) * segs, s));
    segment_bounds_kernel<<<grid(count), threads, 0, s>>>(g, lo, hi, o.seg_shift, o.seg_min,
                                                          o.seg_max);
    ++*launches;
    HANF_BUILD_TRY(cudaGetLastError());
  }
  int h_bad = 0;
  HANF_BUILD_TRY(read_back(&h_bad, d_bad, sizeof(int), s));
  HANF_BUILD_TRY(cudaFreeAsync(keys, s));
  HANF_BUILD_TRY(cudaFreeAsync(vals, s));
  HANF_BUILD_TRY(cudaFreeAsync(skeys, s));
  HANF_BUILD_TRY(cudaFreeAsync(svals, s));
  HANF_BUILD_TRY(cudaFreeAsync(counters, s));
  HANF_BUILD_TRY(cudaFreeAsync(d_bad, s));
  if (chunk_begin) HANF_BUILD_TRY(cudaFreeAsync(chunk_begin, s));
  HANF_BUILD_TRY(cudaFreeAsync(trips, s));
  HANF_BUILD_TRY(cudaFreeAsync(scan, s));
  HANF_BUILD_TRY(cudaFreeAsync(d_groups, s));
  HANF_BUILD_TRY(cudaStreamSynchronize(s));
  *bad_input = h_bad;
  return cudaSuccess;
}

void free_tasks_device(TaskBuild* t, cudaStream_t s) {
  void* ptrs[] = {t->order, t->wtasks, t->tos, t->chunk_node, t->chunk_hub,
                  t->hub_nodes, t->hub_first, t->hub_count, t->hub_ticket,
                  t->seg_min, t->seg_max, t->chunk_begin, t->fill_bad};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, s);
  *t = TaskBuild{};
}

}  // namespace hanf
