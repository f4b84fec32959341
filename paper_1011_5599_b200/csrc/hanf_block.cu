// hanf_block.cu -- source-blocked dense sweeps: the build (BlockSplit,
// hanf_internal.h).
//
// On graphs whose counter array is far larger than L2 (config 5: 10.7 GB)
// a dense union sweep pays one random DRAM line per gather of a cold row.
// A fifth of config 5's arcs go from the 2^20 rows of highest out-degree
// to rows past the L2-resident prefix.  Those sources have enough arcs
// (2 200 on average) that their cold successors can be taken one segment of
// the row space at a time: every (segment, source) pair with such arcs is an
// item, the items of a segment are swept together while the segment's rows
// sit in L2 (each line fetched from DRAM once per segment, not once per
// gather), and an item's maximum is left in an extra row of the counter
// array that the source's list names in place of the item's arcs.  The
// registers computed are the same maxima, taken in another order
// (PackedMax::max_into is commutative and associative, broadword.hpp:94-130).
//
// The build is two passes over the sources' arcs, one CTA per source:
//   count    rows through perm once, kept in `rows`; a shared-memory
//            histogram per source gives the item sizes cnt[segment][source]
//   scatter  cold rows to their item (offsets = exclusive scan of cnt in
//            segment-major order, compacted over the non-empty items), the
//            other rows and the items' ids n + 1 + k to the source's new list
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <cstdint>

#include "hanf_internal.h"

namespace hanf {
namespace {

constexpr int kSplitThreads = 256;
constexpr uint32_t kMaxSegments = 4096;  // shared-memory histogram per CTA

struct Widen {
  __host__ __device__ uint64_t operator()(uint32_t c) const { return c; }
};
struct NonEmpty {
  __host__ __device__ uint32_t operator()(uint32_t c) const { return c ? 1u : 0u; }
};

__global__ void source_degree_kernel(const CsrView g, uint64_t sources,
                                     uint64_t* __restrict__ deg) {
  const uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (u < sources) deg[u] = g.end(u) - g.begin(u);
  if (u == sources) deg[u] = 0;
}

// cnt[seg * sources + u] = arcs of source u into segment seg of the cold
// rows; new_deg[u] = rows < cold + non-empty items; rows[hoff[u] + j] = row
// of arc j.
__global__ void __launch_bounds__(kSplitThreads)
split_count_kernel(const CsrView g, uint64_t sources, uint32_t cold, uint32_t seg_shift,
                   uint32_t segs, const uint64_t* __restrict__ hoff, uint32_t* __restrict__ rows,
                   uint32_t* __restrict__ cnt, uint64_t* __restrict__ new_deg) {
  __shared__ uint32_t hist[kMaxSegments];
  __shared__ uint32_t totals[2];
  for (uint64_t u = blockIdx.x; u < sources; u += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < segs; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x < 2) totals[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t a = g.begin(u), d = g.end(u) - a;
    uint32_t* out = rows + hoff[u];
    uint32_t hot = 0;
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) {
      const uint32_t r = g.id(a + j);
      out[j] = r;
      if (r < cold)
        ++hot;
      else
        atomicAdd(&hist[min((r - cold) >> seg_shift, segs - 1)], 1u);  // (ids were checked at create)
    }
    if (hot) atomicAdd(&totals[0], hot);
    __syncthreads();
    uint32_t mine = 0;
    for (uint32_t i = threadIdx.x; i < segs; i += blockDim.x) {
      const uint32_t c = hist[i];
      cnt[static_cast<uint64_t>(i) * sources + u] = c;
      mine += c != 0;
    }
    if (mine) atomicAdd(&totals[1], mine);
    __syncthreads();
    if (threadIdx.x == 0) new_deg[u] = static_cast<uint64_t>(totals[0]) + totals[1];
    __syncthreads();
  }
}

// item_off[k] = arc offset of the k-th non-empty (segment, source) pair
__global__ void item_offsets_kernel(const uint32_t* __restrict__ cnt,
                                    const uint64_t* __restrict__ arc_scan,
                                    const uint32_t* __restrict__ item_scan, uint64_t cells,
                                    uint64_t* __restrict__ item_off) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i <= cells;
       i += stride) {
    if (i == cells)
      item_off[item_scan[cells]] = arc_scan[cells];
    else if (cnt[i])
      item_off[item_scan[i]] = arc_scan[i];
  }
}

__global__ void __launch_bounds__(kSplitThreads)
split_scatter_kernel(uint64_t sources, uint32_t n, uint32_t cold, uint32_t seg_shift, uint32_t segs,
                     const uint64_t* __restrict__ hoff, const uint32_t* __restrict__ rows,
                     const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ arc_scan,
                     const uint32_t* __restrict__ item_scan, const uint64_t* __restrict__ src_off,
                     uint32_t* __restrict__ item_succ, uint32_t* __restrict__ src_succ) {
  __shared__ uint32_t cursor[kMaxSegments];
  __shared__ uint32_t hot_cursor;
  for (uint64_t u = blockIdx.x; u < sources; u += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < segs; i += blockDim.x) cursor[i] = 0;
    if (threadIdx.x == 0) hot_cursor = 0;
    __syncthreads();
    const uint64_t d = hoff[u + 1] - hoff[u];
    const uint32_t* in = rows + hoff[u];
    uint32_t* mine = src_succ + src_off[u];
    for (uint64_t j = threadIdx.x; j < d; j += blockDim.x) {
      const uint32_t r = in[j];
      if (r < cold) {
        mine[atomicAdd(&hot_cursor, 1u)] = r;
      } else {
        const uint32_t seg = min((r - cold) >> seg_shift, segs - 1);
        const uint64_t cell = static_cast<uint64_t>(seg) * sources + u;
        item_succ[arc_scan[cell] + atomicAdd(&cursor[seg], 1u)] = r;
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < segs; i += blockDim.x) {
      const uint64_t cell = static_cast<uint64_t>(i) * sources + u;
      if (cnt[cell]) mine[atomicAdd(&hot_cursor, 1u)] = n + 1 + item_scan[cell];
    }
    __syncthreads();
  }
}

template <class T>
cudaError_t pool_alloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1), s);
}

template <class In, class Out>
cudaError_t exclusive_sum(In in, Out* out, uint64_t count, cudaStream_t s, uint64_t* launches) {
  size_t tb = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, static_cast<int64_t>(count), s);
  if (e != cudaSuccess) return e;
  void* temp = nullptr;
  e = cudaMallocAsync(&temp, tb ? tb : 1, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(temp, tb, in, out, static_cast<int64_t>(count), s);
  ++*launches;
  cudaFreeAsync(temp, s);
  return e;
}

}  // namespace

#define HANF_BLOCK_TRY(expr)          \
  do {                                \
    const cudaError_t _e = (expr);    \
    if (_e != cudaSuccess) {          \
      free_scratch();                 \
      free_block_split(out, s);       \
      return _e;                      \
    }                                 \
  } while (0)

cudaError_t build_block_split(const CsrView& g, uint64_t n, uint64_t sources, uint64_t cold,
                              uint32_t seg_shift, cudaStream_t s, BlockSplit* out,
                              uint64_t* launches) {
  *out = BlockSplit{};
  uint64_t *deg = nullptr, *hoff = nullptr, *new_deg = nullptr, *arc_scan = nullptr;
  uint32_t *rows = nullptr, *cnt = nullptr, *item_scan = nullptr;
  auto free_scratch = [&] {
    void* ptrs[] = {deg, hoff, new_deg, arc_scan, rows, cnt, item_scan};
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, s);
  };
  if (sources == 0 || sources > n || cold > n || seg_shift > 31 || n + 1 >= 0xffffffffull)
    return cudaErrorInvalidValue;
  const uint64_t segs64 = cold < n ? ((n - cold - 1) >> seg_shift) + 1 : 1;
  if (segs64 > kMaxSegments) return cudaErrorInvalidValue;
  const uint32_t segs = static_cast<uint32_t>(segs64);
  const uint64_t cells = segs64 * sources;

  HANF_BLOCK_TRY(pool_alloc(&deg, sources + 1, s));
  HANF_BLOCK_TRY(pool_alloc(&hoff, sources + 1, s));
  source_degree_kernel<<<static_cast<uint32_t>((sources + 256) / 256), 256, 0, s>>>(g, sources, deg);
  ++*launches;
  HANF_BLOCK_TRY(cudaGetLastError());
  HANF_BLOCK_TRY(exclusive_sum(deg, hoff, sources + 1, s, launches));
  uint64_t hot_arcs = 0;
  HANF_BLOCK_TRY(cudaMemcpyAsync(&hot_arcs, hoff + sources, 8, cudaMemcpyDeviceToHost, s));
  HANF_BLOCK_TRY(cudaStreamSynchronize(s));

  HANF_BLOCK_TRY(pool_alloc(&rows, hot_arcs, s));
  HANF_BLOCK_TRY(pool_alloc(&cnt, cells + 1, s));
  HANF_BLOCK_TRY(pool_alloc(&new_deg, sources + 1, s));
  HANF_BLOCK_TRY(cudaMemsetAsync(cnt + cells, 0, sizeof(uint32_t), s));
  HANF_BLOCK_TRY(cudaMemsetAsync(new_deg + sources, 0, sizeof(uint64_t), s));
  const uint32_t grid = static_cast<uint32_t>(sources < 148ull * 8 ? sources : 148ull * 8);
  split_count_kernel<<<grid, kSplitThreads, 0, s>>>(g, sources, static_cast<uint32_t>(cold),
                                                    seg_shift, segs, hoff, rows, cnt, new_deg);
  ++*launches;
  HANF_BLOCK_TRY(cudaGetLastError());

  // item sizes -> arc offsets and item numbers, segment-major
  HANF_BLOCK_TRY(pool_alloc(&arc_scan, cells + 1, s));
  HANF_BLOCK_TRY(pool_alloc(&item_scan, cells + 1, s));
  HANF_BLOCK_TRY(exclusive_sum(cub::TransformInputIterator<uint64_t, Widen, const uint32_t*>(cnt, Widen{}),
                               arc_scan, cells + 1, s, launches));
  HANF_BLOCK_TRY(exclusive_sum(cub::TransformInputIterator<uint32_t, NonEmpty, const uint32_t*>(cnt, NonEmpty{}),
                               item_scan, cells + 1, s, launches));
  uint32_t items32 = 0;
  HANF_BLOCK_TRY(cudaMemcpyAsync(&out->blocked_arcs, arc_scan + cells, 8, cudaMemcpyDeviceToHost, s));
  HANF_BLOCK_TRY(cudaMemcpyAsync(&items32, item_scan + cells, 4, cudaMemcpyDeviceToHost, s));
  HANF_BLOCK_TRY(exclusive_sum(new_deg, deg, sources + 1, s, launches));  // deg := new offsets
  HANF_BLOCK_TRY(cudaMemcpyAsync(&out->src_arcs, deg + sources, 8, cudaMemcpyDeviceToHost, s));
  HANF_BLOCK_TRY(cudaStreamSynchronize(s));
  out->items = items32;
  if (n + 1 + out->items >= 0xffffffffull) HANF_BLOCK_TRY(cudaErrorInvalidValue);

  HANF_BLOCK_TRY(pool_alloc(&out->item_off, out->items + 1, s));
  HANF_BLOCK_TRY(pool_alloc(&out->item_succ, out->blocked_arcs, s));
  HANF_BLOCK_TRY(pool_alloc(&out->src_succ, out->src_arcs, s));
  out->src_off = deg;
  deg = nullptr;
  item_offsets_kernel<<<148 * 16, 256, 0, s>>>(cnt, arc_scan, item_scan, cells, out->item_off);
  ++*launches;
  HANF_BLOCK_TRY(cudaGetLastError());
  split_scatter_kernel<<<grid, kSplitThreads, 0, s>>>(
      sources, static_cast<uint32_t>(n), static_cast<uint32_t>(cold), seg_shift, segs, hoff, rows,
      cnt, arc_scan, item_scan, out->src_off, out->item_succ, out->src_succ);
  ++*launches;
  HANF_BLOCK_TRY(cudaGetLastError());
  free_scratch();
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) free_block_split(out, s);
  return e;
}
#undef HANF_BLOCK_TRY

void free_block_split(BlockSplit* b, cudaStream_t s) {
  void* ptrs[] = {b->item_off, b->item_succ, b->src_off, b->src_succ};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, s);
  *b = BlockSplit{};
}

}  // namespace hanf
