// hanf_sparse.cu -- the worklist ("systolic") step, engine.hpp:210-224.
//
// Once few counters change per iteration, scanning every arc is wasted: a
// counter can only grow if one of its successors changed in the previous
// iteration.  The sparse step
//   1. lists the counters that changed (the modified bitmap),
//   2. signals their predecessors through the transpose (built once, on the
//      device, from the shard's CSR; graph.hpp:72-84),
//   3. forms the worklist = signalled nodes plus nodes whose next-generation
//      slot is stale (changed last step), and
//   4. recomputes only those, one warp per node, gathering only successors
//      whose modified bit is set (engine.hpp:173).
// The results are bit-identical to the dense sweep (skipping is exact, as
// in the reference: test_engine.cpp:162-184).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <cstdint>

#include "hanf_device.cuh"
#include "hanf_internal.h"

namespace hanf {
namespace {

// ---- transpose (counting sort by destination; row order is irrelevant) ----
__global__ void tr_count_kernel(const uint32_t* __restrict__ succ, uint64_t arcs,
                                unsigned long long* __restrict__ count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < arcs;
       i += stride)
    atomicAdd(count + succ[i], 1ull);
}

__global__ void tr_scatter_kernel(const uint64_t* __restrict__ off, uint64_t lo, uint64_t count,
                                  const uint32_t* __restrict__ succ, uint64_t succ_base,
                                  unsigned long long* __restrict__ cursor,
                                  uint32_t* __restrict__ tr_succ) {
  // one warp per source node
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
       i < count; i += warps) {
    const uint64_t s = off[i], e = off[i + 1];
    for (uint64_t k = s + lane; k < e; k += 32) {
      const uint32_t w = succ[k - succ_base];
      const unsigned long long pos = atomicAdd(cursor + w, 1ull);
      tr_succ[pos] = static_cast<uint32_t>(lo + i);
    }
  }
}

// ---- worklist -------------------------------------------------------------
// Modified nodes as signal tasks: one entry per kSignalChunk predecessors,
// so a node with a huge in-degree is spread over many warps.
__global__ void modified_chunks_kernel(const uint64_t* __restrict__ bits, uint64_t words,
                                       uint64_t n, const unsigned long long* __restrict__ tr_off,
                                       unsigned long long* __restrict__ list,
                                       unsigned int* __restrict__ len) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
       w += stride) {
    uint64_t word = bits[w];
    if (!word) continue;
    unsigned int total = 0;
    for (uint64_t x = word; x; x &= x - 1) {
      const uint64_t v = (w << 6) + (__ffsll(static_cast<long long>(x)) - 1);
      if (v < n)
        total += static_cast<unsigned int>((tr_off[v + 1] - tr_off[v] + kSignalChunk - 1) /
                                           kSignalChunk);
    }
    if (!total) continue;
    unsigned int pos = atomicAdd(len, total);
    for (; word; word &= word - 1) {
      const uint64_t v = (w << 6) + (__ffsll(static_cast<long long>(word)) - 1);
      if (v >= n) continue;
      const uint64_t c = (tr_off[v + 1] - tr_off[v] + kSignalChunk - 1) / kSignalChunk;
      for (uint64_t k = 0; k < c; ++k) list[pos++] = (v << 32) | k;
    }
  }
}

// signalled[pred] = 1 for the predecessors (in this shard) of each listed
// chunk; the 8 ids per lane are loaded before any atomic is issued
__global__ void signal_kernel(const unsigned long long* __restrict__ list,
                              const unsigned int* __restrict__ len,
                              const unsigned long long* __restrict__ tr_off,
                              const uint32_t* __restrict__ tr_succ, uint64_t* __restrict__ sig) {
  constexpr int kPer = kSignalChunk / 32;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const unsigned int m = *len;
  for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < m;
       i += warps) {
    const unsigned long long e = list[i];
    const uint32_t u = static_cast<uint32_t>(e >> 32);
    const uint64_t s = tr_off[u] + (e & 0xffffffffull) * kSignalChunk;
    const uint64_t t = tr_off[u + 1];
    uint32_t p[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint64_t k = s + lane + 32 * j;
      p[j] = k < t ? tr_succ[k] : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (p[j] != 0xffffffffu)
        atomicOr(reinterpret_cast<unsigned long long*>(sig) + (p[j] >> 6), 1ull << (p[j] & 63));
  }
}

// worklist = signalled | stale over this shard's words: hubs contribute all
// their chunk tasks (run by the dense kernel), other nodes a worklist entry
__global__ void worklist_kernel(const uint64_t* __restrict__ sig, const uint64_t* __restrict__ stale,
                                uint64_t w0, uint64_t w1, uint64_t hi,
                                const uint32_t* __restrict__ hub_index,
                                const uint32_t* __restrict__ hub_first,
                                const uint32_t* __restrict__ hub_count,
                                uint32_t* __restrict__ work, uint32_t* __restrict__ hub_tasks,
                                unsigned int* __restrict__ lens) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = w0 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < w1;
       w += stride) {
    uint64_t word = sig[w] | stale[w];
    const uint64_t first = w << 6;
    if (first + 64 > hi) word &= hi > first ? (~0ull >> (first + 64 - hi)) : 0ull;
    if (!word) continue;
    unsigned int light = 0, chunks = 0;
    for (uint64_t x = word; x; x &= x - 1) {
      const uint32_t v = static_cast<uint32_t>(first + __ffsll(static_cast<long long>(x)) - 1);
      const uint32_t h = hub_index[v];
      if (h == 0xffffffffu) ++light; else chunks += hub_count[h];
    }
    unsigned int pl = light ? atomicAdd(lens + 1, light) : 0;
    unsigned int ph = chunks ? atomicAdd(lens + 2, chunks) : 0;
    for (; word; word &= word - 1) {
      const uint32_t v = static_cast<uint32_t>(first + __ffsll(static_cast<long long>(word)) - 1);
      const uint32_t h = hub_index[v];
      if (h == 0xffffffffu) {
        work[pl++] = v;
      } else {
        for (uint32_t k = 0; k < hub_count[h]; ++k) hub_tasks[ph++] = hub_first[h] + k;
      }
    }
  }
}

__global__ void hub_index_kernel(const uint32_t* __restrict__ hub_nodes, uint32_t hubs,
                                 uint32_t* __restrict__ index) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < hubs) index[hub_nodes[h]] = h;
}

// ---- sparse union: one warp per worklist node -----------------------------
template <class Lay, bool kVec16>
__global__ void __launch_bounds__(256) sparse_union_kernel(const SparseArgs a) {
  constexpr int NL = Lay::kLimbs;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const unsigned int m = *a.work_len;
  const uint32_t words = a.pitch;
  const uint32_t zero_row = static_cast<uint32_t>(a.n);
  for (uint64_t i = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; i < m;
       i += warps) {
    const uint32_t v = a.work[i];
    HANF_DCHECK(v >= a.node_base && v < a.hi);
    const uint64_t s = a.off[v - a.node_base], e = a.off[v - a.node_base + 1];
    HANF_DCHECK(s <= e && e - s <= kHubDegree);
    uint32_t acc[NL];
    if (lane == 0)
      load_chunk<Lay, kVec16>(acc, a.cur + static_cast<uint64_t>(v) * words);
    else
      sfor<0, NL>([&](auto I) { acc[decltype(I)::value] = 0u; });
    // out-degree <= kHubDegree here (hubs run as dense chunk tasks): at
    // most 32 successors per lane, ids and bitmap probes loaded 4 at a time
    for (uint64_t k0 = s + lane; k0 < e; k0 += 128) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t k = k0 + 32 * j;
        w[j] = k < e ? a.succ[k - a.succ_base] : zero_row;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        HANF_DCHECK(w[j] <= zero_row);
        if (!((__ldg(a.mod_cur + (w[j] >> 6)) >> (w[j] & 63)) & 1)) w[j] = zero_row;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (w[j] != zero_row) {
          uint32_t y[NL];
          load_chunk<Lay, kVec16>(y, a.cur + static_cast<uint64_t>(w[j]) * words);
          swar_max<Lay>(acc, y);
        }
      }
    }
    for (uint32_t off = 16; off >= 1; off >>= 1) shfl_max<Lay>(acc, off);
    if (lane == 0) {
      uint32_t own[NL];
      load_chunk<Lay, kVec16>(own, a.cur + static_cast<uint64_t>(v) * words);
      const bool changed = limbs_differ<Lay>(acc, own);
      const bool stale = (a.mod_cur[v >> 6] >> (v & 63)) & 1;
      if (changed || stale) {
        const uint64_t off = static_cast<uint64_t>(v) * words;
        store_chunk<Lay, kVec16>(a.next + off, acc);
        for (uint32_t p = 0; p < a.peers.count; ++p)  // sharded peer-push
          if (peer_wants(a.peers, p, v)) store_chunk<Lay, kVec16>(a.peers.next[p] + off, acc);
      }
      if (changed) {
        a.est[a.est_index ? a.est_index[v] : v] = estimate_limbs<Lay>(acc, a.ep);
        atomicOr(reinterpret_cast<unsigned long long*>(a.mod_next) + (v >> 6), 1ull << (v & 63));
        if (a.dirty_next) {
          const uint32_t o = a.orig_of[v];
          atomicOr(reinterpret_cast<unsigned long long*>(a.dirty_next) + (o >> 6), 1ull << (o & 63));
        }
      }
    }
  }
}

template <int R, int NREG, bool V>
cudaError_t sparse_launch(const SparseArgs& a, uint32_t blocks, cudaStream_t s) {
  sparse_union_kernel<Layout<R, NREG>, V><<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}
template <int M>
cudaError_t sparse_launch_bytes(const SparseArgs& a, uint32_t blocks, cudaStream_t s) {
  sparse_union_kernel<ByteLayout<M>, true><<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t build_transpose_device(const uint64_t* d_off, const uint32_t* d_succ, uint64_t lo,
                                   uint64_t hi, uint64_t succ_base, uint64_t n, cudaStream_t s,
                                   unsigned long long** tr_off, uint32_t** tr_succ,
                                   uint64_t* launches) {
  const uint64_t count = hi - lo;
  uint64_t arcs = 0;
  if (count) {
    uint64_t first = 0, last = 0;
    cudaError_t e = cudaMemcpyAsync(&first, d_off, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last, d_off + count, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    arcs = last - first;
  }
  unsigned long long* cnt = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&cnt), sizeof(unsigned long long) * (n + 1), s);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync(reinterpret_cast<void**>(tr_off), sizeof(unsigned long long) * (n + 1), s);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync(reinterpret_cast<void**>(tr_succ), sizeof(uint32_t) * (arcs ? arcs : 1), s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (n + 1), s);
  if (arcs) {
    const uint32_t blocks = 148 * 16;
    tr_count_kernel<<<blocks, 256, 0, s>>>(d_succ, arcs, cnt);
    ++*launches;
  }
  size_t tb = 0;
  e = cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, *tr_off, static_cast<int64_t>(n + 1), s);
  if (e != cudaSuccess) return e;
  void* temp = nullptr;
  e = cudaMallocAsync(&temp, tb ? tb : 1, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt, *tr_off, static_cast<int64_t>(n + 1), s);
  if (e != cudaSuccess) return e;
  ++*launches;
  cudaFreeAsync(temp, s);
  // cursor = tr_off (copy), then scatter
  e = cudaMemcpyAsync(cnt, *tr_off, sizeof(unsigned long long) * (n + 1), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  if (arcs) {
    tr_scatter_kernel<<<148 * 16, 256, 0, s>>>(d_off, lo, count, d_succ, succ_base, cnt, *tr_succ);
    ++*launches;
  }
  cudaFreeAsync(cnt, s);
  return cudaGetLastError();
}

// Stages 3-4 of the worklist step: the worklist from sig | stale, then the
// sparse union (hubs go to the dense kernel through hub_tasks, by the caller)
cudaError_t sparse_tail_stages(const SparseArgs& a, uint64_t w0, uint64_t w1,
                               uint32_t register_bits, uint32_t registers, cudaStream_t s,
                               uint64_t* launches);

cudaError_t launch_sparse_step(const SparseArgs& a, uint64_t w0, uint64_t w1, uint32_t register_bits,
                               uint32_t registers, cudaStream_t s, uint64_t* launches) {
  const uint32_t blocks = 148 * 8;
  cudaError_t e = cudaMemsetAsync(a.lens, 0, 3 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  // modified chunks (whole bitmap: successors anywhere signal this shard)
  modified_chunks_kernel<<<blocks, 256, 0, s>>>(a.mod_cur, a.blocks, a.n, a.tr_off, a.mod_list,
                                               a.lens);
  ++*launches;
  e = cudaMemsetAsync(a.sig + w0, 0, sizeof(uint64_t) * (w1 - w0), s);
  if (e != cudaSuccess) return e;
  signal_kernel<<<blocks, 256, 0, s>>>(a.mod_list, a.lens, a.tr_off, a.tr_succ, a.sig);
  ++*launches;
  return sparse_tail_stages(a, w0, w1, register_bits, registers, s, launches);
}

cudaError_t sparse_tail_stages(const SparseArgs& a, uint64_t w0, uint64_t w1,
                               uint32_t register_bits, uint32_t registers, cudaStream_t s,
                               uint64_t* launches) {
  const uint32_t blocks = 148 * 8;
  worklist_kernel<<<blocks, 256, 0, s>>>(a.sig, a.mod_cur, w0, w1, a.hi, a.hub_index, a.hub_first,
                                         a.hub_count, a.work, a.hub_tasks, a.lens);
  ++*launches;
  SparseArgs b = a;
  b.work_len = a.lens + 1;
  ++*launches;
  if (b.bytes) switch (registers) {
      case 16: return sparse_launch_bytes<16>(b, blocks, s);
      case 32: return sparse_launch_bytes<32>(b, blocks, s);
      case 64: return sparse_launch_bytes<64>(b, blocks, s);
      case 128: return sparse_launch_bytes<128>(b, blocks, s);
      default: return cudaErrorInvalidValue;
    }
  switch (register_bits * 1000 + registers) {
    case 5032: return sparse_launch<5, 32, false>(b, blocks, s);
    case 5064: return sparse_launch<5, 64, false>(b, blocks, s);
    case 5128: return sparse_launch<5, 128, true>(b, blocks, s);
    case 5016: return sparse_launch<5, 16, true>(b, blocks, s);
    case 6016: return sparse_launch<6, 16, true>(b, blocks, s);
    case 6032: return sparse_launch<6, 32, false>(b, blocks, s);
    case 7016: return sparse_launch<7, 16, true>(b, blocks, s);
    case 7032: return sparse_launch<7, 32, true>(b, blocks, s);
    case 7064: return sparse_launch<7, 64, false>(b, blocks, s);
    case 8016: return sparse_launch<8, 16, true>(b, blocks, s);
    default: return cudaErrorInvalidValue;  // multi-chunk layouts use the dense sweep
  }
}

// ---- changed-rows exchange (hanf_shard_pack / hanf_shard_unpack) ----------
// rows of [lo, hi) that the step wrote (changed now, or stale = changed by the
// previous step): ids appended in any order
__global__ void pack_ids_kernel(const uint64_t* __restrict__ mod_next,
                                const uint64_t* __restrict__ mod_cur, uint64_t lo, uint64_t hi,
                                uint32_t* __restrict__ ids, unsigned long long cap,
                                unsigned long long* __restrict__ count) {
  const uint64_t w0 = lo >> 6, w1 = (hi + 63) >> 6;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = w0 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < w1;
       w += stride) {
    uint64_t word = mod_next[w] | mod_cur[w];
    const uint64_t first = w << 6;
    if (first < lo) word &= ~0ull << (lo - first);
    if (first + 64 > hi) word &= hi > first ? (~0ull >> (first + 64 - hi)) : 0ull;
    if (!word) continue;
    unsigned long long pos = atomicAdd(count, static_cast<unsigned long long>(__popcll(word)));
    for (; word; word &= word - 1, ++pos)
      if (pos < cap) ids[pos] = static_cast<uint32_t>(first + __ffsll(static_cast<long long>(word)) - 1);
  }
}

// rows[i] <-> counters[ids[i]] (pitch words each); ids past n are padding
__global__ void move_rows_kernel(const uint32_t* __restrict__ ids, uint64_t count, uint64_t n,
                                 uint32_t pitch, const uint64_t* __restrict__ src, bool gather,
                                 uint64_t* __restrict__ dst) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       k < count * pitch; k += stride) {
    const uint64_t i = k / pitch, w = k % pitch;
    const uint64_t id = ids[i];
    if (id >= n) continue;
    if (gather)
      dst[k] = src[id * pitch + w];
    else
      dst[id * pitch + w] = src[k];
  }
}

cudaError_t launch_pack_rows(const uint64_t* mod_next, const uint64_t* mod_cur, uint64_t lo,
                             uint64_t hi, const uint64_t* counters, uint32_t pitch, uint32_t* ids,
                             uint64_t* rows, uint64_t cap, unsigned long long* d_count,
                             uint64_t* count, cudaStream_t s, uint64_t* launches) {
  cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const uint64_t words = ((hi + 63) >> 6) - (lo >> 6);
  if (words) {
    pack_ids_kernel<<<static_cast<uint32_t>((words + 255) / 256), 256, 0, s>>>(
        mod_next, mod_cur, lo, hi, ids, cap, d_count);
    ++*launches;
  }
  unsigned long long h = 0;
  e = cudaMemcpyAsync(&h, d_count, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *count = h;
  if (h == 0 || h > cap) return cudaGetLastError();
  uint64_t blocks = (h * pitch + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  move_rows_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(ids, h, ~0ull, pitch, counters,
                                                                 true, rows);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_unpack_rows(const uint32_t* ids, const uint64_t* rows, uint64_t count, uint64_t n,
                               uint32_t pitch, uint64_t* counters, cudaStream_t s,
                               uint64_t* launches) {
  if (count == 0) return cudaSuccess;
  uint64_t blocks = (count * pitch + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  move_rows_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(ids, count, n, pitch, rows, false,
                                                                 counters);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t build_hub_index(const uint32_t* hub_nodes, uint32_t hubs, uint64_t n, cudaStream_t s,
                            uint32_t** out, uint64_t* launches) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), sizeof(uint32_t) * (n ? n : 1), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(*out, 0xff, sizeof(uint32_t) * (n ? n : 1), s);
  if (e != cudaSuccess) return e;
  if (hubs) {
    hub_index_kernel<<<(hubs + 255) / 256, 256, 0, s>>>(hub_nodes, hubs, *out);
    ++*launches;
  }
  return cudaGetLastError();
}

bool sparse_supported(uint32_t register_bits, uint32_t registers) {
  switch (register_bits * 1000 + registers) {
    case 5032: case 5064: case 5128: case 5016: case 6016: case 6032:
    case 7016: case 7032: case 7064: case 8016:
      return true;
    default:
      return false;
  }
}

}  // namespace hanf
