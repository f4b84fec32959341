// hanf_batch.cu -- K independent HyperANF runs in one engine (SURVEY 8(f)
// item 2, the reference's multirun: main.cpp:263-283 runs estimate_nf for
// seeds base + i).
//
// The graph is lifted to K copies: node v of run k is row v*K + k and its
// successors are the rows w*K + k.  Every kernel of the single-run engine
// then runs unchanged on the lifted graph, and the layout does the work:
// run k's counter of w sits next to the other runs' counters of w, the K
// rows of a node have equal degree and land in adjacent lanes of the same
// warp (the task sort is stable in id), so one trip of those K lanes reads
// K consecutive rows - one coalesced segment instead of K scattered ones.
//
// Only the sums differ: run k's N(t) is the sum, in the reference's order,
// of its own 64-node blocks, i.e. rows (64b + i)*K + k (finish_batch_kernel).
#include <cuda_runtime.h>

#include <cstdint>

#include "hanf_internal.h"

namespace hanf {
namespace {

__global__ void lift_offsets_kernel(const uint64_t* __restrict__ off, uint64_t n, uint32_t K,
                                    uint64_t* __restrict__ voff) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v <= n;
       v += stride) {
    if (v == n) {
      voff[n * K] = off[n] * K;
      continue;
    }
    const uint64_t a = off[v], b = off[v + 1];
    const uint64_t d = b >= a ? b - a : 0;  // malformed rows are flagged by the task build
    for (uint32_t k = 0; k < K; ++k) voff[v * K + k] = a * K + k * d;
  }
}

// warp per real node: successor j of run k is w*K + k
__global__ void lift_arcs_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ succ,
                                 uint64_t n, uint32_t K, const uint64_t* __restrict__ voff,
                                 uint32_t* __restrict__ vsucc) {
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t v = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; v < n;
       v += warps) {
    const uint64_t a = off[v], b = off[v + 1];
    if (b <= a) continue;
    const uint64_t d = b - a;
    for (uint64_t j = lane; j < d; j += 32) {
      const uint32_t w = succ[a + j];
      // out-of-range ids stay out of range (the task build flags them)
      const uint64_t lw = w < n ? static_cast<uint64_t>(w) * K : 0xffffffffull;
      for (uint32_t k = 0; k < K; ++k)
        vsucc[voff[v * K + k] + j] = static_cast<uint32_t>(lw == 0xffffffffull ? lw : lw + k);
    }
  }
}

// Thread per real 64-node block b: for each run k, the dirty flag and the
// modified count come from the K bitmap words of rows [64bK, 64(b+1)K)
// masked to run k's bit positions; a dirty block's sum is redone
// sequentially over rows (64b + i)*K + k (engine.hpp:109-111).
__global__ void finish_batch_kernel(const double* __restrict__ est,
                                    const uint64_t* __restrict__ bits, uint64_t n_real,
                                    uint32_t K, uint64_t blocks, bool recompute,
                                    double* __restrict__ block_sums,
                                    unsigned long long* __restrict__ counts) {
  const uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t k = 0; k < K; ++k) {
    unsigned long long cnt = 0;
    if (b < blocks) {
      // run k's positions inside a word: p % K == k (K divides 64)
      uint64_t mask = 0;
      for (uint32_t p = k; p < 64; p += K) mask |= 1ull << p;
      uint64_t any = 0;
      const uint64_t words = (n_real * K + 63) / 64;  // the bitmap's length
      for (uint32_t j = 0; j < K && b * K + j < words; ++j) {
        const uint64_t w = bits[b * K + j] & mask;
        any |= w;
        cnt += __popcll(w);
      }
      if (recompute && any) {
        const uint64_t first = b * 64;
        const uint32_t last = n_real - first < 64 ? static_cast<uint32_t>(n_real - first) : 64u;
        double s = 0.0;
        for (uint32_t i = 0; i < last; ++i) s = __dadd_rn(s, est[(first + i) * K + k]);
        block_sums[k * blocks + b] = s;
      }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(counts + k, cnt);
  }
}

}  // namespace

cudaError_t lift_graph_device(const uint64_t* d_off, const uint32_t* d_succ, uint64_t n, uint64_t arcs,
                              uint32_t K, cudaStream_t s, uint64_t** voff, uint32_t** vsucc,
                              uint64_t* launches) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(voff), sizeof(uint64_t) * (n * K + 1), s);
  if (e != cudaSuccess) return e;
  e = cudaMallocAsync(reinterpret_cast<void**>(vsucc), sizeof(uint32_t) * (arcs * K ? arcs * K : 1), s);
  if (e != cudaSuccess) return e;
  uint64_t blocks = (n + 256) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  lift_offsets_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(d_off, n, K, *voff);
  ++*launches;
  if (n && arcs) {
    uint64_t ctas = (n + 7) / 8;
    if (ctas > 148ull * 16) ctas = 148ull * 16;
    lift_arcs_kernel<<<static_cast<uint32_t>(ctas), 256, 0, s>>>(d_off, d_succ, n, K, *voff, *vsucc);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_finish_batch(const double* est, const uint64_t* bits, uint64_t n_real, uint32_t K,
                                bool recompute, double* block_sums, unsigned long long* counts,
                                cudaStream_t s, uint64_t* launches) {
  const uint64_t blocks = (n_real + 63) / 64;
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * K, s);
  if (e != cudaSuccess || blocks == 0) return e;
  finish_batch_kernel<<<static_cast<uint32_t>((blocks + 127) / 128), 128, 0, s>>>(
      est, bits, n_real, K, blocks, recompute, block_sums, counts);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace hanf
