// hanf_exact.cu -- exact neighbourhood function on the device (SURVEY 8(f)
// item 4; the reference's all-pairs BFS, oracle.hpp:38-104).
//
// The exact balls obey the same recurrence as the HyperANF counters, with
// sets instead of sketches: B(x, t+1) = {x} u U_{w in succ(x)} B(x_w, t).
// Targets are processed in batches of S = 64 K bits: row x of a batch is
// the bitset B(x, t) restricted to the batch, the union over successors
// is a word-wise OR (warp per node, lane j owns word j of every row, so a
// successor row is one coalesced load), and the batch's contribution to
// N(t) is the popcount of all rows.  A batch stops at its first iteration
// without a change; N(t) = sum over batches of their count at min(t, depth).
// Work ~ (n / 64) * iterations * arcs word ORs, memory 2 * n * S / 8 bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hanf.h"
#include "hanf_graph_internal.h"

namespace {

constexpr uint32_t kBatchWords = 32;  // S = 2048 targets per batch

// B(x, 0) = {x} restricted to targets [t0, t0 + 64 * words)
__global__ void exact_init_kernel(uint64_t* __restrict__ rows, uint64_t n, uint64_t t0,
                                  uint32_t words) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       k < n * words; k += stride) {
    const uint64_t x = k / words, j = k % words;
    uint64_t w = 0;
    if (x >= t0 && x < t0 + 64ull * words && (x - t0) / 64 == j) w = 1ull << ((x - t0) % 64);
    rows[k] = w;
  }
}

// next[x] = cur[x] | OR cur[succ]; counts popcounts and changed rows
__global__ void __launch_bounds__(256) exact_step_kernel(
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ succ, uint64_t n,
    uint32_t words, const uint64_t* __restrict__ cur, uint64_t* __restrict__ next,
    unsigned long long* __restrict__ out /* [0] popcount, [1] changed rows */) {
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long pop = 0, changed = 0;
  for (uint64_t x = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; x < n;
       x += warps) {
    const uint64_t own = lane < words ? cur[x * words + lane] : 0;
    uint64_t acc = own;
    const uint64_t s = off[x], e = off[x + 1];
    if (lane < words)
      for (uint64_t k = s; k < e; ++k) acc |= __ldg(cur + static_cast<uint64_t>(succ[k]) * words + lane);
    if (lane < words) next[x * words + lane] = acc;
    pop += __popcll(acc);
    if (__any_sync(0xffffffffu, acc != own) && lane == 0) ++changed;
  }
  for (int o = 16; o > 0; o >>= 1) {
    pop += __shfl_down_sync(0xffffffffu, pop, o);
    changed += __shfl_down_sync(0xffffffffu, changed, o);
  }
  if (lane == 0) {
    if (pop) atomicAdd(out + 0, pop);
    if (changed) atomicAdd(out + 1, changed);
  }
}

hanf_status fail(hanf_status st, const std::string& msg) {
  hanf_host_detail::set_error(msg);
  return st;
}
hanf_status cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? HANF_OUT_OF_MEMORY : HANF_CUDA_ERROR,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define EX_TRY(expr)                                    \
  do {                                                  \
    const cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

}  // namespace

extern "C" {

hanf_status hanf_exact_nf(const hanf_graph_view* g, int32_t device, uint64_t max_nodes,
                          uint64_t max_work, uint64_t* values, uint64_t cap, uint64_t* len) {
  if (!g || !len || (cap && !values)) return fail(HANF_INVALID_ARGUMENT, "null argument");
  const uint64_t n = g->n, a = g->num_arcs;
  if (n > max_nodes)
    return fail(HANF_GUARD, "exact nf: node count exceeds guard (" + std::to_string(n) + " > " +
                                std::to_string(max_nodes) + ")");
  if (n > 0 && a > max_work / n) return fail(HANF_GUARD, "exact nf: n * arcs exceeds guard");
  if (n == 0) {
    *len = 1;
    if (cap < 1) return HANF_CAPACITY;
    values[0] = 0;
    return HANF_OK;
  }
  if (!g->offsets || (a && !g->arcs)) return fail(HANF_INVALID_ARGUMENT, "null graph arrays");
  if (g->offsets[0] != 0 || g->offsets[n] != a)
    return fail(HANF_INVALID_ARGUMENT, "offsets must run from 0 to the arc count");
  for (uint64_t v = 0; v < n; ++v)
    if (g->offsets[v + 1] < g->offsets[v])
      return fail(HANF_INVALID_ARGUMENT, "offsets not non-decreasing");
  for (uint64_t i = 0; i < a; ++i)
    if (g->arcs[i] >= n) return fail(HANF_INVALID_ARGUMENT, "arc endpoint out of range");

  EX_TRY(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  EX_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct Res {
    cudaStream_t s;
    uint64_t* off = nullptr;
    uint32_t* succ = nullptr;
    uint64_t* rows[2] = {nullptr, nullptr};
    unsigned long long* out = nullptr;
    ~Res() {
      cudaFreeAsync(off, s);
      cudaFreeAsync(succ, s);
      cudaFreeAsync(rows[0], s);
      cudaFreeAsync(rows[1], s);
      cudaFreeAsync(out, s);
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } r{s};
  const uint64_t batches = (n + 64ull * kBatchWords - 1) / (64ull * kBatchWords);
  const uint32_t words = static_cast<uint32_t>(
      std::min<uint64_t>(kBatchWords, (n + 63) / 64));  // small graphs: one narrower batch
  EX_TRY(cudaMallocAsync(reinterpret_cast<void**>(&r.off), sizeof(uint64_t) * (n + 1), s));
  EX_TRY(cudaMallocAsync(reinterpret_cast<void**>(&r.succ), sizeof(uint32_t) * (a ? a : 1), s));
  EX_TRY(cudaMallocAsync(reinterpret_cast<void**>(&r.rows[0]), sizeof(uint64_t) * n * words, s));
  EX_TRY(cudaMallocAsync(reinterpret_cast<void**>(&r.rows[1]), sizeof(uint64_t) * n * words, s));
  EX_TRY(cudaMallocAsync(reinterpret_cast<void**>(&r.out), 2 * sizeof(unsigned long long), s));
  EX_TRY(cudaMemcpyAsync(r.off, g->offsets, sizeof(uint64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  if (a) EX_TRY(cudaMemcpyAsync(r.succ, g->arcs, sizeof(uint32_t) * a, cudaMemcpyHostToDevice, s));

  const uint64_t init_blocks = std::min<uint64_t>((n * words + 255) / 256, 148ull * 64);
  const uint64_t step_blocks = std::min<uint64_t>((n + 7) / 8, 148ull * 32);
  std::vector<uint64_t> total;  // N(t) over the batches done so far
  for (uint64_t bt = 0; bt < batches; ++bt) {
    const uint64_t t0 = bt * 64ull * words;
    exact_init_kernel<<<static_cast<uint32_t>(init_blocks), 256, 0, s>>>(r.rows[0], n, t0, words);
    EX_TRY(cudaGetLastError());
    std::vector<uint64_t> series{std::min<uint64_t>(64ull * words, n - t0)};  // t = 0
    int c = 0;
    for (;;) {
      unsigned long long h[2] = {0, 0};
      EX_TRY(cudaMemsetAsync(r.out, 0, sizeof h, s));
      exact_step_kernel<<<static_cast<uint32_t>(step_blocks), 256, 0, s>>>(
          r.off, r.succ, n, words, r.rows[c], r.rows[1 - c], r.out);
      EX_TRY(cudaGetLastError());
      EX_TRY(cudaMemcpyAsync(h, r.out, sizeof h, cudaMemcpyDeviceToHost, s));
      EX_TRY(cudaStreamSynchronize(s));
      if (h[1] == 0) break;  // no ball grew: this batch is complete
      series.push_back(h[0]);
      c = 1 - c;
    }
    // N(t) += this batch's count at min(t, depth); extend the earlier
    // batches' totals with their final values
    const uint64_t old_len = total.size();
    const uint64_t len_now = std::max<uint64_t>(old_len, series.size());
    const uint64_t old_last = old_len ? total.back() : 0;
    total.resize(len_now, old_last);
    for (uint64_t t = 0; t < len_now; ++t) total[t] += series[std::min<uint64_t>(t, series.size() - 1)];
  }
  *len = total.size();
  if (total.size() > cap) return HANF_CAPACITY;
  std::copy(total.begin(), total.end(), values);
  return HANF_OK;
}

}  // extern "C"
