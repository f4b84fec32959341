// hanf_graphgen.cu -- graph construction on the device:
// Graph::from_edges (graph.hpp:29-44) and the R-MAT generator of BASELINE
// configs 2 and 5, as device radix sorts instead of host counting sorts.
//
//   1. every arc becomes one 64-bit key (source << 32 | target); R-MAT draws
//      are generated in place from the shared counter-based stream
//      (hanf_rng.h), so the graph is the host generator's bit for bit;
//   2. CUB radix sort over the key bits that can be set;
//   3. CUB unique: sorted rows without duplicate arcs (graph.hpp:38-41);
//   4. offsets from the row boundaries (one thread per key fills the
//      offsets of the rows that end there), targets = low words.
// Dropped self-loops (R-MAT only) become one sentinel key past every row.
// The CSR is copied into a host hanf_graph: the engine API takes host
// graphs (hanf_create uploads them again).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <cstdint>
#include <new>
#include <string>

#include "../../include/hanf.h"
#include "hanf_graph_internal.h"
#include "hanf_rng.h"

namespace {

__global__ void edge_keys_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                 uint64_t count, uint64_t n, uint64_t* __restrict__ keys,
                                 int* __restrict__ bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  bool oob = false;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += stride) {
    const uint32_t s = src[i], d = dst[i];
    oob |= s >= n || d >= n;
    keys[i] = (static_cast<uint64_t>(s) << 32) | d;
  }
  if (oob) *bad = 1;
}

__global__ void rmat_keys_kernel(uint64_t draws, uint32_t scale, uint32_t ta, uint32_t tb,
                                 uint32_t tc, uint64_t seed, hanf_rng::Feistel perm,
                                 uint64_t sentinel, uint64_t* __restrict__ keys) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < draws;
       i += stride) {
    uint64_t u = 0, v = 0;
    hanf_rng::rmat_draw(seed, i, scale, ta, tb, tc, &u, &v);
    const uint64_t pu = perm(u), pv = perm(v);
    keys[i] = pu == pv ? sentinel : (pu << 32) | pv;  // self-loops dropped
  }
}

// offsets[r] = first key index of row r; key i fills the rows in
// (row of key i-1, row of key i]; rows past the last key get m.
__global__ void row_offsets_kernel(const uint64_t* __restrict__ keys, uint64_t m, uint64_t n,
                                   uint64_t* __restrict__ off) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i <= m;
       i += stride) {
    const uint64_t hi = i < m ? keys[i] >> 32 : n;
    const uint64_t lo = i > 0 ? (keys[i - 1] >> 32) + 1 : 0;
    for (uint64_t r = lo; r <= hi; ++r) off[r] = i;
  }
}

__global__ void low_words_kernel(const uint64_t* __restrict__ keys, uint64_t m,
                                 uint32_t* __restrict__ arcs) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += stride)
    arcs[i] = static_cast<uint32_t>(keys[i]);
}

uint32_t grid_for(uint64_t items) {
  const uint64_t b = (items + 255) / 256;
  return static_cast<uint32_t>(b < 148ull * 64 ? (b ? b : 1) : 148ull * 64);
}

hanf_status fail(hanf_status st, const std::string& msg) {
  hanf_host_detail::set_error(msg);
  return st;
}
hanf_status cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? HANF_OUT_OF_MEMORY : HANF_CUDA_ERROR,
              std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer (stream-ordered pool)
template <class T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

#define GG_TRY(expr)                                   \
  do {                                                 \
    const cudaError_t _e = (expr);                     \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// Sorts keys[0, count) (bits [0, end_bit)), removes duplicates, drops keys
// >= sentinel and emits the CSR of n rows into a new host graph.
hanf_status keys_to_graph(cudaStream_t s, DevBuf<uint64_t>& keys, uint64_t count, int end_bit,
                          uint64_t n, uint64_t sentinel, hanf_graph** out) {
  DevBuf<uint64_t> alt{nullptr, s};
  GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&alt.p), sizeof(uint64_t) * (count ? count : 1), s));
  uint64_t* sorted = keys.p;
  if (count) {
    cub::DoubleBuffer<uint64_t> db(keys.p, alt.p);
    size_t tb = 0;
    GG_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, static_cast<int64_t>(count), 0, end_bit, s));
    DevBuf<uint8_t> temp{nullptr, s};
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&temp.p), tb ? tb : 1, s));
    GG_TRY(cub::DeviceRadixSort::SortKeys(temp.p, tb, db, static_cast<int64_t>(count), 0, end_bit, s));
    sorted = db.Current();
  }
  uint64_t* uniq = sorted == keys.p ? alt.p : keys.p;
  DevBuf<uint64_t> num{nullptr, s};
  GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&num.p), sizeof(uint64_t), s));
  GG_TRY(cudaMemsetAsync(num.p, 0, sizeof(uint64_t), s));
  if (count) {
    size_t tb = 0;
    GG_TRY(cub::DeviceSelect::Unique(nullptr, tb, sorted, uniq, num.p, static_cast<int64_t>(count), s));
    DevBuf<uint8_t> temp{nullptr, s};
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&temp.p), tb ? tb : 1, s));
    GG_TRY(cub::DeviceSelect::Unique(temp.p, tb, sorted, uniq, num.p, static_cast<int64_t>(count), s));
  }
  uint64_t m = 0, last = 0;
  GG_TRY(cudaMemcpyAsync(&m, num.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  GG_TRY(cudaStreamSynchronize(s));
  if (m) {
    GG_TRY(cudaMemcpyAsync(&last, uniq + m - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    GG_TRY(cudaStreamSynchronize(s));
    if (last >= sentinel) --m;  // all dropped self-loops collapsed into one key
  }
  DevBuf<uint64_t> off{nullptr, s};
  DevBuf<uint32_t> arcs{nullptr, s};
  GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&off.p), sizeof(uint64_t) * (n + 1), s));
  GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&arcs.p), sizeof(uint32_t) * (m ? m : 1), s));
  row_offsets_kernel<<<grid_for(m + 1), 256, 0, s>>>(uniq, m, n, off.p);
  GG_TRY(cudaGetLastError());
  if (m) {
    low_words_kernel<<<grid_for(m), 256, 0, s>>>(uniq, m, arcs.p);
    GG_TRY(cudaGetLastError());
  }
  hanf_graph* g = new (std::nothrow) hanf_graph();
  if (!g) return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  try {
    g->n = n;
    g->offsets.resize(n + 1);
    g->succ.resize(m);
  } catch (const std::bad_alloc&) {
    delete g;
    return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  }
  cudaError_t e = cudaMemcpyAsync(g->offsets.data(), off.p, sizeof(uint64_t) * (n + 1),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && m)
    e = cudaMemcpyAsync(g->succ.data(), arcs.p, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "graph read-back");
  }
  *out = g;
  return HANF_OK;
}

int bits_for(uint64_t x) {  // bits needed to represent values < x
  int b = 0;
  while (b < 64 && (1ull << b) < x) ++b;
  return b;
}

}  // namespace

extern "C" {

hanf_status hanf_graph_from_edges_gpu(int32_t device, uint64_t n, const uint32_t* src,
                                      const uint32_t* dst, uint64_t count, hanf_graph** out) {
  if (!out || (count && (!src || !dst))) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (n > 0xffffffffull) return fail(HANF_INVALID_ARGUMENT, "graph too large for 32-bit node ids");
  *out = nullptr;
  GG_TRY(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  GG_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{s};
  hanf_status st = HANF_OK;
  {
    DevBuf<uint32_t> ds{nullptr, s}, dd{nullptr, s};
    DevBuf<uint64_t> keys{nullptr, s};
    DevBuf<int> bad{nullptr, s};
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ds.p), sizeof(uint32_t) * (count ? count : 1), s));
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dd.p), sizeof(uint32_t) * (count ? count : 1), s));
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&keys.p), sizeof(uint64_t) * (count ? count : 1), s));
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&bad.p), sizeof(int), s));
    GG_TRY(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    if (count) {
      GG_TRY(cudaMemcpyAsync(ds.p, src, sizeof(uint32_t) * count, cudaMemcpyHostToDevice, s));
      GG_TRY(cudaMemcpyAsync(dd.p, dst, sizeof(uint32_t) * count, cudaMemcpyHostToDevice, s));
      edge_keys_kernel<<<grid_for(count), 256, 0, s>>>(ds.p, dd.p, count, n, keys.p, bad.p);
      GG_TRY(cudaGetLastError());
    }
    int h_bad = 0;
    GG_TRY(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    GG_TRY(cudaStreamSynchronize(s));
    if (h_bad) return fail(HANF_INVALID_ARGUMENT, "arc endpoint out of range");
    const uint64_t sentinel = n << 32;  // no sentinels here; rows are < n
    st = keys_to_graph(s, keys, count, 32 + bits_for(n), n, sentinel, out);
  }
  return st;
}

hanf_status hanf_gen_rmat_gpu(int32_t device, uint32_t scale, uint32_t edge_factor, double a,
                              double b, double c, uint64_t seed, uint64_t permute_seed,
                              hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (scale < 2 || scale > 31) return fail(HANF_INVALID_ARGUMENT, "R-MAT scale must be in [2, 31]");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
    return fail(HANF_INVALID_ARGUMENT, "R-MAT probabilities must be non-negative, a+b+c <= 1");
  *out = nullptr;
  const uint64_t n = 1ull << scale;
  const uint64_t draws = n * edge_factor;
  const uint32_t ta = static_cast<uint32_t>(a * 65536.0);
  const uint32_t tb = static_cast<uint32_t>((a + b) * 65536.0);
  const uint32_t tc = static_cast<uint32_t>((a + b + c) * 65536.0);
  GG_TRY(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  GG_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{s};
  hanf_status st = HANF_OK;
  {
    DevBuf<uint64_t> keys{nullptr, s};
    GG_TRY(cudaMallocAsync(reinterpret_cast<void**>(&keys.p), sizeof(uint64_t) * (draws ? draws : 1), s));
    const uint64_t sentinel = n << 32;  // past every row: self-loops sort last
    rmat_keys_kernel<<<grid_for(draws), 256, 0, s>>>(draws, scale, ta, tb, tc, seed,
                                                      hanf_rng::Feistel(scale, permute_seed),
                                                      sentinel, keys.p);
    GG_TRY(cudaGetLastError());
    st = keys_to_graph(s, keys, draws, 33 + scale, n, sentinel, out);
  }
  return st;
}

}  // extern "C"
