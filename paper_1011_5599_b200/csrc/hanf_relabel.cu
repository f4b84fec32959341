// hanf_relabel.cu -- locality relabelling of the graph on the device
// (engine-internal layout; results are bit-identical to the reference).
//
// Gathers dominate the union sweep, and a node's counter is gathered once
// per in-arc.  On graphs whose ids carry no locality (R-MAT / BA with
// permuted ids) the hot counters are scattered one per 128-byte line.
// Renumbering nodes by descending out-degree packs the hot counters
// together (profiles/r01_relabel.md).  Graphs whose ids are already local
// (the copying model's windows) keep their labels: hanf_engine.cu decides
// with a sampled locality test.
//
// The engine works on the relabelled CSR in "row" space (counters, the
// modified bitmaps the skips and the worklist read, and by default the
// estimates); everything the caller sees stays in the original id space:
//   order[row] = original id   (seed hash input; a changed row sets its bit
//                               in the original-id dirty bitmap)
//   perm[id]   = row           (counter read-back; finish_kernel gathers
//                               est[perm[o]] for the original-id blocks)
// so N(t) is still summed over original-id blocks in the reference order.
// Estimates in row order cost the finish a random gather; scattered to the
// original slots (a round-1 variant, removed) they cost the union sweep
// partial-sector writes.  Measured per dense step: BA 2^25 13.38 ms
// (rows) vs 13.89 ms (scatter), R-MAT 26 12.84 vs 12.73 ms.
//
// Relabelling pays where the counters do not fit in L2 (measured 2.4x on
// R-MAT 26, 1.25x on BA 2^25).  On the L2-resident config 2 it gains 5% on
// the union sweep but costs ~1 ms at create (the seed and task build can no
// longer overlap the upload), so it is off there by default.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "hanf_internal.h"

namespace hanf {
namespace {

// keys = ~out-degree: descending out-degree, stable in id.  (Total degree
// needs an in-degree pass of contended atomics - 160 ms on R-MAT 28 - and
// measured no better: R-MAT's and BA's in- and out-degrees go together, and
// rows in out-degree order make the union's task order match the row order.)
__global__ void score_keys_kernel(const uint64_t* __restrict__ off, uint64_t n,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                  int* __restrict__ bad) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < n;
       v += stride) {
    const uint64_t a = off[v], b = off[v + 1];
    uint64_t d = 0;
    if (b < a)
      *bad = 1;
    else
      d = b - a;
    keys[v] = ~static_cast<uint32_t>(d < 0xffffffffull ? d : 0xffffffffull);
    vals[v] = static_cast<uint32_t>(v);
  }
}

// Line-aligned slots.  A W-word row with W odd (40 bytes for m = 64)
// straddles a 128-byte line at 4 of every 16 row offsets; a random gather
// of such a row costs two DRAM line fetches instead of one.  Past a hot
// prefix (rows that live in L2 anyway, kept dense), degree ranks fill the
// rows that sit inside one line first and the straddling rows last, so the
// coldest nodes - the ones almost never gathered - take the straddling
// slots.
struct Slots {
  uint64_t hot;    // rows [0, hot) of a range keep rank order (multiple of 16)
  uint32_t n_in;   // offsets (mod 16) whose row lies inside one line
  uint32_t n_st;   // offsets whose row straddles a line
  uint8_t in[16];  // ascending
  uint8_t st[16];  // ascending
};

// Local rank j of a range of `per` rows (per - hot arbitrary) -> local row.
__device__ __forceinline__ uint64_t slot_of(const Slots& sl, uint64_t per, uint64_t j) {
  if (sl.n_st == 0 || j < sl.hot) return j;
  const uint64_t len = per - sl.hot, full = len / 16, rem = len % 16;
  uint64_t in_total = full * sl.n_in;
  for (uint32_t k = 0; k < sl.n_in; ++k) in_total += sl.in[k] < rem;
  uint64_t k = j - sl.hot;
  if (k < in_total) return sl.hot + 16 * (k / sl.n_in) + sl.in[k % sl.n_in];
  k -= in_total;
  return sl.hot + 16 * (k / sl.n_st) + sl.st[k % sl.n_st];
}

// Degree rank i -> row (i mod ways) * (n / ways) + slot(i / ways): relabelled
// shards (ways > 1) get the same degree profile with their hot rows first.
__global__ void interleave_kernel(const uint32_t* __restrict__ sorted, uint64_t n, uint32_t ways,
                                  const Slots sl, uint32_t* __restrict__ order) {
  const uint64_t per = n / ways;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    order[(i % ways) * per + slot_of(sl, per, i / ways)] = sorted[i];
}

Slots make_slots(uint32_t pitch, uint64_t per, uint32_t ways) {
  Slots sl{};
  // HANF_SLOTS=0: plain rank order.  HANF_SLOTS_HOT: dense hot prefix (rows
  // per range), default 2^22 rows (measured best on config 5, profiles/r02_union_probes.md)
  const char* e = std::getenv("HANF_SLOTS");
  if ((e && e[0] == '0') || pitch % 2 == 0 || pitch >= 16) return sl;
  uint64_t hot = 1ull << 22;
  if (const char* h = std::getenv("HANF_SLOTS_HOT")) hot = std::strtoull(h, nullptr, 10);
  hot = (hot / ways) & ~15ull;  // the hot rows spread over the shards
  if (hot >= per) return sl;
  sl.hot = hot;
  for (uint32_t o = 0; o < 16; ++o) {
    const uint32_t start = (8 * pitch * o) % 128;
    if (start + 8 * pitch > 128)
      sl.st[sl.n_st++] = static_cast<uint8_t>(o);
    else
      sl.in[sl.n_in++] = static_cast<uint8_t>(o);
  }
  return sl;
}

// perm[order[r]] = r; new degree of row r (for the offsets scan)
__global__ void invert_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ order,
                              uint64_t n, uint32_t* __restrict__ perm, uint64_t* __restrict__ ndeg) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r <= n;
       r += stride) {
    if (r == n) {
      ndeg[n] = 0;
      continue;
    }
    const uint32_t v = order[r];
    perm[v] = static_cast<uint32_t>(r);
    const uint64_t a = off[v], b = off[v + 1];
    ndeg[r] = b >= a ? b - a : 0;
  }
}

// Arc-parallel rewrite in destination order: warp w writes new arcs
// [w*1024, (w+1)*1024), 32 at a time (lane l takes arc base + 32j + l), so
// the stores are coalesced and hub rows cost no more than any other 1024
// arcs.  Lane 0 finds the row of the warp's first arc by binary search in
// the new offsets; after that each lane steps forward from the row of the
// previous 32 arcs' last arc.  New arc i of row r is old arc
// off[order[r]] + (i - noff[r]), relabelled through perm.  (Writing in
// source order instead scatters 4-byte stores over the new rows: 6x
// slower on R-MAT 26.)
__global__ void rewrite_arcs_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ succ,
                                    uint64_t n, uint64_t arcs, const uint32_t* __restrict__ order,
                                    const uint32_t* __restrict__ perm,
                                    const uint64_t* __restrict__ noff, uint32_t* __restrict__ out,
                                    int* __restrict__ bad) {
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  bool oob = false;
  for (uint64_t wb = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
       wb * 1024 < arcs; wb += warps) {
    const uint64_t base = wb * 1024;
    uint64_t r0 = 0;
    if (lane == 0) {  // last r with noff[r] <= base
      uint64_t lo = 0, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) / 2;
        if (noff[mid] <= base) lo = mid; else hi = mid - 1;
      }
      r0 = lo;
    }
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    for (uint32_t j = 0; j < 32; ++j) {
      const uint64_t i = base + 32ull * j + lane;
      uint64_t r = r0;
      if (i < arcs) {
        while (r < n && noff[r + 1] <= i) ++r;
        uint32_t val = 0;
        if (r < n) {  // else malformed offsets (flagged by score_keys_kernel)
          const uint64_t src = off[order[r]] + (i - noff[r]);
          const uint32_t w = src < arcs ? succ[src] : 0xffffffffu;
          if (w < n)
            val = perm ? perm[w] : w;  // (null: the upload mapped the ids already)
          else
            oob = true;
        }
        out[i] = val;
      }
      r0 = __shfl_sync(0xffffffffu, r, 31);
      if (base + 32ull * (j + 1) >= arcs) break;
    }
  }
  if (oob) *bad = 1;  // arc endpoint >= n
}

template <class T>
cudaError_t pool_alloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1), s);
}

}  // namespace

#define HANF_RELABEL_TRY(expr)          \
  do {                                  \
    const cudaError_t _e = (expr);      \
    if (_e != cudaSuccess) return _e;   \
  } while (0)

namespace {
struct Phases {  // HANF_PROFILE=1: synchronising phase times
  cudaStream_t s;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  bool on = [] {
    const char* p = std::getenv("HANF_PROFILE");
    return p && p[0] == '1';
  }();
  void operator()(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hanf]   relabel %-8s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
}  // namespace

cudaError_t relabel_order_device(const uint64_t* d_off, uint64_t n, uint32_t ways, uint32_t pitch,
                                 cudaStream_t s, RelabelOut* out, uint64_t* launches) {
  *out = RelabelOut{};
  if (n == 0) return cudaSuccess;
  Phases phase{s};
  const uint32_t threads = 256;
  auto grid = [](uint64_t items) {
    const uint64_t b = (items + 255) / 256;
    return static_cast<uint32_t>(b < 148ull * 32 ? (b ? b : 1) : 148ull * 32);
  };
  uint32_t *keys = nullptr, *vals = nullptr, *skeys = nullptr;
  int* d_bad = nullptr;  // decreasing offsets: the task build flags them too
  uint64_t* ndeg = nullptr;
  HANF_RELABEL_TRY(pool_alloc(&d_bad, 1, s));
  HANF_RELABEL_TRY(pool_alloc(&keys, n, s));
  HANF_RELABEL_TRY(pool_alloc(&vals, n, s));
  score_keys_kernel<<<grid(n), threads, 0, s>>>(d_off, n, keys, vals, d_bad);
  ++*launches;
  HANF_RELABEL_TRY(pool_alloc(&skeys, n, s));
  HANF_RELABEL_TRY(pool_alloc(&out->order, n, s));
  {
    size_t tb = 0;
    HANF_RELABEL_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, skeys, vals, out->order,
                                                     static_cast<int64_t>(n), 0, 32, s));
    void* temp = nullptr;
    HANF_RELABEL_TRY(cudaMallocAsync(&temp, tb ? tb : 1, s));
    HANF_RELABEL_TRY(cub::DeviceRadixSort::SortPairs(temp, tb, keys, skeys, vals, out->order,
                                                     static_cast<int64_t>(n), 0, 32, s));
    ++*launches;
    HANF_RELABEL_TRY(cudaFreeAsync(temp, s));
  }
  HANF_RELABEL_TRY(cudaFreeAsync(keys, s));
  HANF_RELABEL_TRY(cudaFreeAsync(vals, s));
  HANF_RELABEL_TRY(cudaFreeAsync(skeys, s));
  HANF_RELABEL_TRY(cudaFreeAsync(d_bad, s));
  if (ways > 1 && n % (64ull * ways) != 0) return cudaErrorInvalidValue;
  if (ways == 0) ways = 1;
  const Slots sl = make_slots(pitch, n / ways, ways);
  if (ways > 1 || sl.n_st) {
    uint32_t* inter = nullptr;
    HANF_RELABEL_TRY(pool_alloc(&inter, n, s));
    interleave_kernel<<<grid(n), threads, 0, s>>>(out->order, n, ways, sl, inter);
    ++*launches;
    HANF_RELABEL_TRY(cudaFreeAsync(out->order, s));
    out->order = inter;
  }
  phase("sort");
  HANF_RELABEL_TRY(pool_alloc(&out->perm, n, s));
  HANF_RELABEL_TRY(pool_alloc(&ndeg, n + 1, s));
  invert_kernel<<<grid(n + 1), threads, 0, s>>>(d_off, out->order, n, out->perm, ndeg);
  ++*launches;
  HANF_RELABEL_TRY(pool_alloc(&out->off, n + 1, s));
  {
    size_t tb = 0;
    HANF_RELABEL_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, ndeg, out->off,
                                                   static_cast<int64_t>(n + 1), s));
    void* temp = nullptr;
    HANF_RELABEL_TRY(cudaMallocAsync(&temp, tb ? tb : 1, s));
    HANF_RELABEL_TRY(cub::DeviceScan::ExclusiveSum(temp, tb, ndeg, out->off,
                                                   static_cast<int64_t>(n + 1), s));
    ++*launches;
    HANF_RELABEL_TRY(cudaFreeAsync(temp, s));
  }
  HANF_RELABEL_TRY(cudaFreeAsync(ndeg, s));
  phase("offsets");
  return cudaGetLastError();
}

// ids[i] = perm[ids[i]] in place (ids >= n stay: the TOS fill flags them)
__global__ void map_ids_kernel(uint32_t* __restrict__ ids, uint64_t count,
                               const uint32_t* __restrict__ perm, uint64_t n) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += stride) {
    const uint32_t w = ids[i];
    if (w < n) ids[i] = perm[w];
  }
}

cudaError_t launch_map_ids(uint32_t* ids, uint64_t count, const uint32_t* perm, uint64_t n,
                           cudaStream_t s, uint64_t* launches) {
  if (count == 0) return cudaSuccess;
  uint64_t blocks = (count + 1023) / 1024;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  map_ids_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(ids, count, perm, n);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t relabel_arcs_device(const uint64_t* d_off, const uint32_t* d_succ, uint64_t n,
                                uint64_t arcs, const RelabelOut& r, cudaStream_t s,
                                uint32_t** succ_out, int* bad, uint64_t* launches) {
  *succ_out = nullptr;
  *bad = 0;
  Phases phase{s};
  int* d_bad = nullptr;
  HANF_RELABEL_TRY(pool_alloc(&d_bad, 1, s));
  HANF_RELABEL_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
  HANF_RELABEL_TRY(pool_alloc(succ_out, arcs, s));
  if (arcs) {
    const uint64_t blocks = (arcs + 1023) / 1024;  // warp blocks of 1024 arcs
    uint64_t ctas = (blocks + 7) / 8;
    if (ctas > 148ull * 16) ctas = 148ull * 16;
    rewrite_arcs_kernel<<<static_cast<uint32_t>(ctas), 256, 0, s>>>(
        d_off, d_succ, n, arcs, r.order, r.perm, r.off, *succ_out, d_bad);
    ++*launches;
  }
  int h_bad = 0;
  HANF_RELABEL_TRY(cudaMemcpyAsync(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  HANF_RELABEL_TRY(cudaFreeAsync(d_bad, s));
  HANF_RELABEL_TRY(cudaStreamSynchronize(s));
  phase("arcs");
  *bad = h_bad;
  return cudaGetLastError();
}

}  // namespace hanf
