// hanf_kernels.cu -- sm_100a kernels of the HyperANF iteration.
//
//   seed_kernel        NfEngine ctor seeding (engine.hpp:84-85, hll.hpp:104-117)
//   union_kernel       the union sweep of NfEngine::step (engine.hpp:157-185,
//                      PackedMax::max_into broadword.hpp:94-130), degree-binned
//   hub_finalize       combines the partial maxima of split high-degree nodes
//   estimate_kernel    counter_estimate + per-64-counter block sums
//                      (hll.hpp:122-141, engine.hpp:100-113), dirty blocks only
//   reduce kernels     deterministic total of the block sums and the modified
//                      count (engine.hpp:115-117, 202-208)
#include <cuda_runtime.h>

#include <cstdint>

#include "hanf_device.cuh"
#include "hanf_internal.h"

namespace hanf {

// ---------------------------------------------------------------------------
// Seeding: counter v := zero, then counter_add(v, item v).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // hash.hpp:8-15
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}

__global__ void seed_kernel(uint64_t* __restrict__ a, uint64_t* __restrict__ b,
                            uint64_t* __restrict__ mod, uint64_t n, uint64_t node_begin,
                            uint64_t node_end, uint32_t bucket_bits, uint32_t register_bits,
                            uint32_t words, uint64_t seed_mix) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = node_begin + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       v < node_end; v += stride) {
    const uint64_t h = mix64(v ^ seed_mix);  // item_hash, hash.hpp:20-22
    const uint32_t bucket = static_cast<uint32_t>(h >> (64 - bucket_bits));
    const uint64_t rest = h << bucket_bits;
    uint32_t rho = rest == 0 ? (64 - bucket_bits) + 1 : __clzll(rest) + 1;
    const uint32_t maxv = (1u << register_bits) - 1;
    rho = rho < maxv ? rho : maxv;
    const uint64_t bit = static_cast<uint64_t>(bucket) * register_bits;
    const uint64_t wi = bit >> 6;
    const uint32_t off = bit & 63;
    uint64_t* ca = a + v * words;
    uint64_t* cb = b + v * words;
    for (uint32_t k = 0; k < words; ++k) {
      uint64_t word = 0;
      if (k == wi) word |= static_cast<uint64_t>(rho) << off;
      if (k == wi + 1 && off + register_bits > 64) word |= static_cast<uint64_t>(rho) >> (64 - off);
      ca[k] = word;
      cb[k] = word;
    }
  }
  // every seeded counter counts as modified (engine.hpp:86)
  const uint64_t wbegin = node_begin >> 6, wend = (node_end + 63) >> 6;
  for (uint64_t w = wbegin + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       w < wend; w += stride) {
    uint64_t bits = ~0ull;
    const uint64_t first = w << 6;
    if (first < node_begin) bits &= ~0ull << (node_begin - first);
    if (first + 64 > node_end) bits &= ~0ull >> (first + 64 - node_end);
    mod[w] = bits;  // shard ranges are 64-aligned except the last one
  }
}

cudaError_t launch_seed(uint64_t* a, uint64_t* b, uint64_t* mod, uint64_t n,
                        uint64_t node_begin, uint64_t node_end, uint32_t bucket_bits,
                        uint32_t register_bits, uint32_t words, uint64_t seed,
                        cudaStream_t s, uint64_t* launches) {
  if (node_end <= node_begin) return cudaSuccess;
  const uint64_t items = node_end - node_begin;
  const uint32_t threads = 256;
  uint64_t blocks = (items + threads - 1) / threads;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  seed_kernel<<<static_cast<uint32_t>(blocks), threads, 0, s>>>(
      a, b, mod, n, node_begin, node_end, bucket_bits, register_bits, words,
      mix64(seed ^ 0x9e3779b97f4a7c15ULL));
  ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Union sweep.  One launch covers every node with out-degree >= 1, one warp
// per WarpTask (built once per graph, hanf_engine.cu build_tasks):
//   light task  32/G nodes with G = next_pow2(ceil(deg/32)) lanes each (so a
//               lane walks <= 32 arcs), nodes of equal class in descending
//               degree;
//   hub chunk   <= kHubChunk arcs of one node with out-degree > kHubDegree;
//               the warp writes its partial maximum to `partials`.
// The successor ids are read from the task-ordered successor array (TOS):
// warp row i holds the 32 ids its lanes fold in trip i (lane = node slot *
// G + sub, id = successor i*G + sub of that node; padding = the all-zero
// counter row n), so every id row is one coalesced 128-byte load and the
// trip count is warp-uniform.  Each lane keeps a running register file in
// 32-bit limbs and folds U successor counters per trip (swar_max); the G
// lanes of a node combine with butterfly shuffles; the lead lane compares
// with the old counter, writes the next generation where it changed or
// where next[v] is stale, estimates a changed counter from its registers
// (single-chunk layouts) and sets the node's bit in mod_next.
// Successor gathers: GMODE 0 = per-word loads, 1 = 16-byte windows,
// 2 = 32-byte windows (fewer L1 wavefronts, more selects).
// ---------------------------------------------------------------------------
template <class Lay>
__device__ __forceinline__ void zero_limbs(uint32_t (&x)[Lay::kLimbs]) {
  sfor<0, Lay::kLimbs>([&](auto I) { x[decltype(I)::value] = 0u; });
}

template <class Lay, int GMODE, bool kVec16>
struct Gather;

template <class Lay, bool kVec16>
struct Gather<Lay, 0, kVec16> {
  uint32_t v[Lay::kLimbs];
  __device__ __forceinline__ void issue(const uint64_t* cur, uint32_t w, uint32_t words,
                                        uint32_t woff) {
    load_chunk<Lay, kVec16>(v, cur + static_cast<uint64_t>(w) * words + woff);
  }
  __device__ __forceinline__ void extract(uint32_t (&x)[Lay::kLimbs], uint32_t) const {
    sfor<0, Lay::kLimbs>([&](auto I) { x[decltype(I)::value] = v[decltype(I)::value]; });
  }
};

template <class Lay, bool kVec16>
struct Gather<Lay, 1, kVec16> {
  uint4 raw[Window128<Lay::kWords>::kLoads];
  __device__ __forceinline__ void issue(const uint64_t* cur, uint32_t w, uint32_t, uint32_t) {
    window128_load<Lay::kWords>(raw, cur, w);
  }
  __device__ __forceinline__ void extract(uint32_t (&x)[Lay::kLimbs], uint32_t w) const {
    window128_extract<Lay, Lay::kWords>(x, raw, w);
  }
};

template <class Lay, bool kVec16>
struct Gather<Lay, 2, kVec16> {
  uint32_t raw[Window<Lay::kWords>::kLoads][8];
  __device__ __forceinline__ void issue(const uint64_t* cur, uint32_t w, uint32_t, uint32_t) {
    window_load<Lay::kWords>(raw, cur, w);
  }
  __device__ __forceinline__ void extract(uint32_t (&x)[Lay::kLimbs], uint32_t w) const {
    window_extract<Lay, Lay::kWords>(x, raw, w);
  }
};

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int R, int NREG, int U, int GMODE, bool kVec16>
__global__ void __launch_bounds__(256) union_kernel(const UnionArgs args) {
  using Lay = Layout<R, NREG>;
  constexpr int NL = Lay::kLimbs;
  constexpr int NW = Lay::kWords;
  using G_t = Gather<Lay, GMODE, kVec16>;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (gw >= args.num_wtasks) return;
  const WarpTask task = args.wtasks[gw];
  const bool hub = task.nodes == 0;
  const uint32_t lg = hub ? 5u : task.lg;
  const uint32_t G = 1u << lg;
  const uint32_t sub = lane & (G - 1);
  const uint32_t zero_row = args.zero_row;
  uint32_t v = zero_row;
  bool active = true;
  if (hub) {
    v = args.hub_node[task.item];
  } else {
    const uint32_t j = lane >> lg;
    active = j < task.nodes;
    if (active) v = args.order[task.item + j];
  }
  const bool lead = active && sub == 0 && !hub;
  bool stale = false;
  if (lead && args.stale_valid) stale = (args.mod_cur[v >> 6] >> (v & 63)) & 1;
  const uint64_t* __restrict__ cur = args.cur;
  const uint32_t* __restrict__ ids = args.tos + task.tos + lane;
  const uint32_t words = args.words;
  const uint32_t trips = task.trips;

  bool any_changed = false;
  for (uint32_t ch = 0; ch < args.chunks; ++ch) {
    const uint32_t woff = ch * NW;
    uint32_t acc[NL];
    uint32_t own[NL];
    {
      G_t g;
      g.issue(cur, lead ? v : zero_row, words, woff);
      g.extract(own, lead ? v : zero_row);
    }
    sfor<0, NL>([&](auto I) { acc[decltype(I)::value] = own[decltype(I)::value]; });
    for (uint32_t i = 0; i < trips; i += U) {
      uint32_t w[U];
#pragma unroll
      for (int j = 0; j < U; ++j)
        w[j] = (i + j < trips) ? ld_stream_u32(ids + 32 * (i + j)) : zero_row;
      if (args.check_mod) {
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (!((__ldg(args.mod_cur + (w[j] >> 6)) >> (w[j] & 63)) & 1)) w[j] = zero_row;
      }
      G_t g[U];
#pragma unroll
      for (int j = 0; j < U; ++j) g[j].issue(cur, w[j], words, woff);
#pragma unroll
      for (int j = 0; j < U; ++j) {
        uint32_t y[NL];
        g[j].extract(y, w[j]);
        swar_max<Lay>(acc, y);
      }
    }
    for (uint32_t off = G >> 1; off >= 1; off >>= 1) shfl_max<Lay>(acc, off);

    if (hub) {
      if (lane == 0)
        store_chunk<Lay, kVec16>(args.partials + static_cast<uint64_t>(task.item) * words + woff,
                                 acc);
    } else {
      const bool changed = lead && limbs_differ<Lay>(acc, own);
      any_changed |= changed;
      if (changed || (lead && stale))
        store_chunk<Lay, kVec16>(args.next + static_cast<uint64_t>(v) * words + woff, acc);
      if (changed && args.est) args.est[v] = estimate_limbs<Lay>(acc, args.ep);
    }
  }
  if (any_changed)
    atomicOr(reinterpret_cast<unsigned long long*>(args.mod_next) + (v >> 6),
             1ull << (v & 63));
}

// One warp per split node: max over its chunk partials and its own counter.
template <int R, int NREG, bool kVec16>
__global__ void __launch_bounds__(256) hub_finalize_kernel(const HubArgs args) {
  using Lay = Layout<R, NREG>;
  constexpr int NL = Lay::kLimbs;
  constexpr int NW = Lay::kWords;
  const uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (h >= args.num_hubs) return;
  const uint32_t v = args.hub_nodes[h];
  const uint32_t first = args.hub_first[h];
  const uint32_t count = args.hub_count[h];
  const uint32_t words = args.words;
  bool stale = false;
  if (args.stale_valid) stale = (args.mod_cur[v >> 6] >> (v & 63)) & 1;
  bool any_changed = false;
  for (uint32_t ch = 0; ch < args.chunks; ++ch) {
    const uint32_t woff = ch * NW;
    uint32_t acc[NL];
    if (lane == 0)
      load_chunk<Lay, kVec16>(acc, args.cur + static_cast<uint64_t>(v) * words + woff);
    else
      zero_limbs<Lay>(acc);
    for (uint32_t i = lane; i < count; i += 32) {
      uint32_t y[NL];
      load_chunk_coherent<Lay>(y, args.partials + static_cast<uint64_t>(first + i) * words + woff);
      swar_max<Lay>(acc, y);
    }
    for (uint32_t off = 16; off >= 1; off >>= 1) shfl_max<Lay>(acc, off);
    if (lane == 0) {
      uint32_t own[NL];
      load_chunk<Lay, kVec16>(own, args.cur + static_cast<uint64_t>(v) * words + woff);
      const bool changed = limbs_differ<Lay>(acc, own);
      any_changed |= changed;
      if (changed || stale)
        store_chunk<Lay, kVec16>(args.next + static_cast<uint64_t>(v) * words + woff, acc);
      if (changed && args.est) args.est[v] = estimate_limbs<Lay>(acc, args.ep);
    }
  }
  if (lane == 0 && any_changed)
    atomicOr(reinterpret_cast<unsigned long long*>(args.mod_next) + (v >> 6),
             1ull << (v & 63));
}

namespace {
struct KernelChoice {
  int r, nreg, chunks;
};
KernelChoice choose(uint32_t r, uint32_t m) {
  switch (r) {
    case 5:
      if (m <= 128) return {5, static_cast<int>(m), 1};
      return {5, 64, static_cast<int>(m / 64)};
    case 6:
      if (m == 16) return {6, 16, 1};
      return {6, 32, static_cast<int>(m / 32)};
    case 7:
      if (m <= 64) return {7, static_cast<int>(m), 1};
      return {7, 64, static_cast<int>(m / 64)};
    default:
      return {8, 16, static_cast<int>(m / 16)};
  }
}

template <int R, int NREG, int U, int GM, bool V>
cudaError_t union_launch(UnionArgs a, uint32_t chunks, cudaStream_t s) {
  a.chunks = chunks;
  if (chunks != 1) a.est = nullptr;  // estimates need the whole counter in registers
  if (a.num_wtasks == 0) return cudaSuccess;
  const uint32_t blocks = (a.num_wtasks + 7) / 8;
  union_kernel<R, NREG, U, GM, V><<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

template <int R, int NREG, bool V>
cudaError_t hub_launch(HubArgs a, uint32_t chunks, cudaStream_t s) {
  a.chunks = chunks;
  if (chunks != 1) a.est = nullptr;
  if (a.num_hubs == 0) return cudaSuccess;
  const uint32_t blocks = (a.num_hubs + 7) / 8;
  hub_finalize_kernel<R, NREG, V><<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}
}  // namespace

bool fused_estimates(uint32_t register_bits, uint32_t registers) {
  return choose(register_bits, registers).chunks == 1;
}

cudaError_t launch_union(const UnionArgs& args, uint32_t register_bits, uint32_t registers,
                         int gather_mode, cudaStream_t s, uint64_t* launches) {
  const KernelChoice k = choose(register_bits, registers);
  if (args.num_wtasks == 0) return cudaSuccess;
  ++*launches;
  const uint32_t ch = static_cast<uint32_t>(k.chunks);
  const bool single = ch == 1;
  switch (k.r * 1000 + k.nreg) {
    case 5016: return union_launch<5, 16, 4, 0, true>(args, ch, s);
    case 5032:
      if (single && gather_mode == 2) return union_launch<5, 32, 4, 2, false>(args, ch, s);
      if (single && gather_mode == 1) return union_launch<5, 32, 4, 1, false>(args, ch, s);
      return union_launch<5, 32, 4, 0, false>(args, ch, s);
    case 5064:
      if (single && gather_mode == 2) return union_launch<5, 64, 4, 2, false>(args, ch, s);
      if (single && gather_mode == 1) return union_launch<5, 64, 4, 1, false>(args, ch, s);
      return union_launch<5, 64, 4, 0, false>(args, ch, s);
    case 5128:
      if (gather_mode == 2) return union_launch<5, 128, 2, 2, true>(args, ch, s);
      return union_launch<5, 128, 2, 0, true>(args, ch, s);
    case 6016: return union_launch<6, 16, 4, 0, true>(args, ch, s);
    case 6032: return union_launch<6, 32, 4, 0, false>(args, ch, s);
    case 7016: return union_launch<7, 16, 4, 0, true>(args, ch, s);
    case 7032: return union_launch<7, 32, 4, 0, true>(args, ch, s);
    case 7064: return union_launch<7, 64, 2, 0, false>(args, ch, s);
    default: return union_launch<8, 16, 4, 0, true>(args, ch, s);
  }
}

cudaError_t launch_hub_finalize(const HubArgs& args, uint32_t register_bits, uint32_t registers,
                                cudaStream_t s, uint64_t* launches) {
  if (args.num_hubs == 0) return cudaSuccess;
  const KernelChoice k = choose(register_bits, registers);
  ++*launches;
  const uint32_t ch = static_cast<uint32_t>(k.chunks);
  switch (k.r * 1000 + k.nreg) {
    case 5016: return hub_launch<5, 16, true>(args, ch, s);
    case 5032: return hub_launch<5, 32, false>(args, ch, s);
    case 5064: return hub_launch<5, 64, false>(args, ch, s);
    case 5128: return hub_launch<5, 128, true>(args, ch, s);
    case 6016: return hub_launch<6, 16, true>(args, ch, s);
    case 6032: return hub_launch<6, 32, false>(args, ch, s);
    case 7016: return hub_launch<7, 16, true>(args, ch, s);
    case 7032: return hub_launch<7, 32, true>(args, ch, s);
    case 7064: return hub_launch<7, 64, false>(args, ch, s);
    default: return hub_launch<8, 16, true>(args, ch, s);
  }
}

// ---------------------------------------------------------------------------
// Block sums from cached estimates (union kernels wrote est[v] for every
// changed counter): one thread per 64-counter block, sequential in index
// order (engine.hpp:109-111); clean blocks keep their cached sum (:105).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
block_sum_kernel(const double* __restrict__ est, const uint64_t* __restrict__ dirty,
                 double* __restrict__ block_sums, uint64_t n, uint64_t b0, uint64_t b1) {
  const uint64_t b = b0 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (b >= b1) return;
  if (dirty[b] == 0) return;
  const uint64_t first = b * 64;
  const uint32_t last = n - first < 64 ? static_cast<uint32_t>(n - first) : 64u;
  double sum = 0.0;
  if (last == 64) {
    const double2* p = reinterpret_cast<const double2*>(est + first);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double2 q = __ldg(p + k);
      sum = __dadd_rn(sum, q.x);
      sum = __dadd_rn(sum, q.y);
    }
  } else {
    for (uint32_t i = 0; i < last; ++i) sum = __dadd_rn(sum, est[first + i]);
  }
  block_sums[b] = sum;
}

cudaError_t launch_block_sums(const double* est, const uint64_t* dirty, double* block_sums,
                              uint64_t n, uint64_t b0, uint64_t b1, cudaStream_t s,
                              uint64_t* launches) {
  if (b1 <= b0) return cudaSuccess;
  const uint64_t blocks = (b1 - b0 + 255) / 256;
  block_sum_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(est, dirty, block_sums, n, b0, b1);
  ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Estimates + block sums.  One CTA of 64 threads per 64-counter block
// (engine.hpp:278 kBlock): a block whose dirty word is zero keeps its
// cached sum (engine.hpp:105); otherwise changed counters are re-estimated
// (cached estimates reused for the rest) and thread 0 adds the 64
// estimates sequentially in index order, exactly as engine.hpp:109-111.
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(64) estimate_kernel(const EstimateArgs args) {
  __shared__ double sh[64];
  const uint64_t blk = args.block_begin + blockIdx.x;
  if (blk >= args.block_end) return;
  const uint64_t word = args.dirty ? args.dirty[blk] : ~0ull;
  if (word == 0) return;
  const uint32_t t = threadIdx.x;
  const uint64_t v = blk * 64 + t;
  EstimateParams p{args.alpha, args.m, args.registers, args.register_bits, args.words,
                   args.log_table};
  double e = 0.0;
  if (v < args.n) {
    if ((word >> t) & 1) {
      if constexpr (M > 0)
        e = estimate_counter_r5<M>(args.counters + v * args.words, p);
      else
        e = estimate_counter_generic(args.counters + v * args.words, p);
      args.est[v] = e;
    } else {
      e = args.est[v];
    }
  }
  sh[t] = e;
  __syncthreads();
  if (t == 0) {
    const uint64_t first = blk * 64;
    const uint32_t last = args.n - first < 64 ? static_cast<uint32_t>(args.n - first) : 64u;
    double sum = 0.0;
    for (uint32_t i = 0; i < last; ++i) sum = __dadd_rn(sum, sh[i]);
    args.block_sums[blk] = sum;
  }
}

cudaError_t launch_estimate(const EstimateArgs& args, cudaStream_t s, uint64_t* launches) {
  if (args.block_end <= args.block_begin) return cudaSuccess;
  const uint64_t blocks = args.block_end - args.block_begin;
  ++*launches;
  if (args.register_bits == 5 && args.registers == 32)
    estimate_kernel<32><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args);
  else if (args.register_bits == 5 && args.registers == 64)
    estimate_kernel<64><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args);
  else if (args.register_bits == 5 && args.registers == 128)
    estimate_kernel<128><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args);
  else
    estimate_kernel<0><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Deterministic total of block sums [begin, end) and popcount of the
// modified bitmap over the same blocks: a fixed partition into kReduceCtas
// contiguous ranges, fixed per-thread strides and a fixed tree, so reruns
// are bit-identical (the reference's sequential order of the total is
// reproduced on the host when exact_sum is set).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_tree_sum(double v, double* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int w = kReduceThreads / 2; w >= 1; w >>= 1) {
    if (t < w) sh[t] = __dadd_rn(sh[t], sh[t + w]);
    __syncthreads();
  }
  return sh[0];
}

__device__ __forceinline__ unsigned long long block_count_sum(unsigned long long v,
                                                              unsigned long long* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int w = kReduceThreads / 2; w >= 1; w >>= 1) {
    if (t < w) sh[t] += sh[t + w];
    __syncthreads();
  }
  return sh[0];
}

// Level 1: CTA b reduces the fixed range [begin + b*per, ...) of the block
// sums and of the modified bitmap (bitmap word i <-> block i).
__global__ void __launch_bounds__(kReduceThreads)
reduce_level1(const double* __restrict__ x, const uint64_t* __restrict__ bits, uint64_t begin,
              uint64_t end, ReduceOut* __restrict__ out) {
  __shared__ double sh[kReduceThreads];
  __shared__ unsigned long long shc[kReduceThreads];
  const uint64_t len = end - begin;
  const uint64_t per = (len + kReduceCtas - 1) / kReduceCtas;
  const uint64_t lo = begin + blockIdx.x * per;
  const uint64_t hi = lo + per < end ? lo + per : end;
  double acc = 0.0;
  unsigned long long cnt = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += kReduceThreads) {
    acc = __dadd_rn(acc, x[i]);
    cnt += __popcll(bits[i]);
  }
  const double total = block_tree_sum(acc, sh);
  const unsigned long long count = block_count_sum(cnt, shc);
  if (threadIdx.x == 0) {
    out->partial_sum[blockIdx.x] = total;
    out->partial_count[blockIdx.x] = count;
  }
}

__global__ void __launch_bounds__(kReduceThreads) reduce_level2(ReduceOut* __restrict__ out) {
  __shared__ double sh[kReduceThreads];
  __shared__ unsigned long long shc[kReduceThreads];
  double acc = 0.0;
  unsigned long long cnt = 0;
  for (int i = threadIdx.x; i < kReduceCtas; i += kReduceThreads) {
    acc = __dadd_rn(acc, out->partial_sum[i]);
    cnt += out->partial_count[i];
  }
  const double total = block_tree_sum(acc, sh);
  const unsigned long long count = block_count_sum(cnt, shc);
  if (threadIdx.x == 0) {
    out->total = total;
    out->count = count;
  }
}

cudaError_t launch_reduce(const double* block_sums, const uint64_t* bits, uint64_t begin,
                          uint64_t end, ReduceOut* out, cudaStream_t s, uint64_t* launches) {
  reduce_level1<<<kReduceCtas, kReduceThreads, 0, s>>>(block_sums, bits, begin, end, out);
  reduce_level2<<<1, kReduceThreads, 0, s>>>(out);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace hanf
