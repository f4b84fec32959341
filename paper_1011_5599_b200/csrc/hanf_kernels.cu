// hanf_kernels.cu -- sm_100a kernels of the HyperANF iteration.
//
//   seed_kernel        NfEngine ctor seeding (engine.hpp:84-85, hll.hpp:104-117)
//   union_kernel       the union sweep of NfEngine::step (engine.hpp:157-185,
//                      PackedMax::max_into broadword.hpp:94-130) over the
//                      reference packing, degree-binned warp tasks
//   union_kernel_bytes the same sweep over byte-register rows (ByteLayout),
//                      a group of lanes per gathered counter
//   finalize_hub       combines the partial maxima of split high-degree nodes
//                      (the last chunk to finish, by ticket)
//   estimate_kernel    counter_estimate + per-64-counter block sums
//                      (hll.hpp:122-141, engine.hpp:100-113), dirty blocks only
//   finish_kernel      block sums, deterministic total and modified count
//                      (engine.hpp:109-117, 202-208), report to the host
//   task_scan_kernel,  step mode 4: tasks in reach of a change from one TOS
//   stale_fixup_kernel pass, stale rows outside them copied
//   gather/scatter_rows read-back and restore (packing byte rows)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

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
                            uint32_t words, uint32_t pitch, uint64_t seed_mix,
                            const uint32_t* __restrict__ orig_of, uint32_t batch,
                            const uint64_t* __restrict__ batch_mix, bool bytes) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // One warp per 32 consecutive rows: lane l hashes row v0 + l, then the
  // warp writes the rows' 32 * pitch words with lane-contiguous 8-byte
  // stores (word j of the block belongs to row j / pitch: its one or two
  // non-zero words come from that row's lane by shuffle).  Per-thread rows
  // wrote 8 bytes every `pitch` words: 1.2 TB/s on config 5's 21.5 GB.
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t v0 = node_begin + (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x - lane);
       v0 < node_end; v0 += stride) {
    const uint64_t v = v0 + lane;
    // counter_add(v, v): the item is the node's original id (hash.hpp:20-22);
    // batched runs: row v is node v / batch of run v % batch
    uint32_t wi = 0xffffffffu;  // (rows past the range write nothing)
    uint64_t lo = 0, hi = 0;
    if (v < node_end) {
      uint64_t item = orig_of ? orig_of[v] : v;
      uint64_t mix = seed_mix;
      if (batch > 1) {
        item = v / batch;
        mix = batch_mix[v % batch];
      }
      const uint64_t h = mix64(item ^ mix);
      const uint32_t bucket = static_cast<uint32_t>(h >> (64 - bucket_bits));
      const uint64_t rest = h << bucket_bits;
      uint32_t rho = rest == 0 ? (64 - bucket_bits) + 1 : __clzll(rest) + 1;
      const uint32_t maxv = (1u << register_bits) - 1;
      rho = rho < maxv ? rho : maxv;
      if (bytes) {  // byte layout: register `bucket` is byte `bucket` of the row
        wi = bucket / 8;
        lo = static_cast<uint64_t>(rho) << (8 * (bucket % 8));
      } else {
        const uint64_t bit = static_cast<uint64_t>(bucket) * register_bits;
        const uint32_t off = bit & 63;
        wi = static_cast<uint32_t>(bit >> 6);
        lo = static_cast<uint64_t>(rho) << off;
        if (off + register_bits > 64) hi = static_cast<uint64_t>(rho) >> (64 - off);
      }
    }
    uint64_t* ca = a + v0 * pitch;
    uint64_t* cb = b + v0 * pitch;
    for (uint32_t j = lane; j < 32 * pitch; j += 32) {  // padding words beyond W stay 0
      const uint32_t r = j / pitch, k = j - r * pitch;
      const uint32_t rwi = __shfl_sync(0xffffffffu, wi, r);
      const uint64_t rlo = __shfl_sync(0xffffffffu, lo, r);
      const uint64_t rhi = __shfl_sync(0xffffffffu, hi, r);
      if (rwi == 0xffffffffu) continue;
      const uint64_t word = k == rwi ? rlo : (k == rwi + 1 ? rhi : 0);
      ca[j] = word;
      cb[j] = word;
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
                        uint32_t register_bits, uint32_t words, uint32_t pitch, uint64_t seed,
                        const uint32_t* orig_of, uint32_t batch, const uint64_t* batch_mix,
                        bool bytes, cudaStream_t s, uint64_t* launches) {
  if (node_end <= node_begin) return cudaSuccess;
  const uint64_t items = node_end - node_begin;
  const uint32_t threads = 256;
  uint64_t blocks = (items + threads - 1) / threads;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  seed_kernel<<<static_cast<uint32_t>(blocks), threads, 0, s>>>(
      a, b, mod, n, node_begin, node_end, bucket_bits, register_bits, words, pitch,
      mix64(seed ^ 0x9e3779b97f4a7c15ULL), orig_of, batch, batch_mix, bytes);
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
// Successor gathers: GMODE 0 = per-word (or 16-byte vector) loads, 1 =
// aligned 16-byte windows and a select on the word offset (odd W), 3 = one
// aligned 256-bit load per 4-word row (W = 3 padded to 4).
// ---------------------------------------------------------------------------
template <class Lay>
__device__ __forceinline__ void zero_limbs(uint32_t (&x)[Lay::kLimbs]) {
  sfor<0, Lay::kLimbs>([&](auto I) { x[decltype(I)::value] = 0u; });
}

// GMODE = gather kind (0 per-word loads, 1 16-byte windows, 3 aligned 256-bit rows).
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

template <class Lay, int POL>
struct Gather128 {
  uint4 raw[Window128<Lay::kWords>::kLoads];
  __device__ __forceinline__ void issue(const uint64_t* cur, uint32_t w, uint32_t, uint32_t) {
    window128_load<Lay::kWords, POL>(raw, cur, w);
  }
  __device__ __forceinline__ void extract(uint32_t (&x)[Lay::kLimbs], uint32_t w) const {
    window128_extract<Lay, Lay::kWords>(x, raw, w);
  }
};
template <class Lay, bool kVec16>
struct Gather<Lay, 1, kVec16> : Gather128<Lay, 0> {};

// GMODE 3: rows padded to a multiple of 4 words (row_pitch): counter w
// starts a 32-byte block, ceil(W/4) aligned 256-bit loads, no shifts.
template <class Lay, bool kVec16>
struct Gather<Lay, 3, kVec16> {
  static constexpr int K = (Lay::kWords + 3) / 4;
  uint32_t raw[K][8];
  __device__ __forceinline__ void issue(const uint64_t* cur, uint32_t w, uint32_t pitch,
                                        uint32_t woff) {
    const uint64_t* p = cur + static_cast<uint64_t>(w) * pitch + woff;
    sfor<0, K>([&](auto I) { ldg256(raw[decltype(I)::value], p + 4 * decltype(I)::value); });
  }
  __device__ __forceinline__ void extract(uint32_t (&x)[Lay::kLimbs], uint32_t) const {
    sfor<0, Lay::kLimbs>([&](auto I) {
      constexpr int i = decltype(I)::value;
      x[i] = raw[i / 8][i % 8];
    });
  }
};

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Records that counter row v changed: its bit in the row-space bitmap (skips
// and worklist) and, under relabelling, in the original-id bitmap the block
// sums and counts use.
__device__ __forceinline__ uint32_t est_slot(const uint32_t* orig_of, uint32_t v) {
  return orig_of ? orig_of[v] : v;
}
// Warp-aggregated form for the packed sweep (every lane calls it): lanes
// whose rows share a bitmap word (a warp's light nodes are consecutive
// rows in degree order) set their bits with one atomic (config 5: 56.4 ->
// 55.6 ms; the byte-layout sweep keeps one atomic per node, which measured
// faster there).
__device__ __forceinline__ void mark_changed_warp(uint64_t* mod_next, uint64_t* dirty_next,
                                                  const uint32_t* orig_of, uint32_t v,
                                                  bool changed) {
  const uint32_t word = changed ? v >> 6 : 0xffffffffu;
  const uint32_t peers = __match_any_sync(0xffffffffu, word);
  const uint64_t bit = changed ? 1ull << (v & 63) : 0ull;
  const uint32_t lo = __reduce_or_sync(peers, static_cast<uint32_t>(bit));
  const uint32_t hi = __reduce_or_sync(peers, static_cast<uint32_t>(bit >> 32));
  if (changed && (threadIdx.x & 31) == static_cast<uint32_t>(__ffs(peers) - 1))
    atomicOr(reinterpret_cast<unsigned long long*>(mod_next) + word,
             (static_cast<uint64_t>(hi) << 32) | lo);
  if (changed && dirty_next) {
    const uint32_t o = orig_of[v];
    atomicOr(reinterpret_cast<unsigned long long*>(dirty_next) + (o >> 6), 1ull << (o & 63));
  }
}

__device__ __forceinline__ void mark_changed(uint64_t* mod_next, uint64_t* dirty_next,
                                             const uint32_t* orig_of, uint32_t v) {
  HANF_DCHECK(!dirty_next || orig_of);
  atomicOr(reinterpret_cast<unsigned long long*>(mod_next) + (v >> 6), 1ull << (v & 63));
  if (dirty_next) {
    const uint32_t o = orig_of[v];
    atomicOr(reinterpret_cast<unsigned long long*>(dirty_next) + (o >> 6), 1ull << (o & 63));
  }
}

// Estimate of a changed counter into its slot (and, for relabelled shards,
// into every peer's estimate array: their commits re-sum all blocks).
__device__ __forceinline__ void push_estimate(const UnionArgs& args, uint32_t v, double e) {
  const uint32_t slot = est_slot(args.est_index, v);
  args.est[slot] = e;
  if (args.peers.push_est)
    for (uint32_t p = 0; p < args.peers.count; ++p) args.peers.est[p][slot] = e;
}

// Max over a split node's chunk partials and its own counter (one warp),
// then the usual commit.  Partials were written by other warps of the same
// launch: read through L2 (ld.cg) after the ticket handshake.
template <class Lay, bool kVec16>
__device__ __forceinline__ void finalize_hub(const UnionArgs& args, uint32_t h, uint32_t lane) {
  constexpr int NL = Lay::kLimbs;
  constexpr int NW = Lay::kWords;
  const uint32_t v = args.hub_nodes[h];
  const uint32_t first = args.hub_first[h];
  const uint32_t count = args.hub_count[h];
  HANF_DCHECK(v < args.row_limit && v != args.zero_row && count >= 1);
  const uint32_t words = args.pitch;
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
      if (changed || stale) {
        const uint64_t off = static_cast<uint64_t>(v) * words + woff;
        store_chunk<Lay, kVec16>(args.next + off, acc);
        for (uint32_t p = 0; p < args.peers.count; ++p)
          if (peer_wants(args.peers, p, v)) store_chunk<Lay, kVec16>(args.peers.next[p] + off, acc);
      }
      if (args.est && (changed || (stale && args.peers.push_est)))
        push_estimate(args, v, estimate_limbs<Lay>(acc, args.ep));
    }
  }
  if (lane == 0 && any_changed) mark_changed(args.mod_next, args.dirty_next, args.orig_of, v);
}

// Folds the G lanes of each node, then either stores a hub chunk's partial
// or compares with the old counter (own_load) and commits the changed /
// stale rows, estimating changed counters from registers.
template <class Lay, bool kVec16, class OwnLoad>
__device__ __forceinline__ void node_commit(const UnionArgs& args, const WarpTask& task, bool hub,
                                            bool lead, uint32_t v, bool stale,
                                            uint32_t (&acc)[Lay::kLimbs], uint32_t woff,
                                            uint32_t G, bool live, bool& any_changed,
                                            OwnLoad own_load) {
  constexpr int NL = Lay::kLimbs;
  const uint32_t words = args.pitch;
  if (live)  // (all-zero accumulators need no butterfly)
    for (uint32_t off = G >> 1; off >= 1; off >>= 1) shfl_max<Lay>(acc, off);
  if (hub) {
    if ((threadIdx.x & 31) == 0)
      store_chunk<Lay, kVec16>(args.partials + static_cast<uint64_t>(task.item) * words + woff,
                               acc);
  } else {
    // The fold started from zero: the node's own counter is folded in only
    // now, and only where it can matter.  An all-zero chunk maximum (no
    // successor gathered - skipped or none - or only zero chunks) cannot
    // change the counter, so unless the next slot is stale the own counter
    // is not even read: the skip sweep's tail steps touch no counters of
    // unaffected nodes, and dense steps read each own counter once.
    const bool need = lead && (stale || limbs_nonzero<Lay>(acc));
    uint32_t own[NL];
    own_load(own, need);
    bool changed = false;
    if (need) {
      swar_max<Lay>(acc, own);
      changed = limbs_differ<Lay>(acc, own);
    }
    any_changed |= changed;
    if (changed || (lead && stale)) {
      const uint64_t off = static_cast<uint64_t>(v) * words + woff;
      if (args.chunks == 1)
        store_counter<Lay>(args.next + off, acc);
      else
        store_chunk<Lay, kVec16>(args.next + off, acc);
      // sharded peer-push: the same row into every peer's next generation
      for (uint32_t p = 0; p < args.peers.count; ++p) {
        if (!peer_wants(args.peers, p, v)) continue;
        if (args.chunks == 1)
          store_counter<Lay>(args.peers.next[p] + off, acc);
        else
          store_chunk<Lay, kVec16>(args.peers.next[p] + off, acc);
      }
    }
    // (relabelled shards keep estimates per generation: a stale row's
    // estimate is rewritten with its row)
    if (args.est && (changed || (lead && stale && args.peers.push_est)))
      push_estimate(args, v, estimate_limbs<Lay>(acc, args.ep));
  }
}

// Sets the node's modified bit; the last chunk of a split node to finish
// folds all its partials (ticket handshake).
template <class Lay, bool kVec16>
__device__ __forceinline__ void task_finish(const UnionArgs& args, const WarpTask& task, bool hub,
                                            uint32_t v, bool any_changed, uint32_t lane) {
  mark_changed_warp(args.mod_next, args.dirty_next, args.orig_of, v, any_changed);
  if (hub) {
    const uint32_t h = args.chunk_hub[task.item];
    uint32_t last = 0;
    if (lane == 0) {
      __threadfence();
      last = atomicAdd(args.hub_ticket + h, 1u) == args.hub_count[h] - 1;
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {
      __threadfence();
      finalize_hub<Lay, kVec16>(args, h, lane);
      if (lane == 0) args.hub_ticket[h] = 0;  // ready for the next step
    }
  }
}

// SKIP: compiled for the skip sweeps (args.check_mod); the dense sweep's
// instantiation carries no probe code (register pressure)
template <int R, int NREG, int U, int GMODE, bool kVec16, int MINB, bool PF, bool SKIP>
__device__ __forceinline__ void union_task(const UnionArgs& args, uint32_t task_index,
                                           uint32_t lane, const uint64_t* summ) {
  using Lay = Layout<R, NREG>;
  constexpr int NL = Lay::kLimbs;
  constexpr int NW = Lay::kWords;
  using G_t = Gather<Lay, GMODE, kVec16>;
  HANF_DCHECK(task_index < args.num_wtasks);
  const WarpTask task = args.wtasks[task_index];
  const bool hub = task.nodes == 0;
  if constexpr (SKIP) {
    // segmented tasks: a segment with no modified row among its nodes and
    // their successors has nothing to gather and nothing stale to rewrite
    if (args.seg_live) {
      const uint32_t v0 = hub ? args.hub_node[task.item] : args.order[task.item];
      if (!args.seg_live[v0 >> args.seg_shift]) return;
    }
  }
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
  HANF_DCHECK(v < args.row_limit && (!active || v != zero_row));
  const bool lead = active && sub == 0 && !hub;
  bool stale = false;
  if (lead && args.stale_valid) stale = (args.mod_cur[v >> 6] >> (v & 63)) & 1;
  const uint64_t* __restrict__ cur = args.cur;
  const uint32_t* __restrict__ ids = args.tos + task.tos + lane;
  const uint32_t words = args.pitch;
  const uint32_t trips = task.trips;

  bool any_changed = false;
  for (uint32_t ch = 0; ch < args.chunks; ++ch) {
    const uint32_t woff = ch * NW;
    uint32_t acc[NL];
    zero_limbs<Lay>(acc);  // the own counter joins in node_commit
    bool task_live = !SKIP;  // warp-uniform: some lane gathered something
    // PF: the ids of trip group i+U are requested before group i's gathers
    // so the id load latency overlaps the gathers instead of preceding them.
    uint32_t wn[U];
    if (PF) {
#pragma unroll
      for (int j = 0; j < U; ++j) wn[j] = (j < trips) ? ld_stream_u32(ids + 32 * j) : zero_row;
    }
    for (uint32_t i = 0; i < trips; i += U) {
      uint32_t w[U];
      if (PF) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          w[j] = wn[j];
          wn[j] = (i + U + j < trips) ? ld_stream_u32(ids + 32 * (i + U + j)) : zero_row;
        }
      } else {
#pragma unroll
        for (int j = 0; j < U; ++j)
          w[j] = (i + j < trips) ? ld_stream_u32(ids + 32 * (i + j)) : zero_row;
      }
      if constexpr (SKIP) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          // mode 3: the L1-resident summary (one bit per 2^summ_shift rows)
          // rules most successors out before the bitmap probe reaches L2
          bool keep = true;
          if (summ)  // shared memory: a random probe costs a bank, not an L1 line
            keep = (summ[w[j] >> (args.summ_shift + 6)] >> ((w[j] >> args.summ_shift) & 63)) & 1;
          if (keep) keep = (__ldg(args.mod_cur + (w[j] >> 6)) >> (w[j] & 63)) & 1;
          if (!keep) w[j] = zero_row;
        }
        // a trip group with no live successor in any lane costs nothing
        // more: late skip sweeps are mostly id loads and probes
        bool live = false;
#pragma unroll
        for (int j = 0; j < U; ++j) live |= w[j] != zero_row;
        if (!__any_sync(0xffffffffu, live)) continue;
        task_live = true;
      }
      G_t g[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        HANF_DCHECK(w[j] < args.row_limit);
        g[j].issue(cur, w[j], words, woff);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        uint32_t y[NL];
        g[j].extract(y, w[j]);
        swar_max<Lay>(acc, y);
      }
    }
    node_commit<Lay, kVec16>(args, task, hub, lead, v, stale, acc, woff, G, task_live, any_changed,
                             [&](uint32_t (&own)[NL], bool need) {
                               const uint32_t r = need ? v : zero_row;
                               G_t g;
                               g.issue(cur, r, words, woff);
                               g.extract(own, r);
                             });
  }
  task_finish<Lay, kVec16>(args, task, hub, v, any_changed, lane);
}

// ---------------------------------------------------------------------------
// Union sweep over the byte layout (ByteLayout<M>).  Same tasks and TOS as
// union_task: TOS row i holds the ids of trip i of the warp's 32 streams
// (stream l: node slot l >> lg, sub-stream l & (G-1)).  A counter row is M
// bytes, read by a group of Q = M/16 lanes (16 registers each, one 16-byte
// load), so a gathered counter costs one coalesced M-byte access and three
// instructions per four registers per lane.  Group g walks the streams
// [gQ, gQ + Q) one after the other with a single accumulator: streams of a
// node are consecutive, so a node of G < Q streams is committed every G
// streams, and a node of G >= Q streams is combined across its G/Q groups
// by a butterfly at the end.  The node's group then compares with the old
// counter, writes a changed or stale row (one coalesced store), sums the
// estimator's integer terms of its registers and sets the modified bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 shfl_xor4(const uint4& v, int off) {
  return make_uint4(__shfl_xor_sync(0xffffffffu, v.x, off), __shfl_xor_sync(0xffffffffu, v.y, off),
                    __shfl_xor_sync(0xffffffffu, v.z, off), __shfl_xor_sync(0xffffffffu, v.w, off));
}

template <int Q>
__device__ __forceinline__ uint32_t group_or(uint32_t x) {
#pragma unroll
  for (int off = 1; off < Q; off <<= 1) x |= __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// Group commit of light node slot j (warp-synchronous: every lane calls it;
// `act` is uniform within a group): the row store happens here; the
// estimate's integer terms come back summed over the group so that the
// caller can finish estimates and set modified bits for a whole warp of
// nodes at once (one double division per lane instead of one per group).
struct ByteCommit {
  uint64_t sum;   // sum of 2^(31 - M_j) over the node's registers
  uint32_t zeros;
  uint32_t v;
  bool want;      // the estimate must be written
  bool changed;
};

template <int Q>
__device__ __forceinline__ ByteCommit commit_bytes(const UnionArgs& args, const WarpTask& task,
                                                   uint32_t j, bool act, bool live, const uint4& acc,
                                                   uint32_t k) {
  const uint4* __restrict__ cur = reinterpret_cast<const uint4*>(args.cur);
  act = act && j < task.nodes;
  ByteCommit o{0, 0, args.zero_row, false, false};
  bool st = false;
  if (act) {
    o.v = args.order[task.item + j];
    HANF_DCHECK(o.v < args.zero_row);
    if (args.stale_valid) st = (args.mod_cur[o.v >> 6] >> (o.v & 63)) & 1;
  }
  const bool nz = group_or<Q>(live && (acc.x | acc.y | acc.z | acc.w) != 0);
  const bool need = act && (st || nz);
  uint4 own = make_uint4(0, 0, 0, 0);
  if (need) own = __ldg(cur + static_cast<uint64_t>(o.v) * Q + k);
  const uint4 nx = byte_max4(acc, own);
  o.changed =
      group_or<Q>(need && ((nx.x ^ own.x) | (nx.y ^ own.y) | (nx.z ^ own.z) | (nx.w ^ own.w)));
  if (o.changed || (act && st)) {
    const uint64_t off = static_cast<uint64_t>(o.v) * Q + k;
    reinterpret_cast<uint4*>(args.next)[off] = nx;
    for (uint32_t p = 0; p < args.peers.count; ++p)
      if (peer_wants(args.peers, p, o.v)) reinterpret_cast<uint4*>(args.peers.next[p])[off] = nx;
  }
  o.want = args.est && (o.changed || (act && st && args.peers.push_est));
  if (__any_sync(0xffffffffu, o.want)) {
    byte_terms(nx, o.sum, o.zeros);
#pragma unroll
    for (int off = 1; off < Q; off <<= 1) {
      o.sum += __shfl_xor_sync(0xffffffffu, o.sum, off);
      o.zeros += __shfl_xor_sync(0xffffffffu, o.zeros, off);
    }
  }
  return o;
}

__device__ __forceinline__ void finish_commit(const UnionArgs& args, const ByteCommit& o) {
  if (o.want)
    push_estimate(args, o.v,
                  finish_estimate(args.ep, __dmul_rn(static_cast<double>(o.sum), 0x1p-31), o.zeros));
  if (o.changed) mark_changed(args.mod_next, args.dirty_next, args.orig_of, o.v);
}

template <int M, int U, bool SKIP>
__device__ __forceinline__ void union_task_bytes(const UnionArgs& args, uint32_t task_index,
                                                 uint32_t lane, const uint64_t* summ) {
  using Lay = ByteLayout<M>;
  constexpr int Q = M / 16;  // lanes per counter row
  HANF_DCHECK(task_index < args.num_wtasks);
  const WarpTask task = args.wtasks[task_index];
  const bool hub = task.nodes == 0;
  if constexpr (SKIP) {
    if (args.seg_live) {
      const uint32_t v0 = hub ? args.hub_node[task.item] : args.order[task.item];
      if (!args.seg_live[v0 >> args.seg_shift]) return;
    }
  }
  const uint32_t lg = hub ? 5u : task.lg;
  const uint32_t G = 1u << lg;
  const uint32_t zero_row = args.zero_row;
  const uint32_t grp = lane / Q, k = lane % Q;
  const uint4* __restrict__ cur = reinterpret_cast<const uint4*>(args.cur);
  const uint32_t trips = task.trips;
  bool task_live = !SKIP;
  uint4 acc = make_uint4(0, 0, 0, 0);
  ByteCommit mine{0, 0, zero_row, false, false};  // G < Q: this lane's node of the warp
  // ids of the next trip group are requested before the current group's
  // gathers (across the stream passes too)
  const uint32_t* __restrict__ base = args.tos + task.tos + grp * Q;
  uint32_t wn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) wn[u] = u < static_cast<int>(trips) ? __ldg(base + 32 * u) : zero_row;
#pragma unroll 1
  for (uint32_t s = 0; s < static_cast<uint32_t>(Q); ++s) {
#pragma unroll 1
    for (uint32_t i = 0; i < trips; i += U) {
      uint32_t w[U];
      // next group: trips i+U.. of this stream, or the first of the next
      const bool wrap = i + U >= trips;
      const uint32_t ns = wrap ? s + 1 : s, ni = wrap ? 0 : i + U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        w[u] = wn[u];
        wn[u] = ns < static_cast<uint32_t>(Q) && ni + u < trips ? __ldg(base + ns + 32 * (ni + u))
                                                                : zero_row;
      }
      if constexpr (SKIP) {
        bool live = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bool keep = true;
          if (summ)
            keep = (summ[w[u] >> (args.summ_shift + 6)] >> ((w[u] >> args.summ_shift) & 63)) & 1;
          if (keep) keep = (__ldg(args.mod_cur + (w[u] >> 6)) >> (w[u] & 63)) & 1;
          if (!keep) w[u] = zero_row;
          live |= w[u] != zero_row;
        }
        if (!__any_sync(0xffffffffu, live)) continue;
        task_live = true;
      }
      uint4 y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        HANF_DCHECK(w[u] <= zero_row);
        y[u] = __ldg(cur + static_cast<uint64_t>(w[u]) * Q + k);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = byte_max4(acc, y[u]);
    }
    // a node of G < Q streams ends with stream grp*Q + s; lane s / G of
    // the group keeps its commit for the warp-wide finish
    if (G < static_cast<uint32_t>(Q) && ((s + 1) & (G - 1)) == 0) {
      const uint32_t first = grp * Q + s + 1 - G;
      const ByteCommit o = commit_bytes<Q>(args, task, first >> lg, true, task_live, acc, k);
      if (k == s >> lg) mine = o;
      acc = make_uint4(0, 0, 0, 0);
    }
  }
  if (G < static_cast<uint32_t>(Q)) {
    finish_commit(args, mine);
    return;
  }
  // nodes of G >= Q streams: combine the G/Q groups of each node
  if (task_live)
    for (uint32_t off = 1; off < G / Q; off <<= 1) acc = byte_max4(acc, shfl_xor4(acc, off * Q));
  if (!hub) {
    const ByteCommit o =
        commit_bytes<Q>(args, task, (grp * Q) >> lg, ((grp * Q) & (G - 1)) == 0, task_live, acc, k);
    if (k == 0) finish_commit(args, o);
    return;
  }
  // hub chunk: the partial maximum (every group holds it), then the ticket
  if (grp == 0)
    reinterpret_cast<uint4*>(args.partials)[static_cast<uint64_t>(task.item) * Q + k] = acc;
  const uint32_t h = args.chunk_hub[task.item];
  uint32_t last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(args.hub_ticket + h, 1u) == args.hub_count[h] - 1;
  }
  if (__shfl_sync(0xffffffffu, last, 0)) {
    __threadfence();
    finalize_hub<Lay, true>(args, h, lane);
    if (lane == 0) args.hub_ticket[h] = 0;
  }
}

template <int M, int MINB, bool SKIP>
__global__ void __launch_bounds__(256, MINB) union_kernel_bytes(const UnionArgs args) {
  extern __shared__ uint64_t summ_smem[];
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t* summ = nullptr;
  if (SKIP && args.summ) {
    for (uint32_t i = threadIdx.x; i < args.summ_words; i += blockDim.x) summ_smem[i] = args.summ[i];
    __syncthreads();
    summ = summ_smem;
  }
  if (args.task_list) {
    const uint32_t count = *args.task_count;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = gw; i < count; i += nw)
      union_task_bytes<M, 4, SKIP>(args, args.task_list[i], lane, summ);
    return;
  }
  if (SKIP && summ) {
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = gw; t < args.num_wtasks; t += nw) union_task_bytes<M, 4, SKIP>(args, t, lane, summ);
    return;
  }
  if (gw >= args.num_wtasks) return;
  union_task_bytes<M, 4, SKIP>(args, gw, lane, summ);
}

// One warp per task; with a task list (the worklist step's hub chunks) the
// warps stride over the listed task indices instead.
template <int R, int NREG, int U, int GMODE, bool kVec16, int MINB = 1, bool PF = false,
          bool SKIP = false>
__global__ void __launch_bounds__(256, MINB) union_kernel(const UnionArgs args) {
  extern __shared__ uint64_t summ_smem[];
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t* summ = nullptr;
  if (SKIP && args.summ) {  // mode 3: the modified-bitmap summary, staged once per CTA
    for (uint32_t i = threadIdx.x; i < args.summ_words; i += blockDim.x) summ_smem[i] = args.summ[i];
    __syncthreads();
    summ = summ_smem;
  }
  if (args.task_list) {
    const uint32_t count = *args.task_count;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = gw; i < count; i += nw)
      union_task<R, NREG, U, GMODE, kVec16, MINB, PF, SKIP>(args, args.task_list[i], lane, summ);
    return;
  }
  if (SKIP && summ) {  // persistent grid (launch_union): the staging is paid once per CTA
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = gw; t < args.num_wtasks; t += nw)
      union_task<R, NREG, U, GMODE, kVec16, MINB, PF, SKIP>(args, t, lane, summ);
    return;
  }
  if (gw >= args.num_wtasks) return;
  union_task<R, NREG, U, GMODE, kVec16, MINB, PF, SKIP>(args, gw, lane, summ);
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

// A dense sweep launched with the generation's hot row prefix as an L2
// access-policy window (persisting hits, streaming misses; hanf_engine.cu
// choose_l2_window): a launch attribute, so CUDA graph captures keep it.
template <class K>
cudaError_t launch_windowed(K kernel, uint32_t blocks, size_t smem, cudaStream_t s,
                            const UnionArgs& a) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(blocks);
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow.base_ptr = const_cast<uint64_t*>(a.cur);
  at[0].val.accessPolicyWindow.num_bytes = a.l2_window_bytes;
  at[0].val.accessPolicyWindow.hitRatio = 1.0f;
  at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kernel, a);
}

template <int M, int MINB>
cudaError_t union_launch_bytes(UnionArgs a, cudaStream_t s) {
  a.chunks = 1;
  if (a.num_wtasks == 0) return cudaSuccess;
  uint32_t blocks = (a.num_wtasks + 7) / 8;
  if (a.task_list && blocks > 148 * 4) blocks = 148 * 4;
  if (a.summ && blocks > 148 * 4) blocks = 148 * 4;  // persistent (mode 3)
  const size_t smem = a.summ ? sizeof(uint64_t) * a.summ_words : 0;
  if (a.check_mod) {
    union_kernel_bytes<M, (MINB > 4 ? 4 : MINB), true><<<blocks, 256, smem, s>>>(a);
  } else if (a.l2_window_bytes) {
    return launch_windowed(union_kernel_bytes<M, MINB, false>, blocks, smem, s, a);
  } else {
    union_kernel_bytes<M, MINB, false><<<blocks, 256, smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <int R, int NREG, int U, int GM, bool V, int MINB = 1, bool PF = false>
cudaError_t union_launch(UnionArgs a, uint32_t chunks, cudaStream_t s) {
  a.chunks = chunks;
  if (chunks != 1) a.est = nullptr;  // estimates need the whole counter in registers
  if (a.num_wtasks == 0) return cudaSuccess;
  uint32_t blocks = (a.num_wtasks + 7) / 8;
  if (a.task_list && blocks > 148 * 4) blocks = 148 * 4;
  if (a.summ && blocks > 148 * 4) blocks = 148 * 4;  // persistent (mode 3)
  const size_t smem = a.summ ? sizeof(uint64_t) * a.summ_words : 0;
  // the skip sweep carries the probe code: one CTA/SM fewer keeps it spill-free
  constexpr int SKIP_MINB = MINB > 4 ? 4 : MINB;
  if (a.check_mod && a.l2_window_bytes) {
    return launch_windowed(union_kernel<R, NREG, U, GM, V, SKIP_MINB, PF, true>, blocks, smem, s, a);
  } else if (a.check_mod) {
    union_kernel<R, NREG, U, GM, V, SKIP_MINB, PF, true><<<blocks, 256, smem, s>>>(a);
  } else if (a.l2_window_bytes) {
    return launch_windowed(union_kernel<R, NREG, U, GM, V, MINB, PF, false>, blocks, smem, s, a);
  } else {
    union_kernel<R, NREG, U, GM, V, MINB, PF, false><<<blocks, 256, smem, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace

bool fused_estimates(uint32_t register_bits, uint32_t registers) {
  return choose(register_bits, registers).chunks == 1;
}

bool byte_layout_supported(uint32_t register_bits, uint32_t registers) {
  return register_bits == 5 && registers >= 16 && registers <= 128;
}

// Rows of W = 3 words are padded to 4 (one aligned 32-byte sector per
// counter: +5% on the DRAM-bound BA graph, profiles/r01_row_pitch.md);
// every other layout keeps the reference's dense packing.
uint32_t row_pitch(uint32_t register_bits, uint32_t registers, uint32_t words, bool bytes) {
  if (bytes) return registers / 8;
  if (choose(register_bits, registers).chunks != 1) return words;
  return words == 3 ? 4 : words;
}

// The measured best gather per layout (profiles/r01_*): 16-byte windows
// for m = 64 (3 x LDG.128 per 40-byte counter, U = 3 in flight, <= 48
// registers), aligned 256-bit loads for padded W = 3 rows, 16-byte vector
// loads where rows are 16-byte aligned, per-word loads otherwise.
cudaError_t launch_union(const UnionArgs& args, uint32_t register_bits, uint32_t registers,
                         cudaStream_t s, uint64_t* launches) {
  const KernelChoice k = choose(register_bits, registers);
  if (args.num_wtasks == 0) return cudaSuccess;
  ++*launches;
  if (args.bytes) switch (registers) {
      case 16: return union_launch_bytes<16, 5>(args, s);
      case 32: return union_launch_bytes<32, 5>(args, s);
      case 64: return union_launch_bytes<64, 5>(args, s);
      case 128: return union_launch_bytes<128, 3>(args, s);
      default: return cudaErrorInvalidValue;
    }
  const uint32_t ch = static_cast<uint32_t>(k.chunks);
  const bool single = ch == 1;
  if (single && args.pitch % 4 == 0) switch (k.r * 1000 + k.nreg) {
      case 5032: return union_launch<5, 32, 4, 3, false, 1, true>(args, ch, s);
      case 6032: return union_launch<6, 32, 4, 3, false, 1, true>(args, ch, s);
      case 7032: return union_launch<7, 32, 4, 3, false, 1, true>(args, ch, s);
      default: break;
    }
  switch (k.r * 1000 + k.nreg) {
    case 5016: return union_launch<5, 16, 4, 0, true>(args, ch, s);
    case 5032:
      if (single) return union_launch<5, 32, 4, 1, false, 1, true>(args, ch, s);
      return union_launch<5, 32, 4, 0, false>(args, ch, s);
    case 5064:
      // U = 2, <= 48 registers (5 CTAs/SM), next-trip id prefetch: config 5
      // 54.5 ms against 55.6 (U = 3), 57.8 (U = 2, 6 CTAs/SM), 59.9 (U = 4)
      // and 67.7 (U = 3, 6 CTAs/SM); config 2 packed 0.181 vs 0.184 ms
      if (single) return union_launch<5, 64, 2, 1, false, 5, true>(args, ch, s);
      return union_launch<5, 64, 4, 0, false>(args, ch, s);
    case 5128: return union_launch<5, 128, 2, 0, true, 3, true>(args, ch, s);
    case 6016: return union_launch<6, 16, 4, 0, true>(args, ch, s);
    case 6032: return union_launch<6, 32, 4, 0, false>(args, ch, s);
    case 7016: return union_launch<7, 16, 4, 0, true>(args, ch, s);
    case 7032: return union_launch<7, 32, 4, 0, true>(args, ch, s);
    case 7064: return union_launch<7, 64, 2, 0, false>(args, ch, s);
    default: return union_launch<8, 16, 4, 0, true>(args, ch, s);
  }
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
  EstimateParams p{args.alpha, args.m, args.registers, args.register_bits, args.pitch,
                   args.log_table};
  double e = 0.0;
  if (v < args.n) {
    if ((word >> t) & 1) {
      const uint64_t row = args.row_of ? args.row_of[v] : v;  // v is an original id
      if constexpr (M < 0)
        e = estimate_counter_bytes<-M>(args.counters + row * args.pitch, p);
      else if constexpr (M > 0)
        e = estimate_counter_r5<M>(args.counters + row * args.pitch, p);
      else
        e = estimate_counter_generic(args.counters + row * args.pitch, p);
      args.est[v] = e;
    } else if (args.block_sums) {
      e = args.est[v];
    }
  }
  if (!args.block_sums) return;  // (the caller sums the blocks itself)
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
  if (args.bytes) {
    switch (args.registers) {
      case 16: estimate_kernel<-16><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args); break;
      case 32: estimate_kernel<-32><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args); break;
      case 64: estimate_kernel<-64><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args); break;
      default: estimate_kernel<-128><<<static_cast<uint32_t>(blocks), 64, 0, s>>>(args); break;
    }
    return cudaGetLastError();
  }
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
// Step epilogue, one launch: CTA c owns the fixed range of 64-counter blocks
// [c*256, c*256+256) (one thread per block).
//  1. blocks in [b0, b1) whose dirty word is non-zero get their sum
//     recomputed from the cached per-counter estimates, sequentially in
//     index order (engine.hpp:109-111); other blocks keep their cached sum
//     (engine.hpp:105);
//  2. the CTA reduces its range (fixed tree) and the popcount of the
//     modified bitmap over it (engine.hpp:202-208) into partial[c];
//  3. the last CTA to finish (ticket) reduces the partials in a fixed order
//     into out->total / out->count and re-arms the ticket.
// Every order is fixed, so N(t) is bit-identical across runs; the
// reference's own sequential total is redone on the host under exact_sum.
// ---------------------------------------------------------------------------
// Fixed-order CTA reductions over kFinishThreads values (deterministic).
__device__ __forceinline__ double cta_tree_sum(double v, double* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int w = kFinishThreads / 2; w >= 1; w >>= 1) {
    if (t < w) sh[t] = __dadd_rn(sh[t], sh[t + w]);
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ unsigned long long cta_count_sum(unsigned long long v,
                                                            unsigned long long* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int w = kFinishThreads / 2; w >= 1; w >>= 1) {
    if (t < w) sh[t] += sh[t + w];
    __syncthreads();
  }
  const unsigned long long r = sh[0];
  __syncthreads();
  return r;
}

// CTA c owns the 64-counter blocks [64c, 64c + 64): all kFinishThreads
// threads stage the dirty blocks' estimates (row k = block 64c + k, 64
// doubles, row-major so consecutive threads copy consecutive addresses),
// then thread k < 64 redoes block k's sum sequentially from shared memory.
__global__ void __launch_bounds__(kFinishThreads) finish_kernel(const FinishArgs a) {
  __shared__ double sh[kFinishThreads];
  __shared__ unsigned long long shc[kFinishThreads];
  __shared__ double tile[kFinishBlocks * (64 + 1)];  // row = one block's 64 estimates
  __shared__ uint64_t dirty[kFinishBlocks];
  __shared__ bool is_last;
  const uint32_t t = threadIdx.x;
  const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kFinishBlocks;
  if (t < kFinishBlocks) {
    const uint64_t b = b0 + t;
    dirty[t] = (b < a.blocks && b >= a.b0 && b < a.b1) ? (a.all_dirty ? ~0ull : a.bits[b]) : 0;
  }
  __syncthreads();
  if (a.est) {
    for (uint32_t k = t; k < kFinishBlocks * 64; k += kFinishThreads) {
      const uint32_t row = k >> 6, col = k & 63;
      if (dirty[row] == 0) continue;
      const uint64_t e = (b0 + row) * 64 + col;
      if (e < a.n) {
        const uint32_t dst =
            static_cast<uint32_t>(__cvta_generic_to_shared(&tile[row * 65 + col]));
        const uint64_t src = a.perm ? a.perm[e] : e;  // estimates in row order
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(a.est + src));
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  double sum = 0.0;
  unsigned long long cnt = 0;
  const uint64_t b = b0 + t;
  if (t < kFinishBlocks && b < a.blocks) {
    if (a.clear) a.clear[b] = 0;
    const uint64_t word = a.bits[b];
    cnt = __popcll(word);
    if (a.est && (word != 0 || a.all_dirty) && b >= a.b0 && b < a.b1) {
      const uint64_t first = b * 64;
      const uint32_t last = a.n - first < 64 ? static_cast<uint32_t>(a.n - first) : 64u;
      const double* row = tile + t * 65;
      for (uint32_t i = 0; i < last; ++i) sum = __dadd_rn(sum, row[i]);  // engine.hpp:109-111
      a.block_sums[b] = sum;
    } else {
      sum = a.block_sums[b];
    }
    if (a.host_sums) a.host_sums[b] = sum;
  }
  const double cta_sum = cta_tree_sum(sum, sh);
  const unsigned long long cta_cnt = cta_count_sum(cnt, shc);
  if (threadIdx.x == 0) {
    a.out->partial_sum[blockIdx.x] = cta_sum;
    a.out->partial_count[blockIdx.x] = cta_cnt;
    __threadfence();
    is_last = atomicAdd(&a.out->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double acc = 0.0;
  unsigned long long c = 0;
  for (uint32_t i = threadIdx.x; i < gridDim.x; i += kFinishThreads) {
    acc = __dadd_rn(acc, __ldcg(&a.out->partial_sum[i]));
    c += __ldcg(&a.out->partial_count[i]);
  }
  const double total = cta_tree_sum(acc, sh);
  const unsigned long long count = cta_count_sum(c, shc);
  if (threadIdx.x == 0) {
    a.out->total = total;
    a.out->count = count;
    a.out->ticket = 0;
    if (a.host_out) {  // visible to the host once the stream has synchronised
      a.host_out->total = total;
      a.host_out->count = count;
    }
  }
}

__global__ void derive_dirty_kernel(const uint64_t* __restrict__ rows,
                                    const uint32_t* __restrict__ order, uint64_t words, uint64_t n,
                                    unsigned long long* __restrict__ dirty) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
       w += stride) {
    uint64_t bits = rows[w];
    while (bits) {
      const uint64_t r = w * 64 + __ffsll(static_cast<long long>(bits)) - 1;
      bits &= bits - 1;
      if (r < n) {
        const uint32_t o = order[r];
        atomicOr(dirty + (o >> 6), 1ull << (o & 63));
      }
    }
  }
}

cudaError_t launch_derive_dirty(const uint64_t* rows, const uint32_t* order, uint64_t words,
                                uint64_t n, uint64_t* dirty, cudaStream_t s, uint64_t* launches) {
  if (words == 0) return cudaSuccess;
  uint64_t blocks = (words + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  derive_dirty_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(
      rows, order, words, n, reinterpret_cast<unsigned long long*>(dirty));
  ++*launches;
  return cudaGetLastError();
}

// One warp per segment: does mod_cur have a bit in [seg_min, seg_max]?
__global__ void segment_live_kernel(const uint64_t* __restrict__ mod_cur,
                                    const uint32_t* __restrict__ seg_min,
                                    const uint32_t* __restrict__ seg_max, uint32_t segs,
                                    uint32_t* __restrict__ live) {
  const uint32_t sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (sg >= segs) return;
  const uint32_t lo = seg_min[sg], hi = seg_max[sg];
  bool any = false;
  if (lo <= hi) {
    const uint32_t w0 = lo >> 6, w1 = hi >> 6;
    for (uint32_t w = w0 + lane; w <= w1; w += 32) {
      uint64_t m = mod_cur[w];
      if (w == w0) m &= ~0ull << (lo & 63);
      if (w == w1) m &= ~0ull >> (63 - (hi & 63));
      any |= m != 0;
      if (__any_sync(__activemask(), any)) break;
    }
  }
  any = __any_sync(0xffffffffu, any);
  if (lane == 0) live[sg] = any ? 1u : 0u;
}

cudaError_t launch_segment_live(const uint64_t* mod_cur, const uint32_t* seg_min,
                                const uint32_t* seg_max, uint32_t segs, uint32_t* live,
                                cudaStream_t s, uint64_t* launches) {
  segment_live_kernel<<<(segs + 7) / 8, 256, 0, s>>>(mod_cur, seg_min, seg_max, segs, live);
  ++*launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Task-scan step (late iterations of large graphs, step mode 4).  Instead of
// walking every task, one flat, coalesced pass over the TOS finds the id
// rows holding a successor modified by the previous step (summary bit in
// shared memory, then the bitmap) and lists their tasks (every chunk of a
// hub, so the hub ticket completes); the skip sweep then runs on that list
// only (union_kernel task_list).  Nodes changed by the previous step whose
// task is not listed cannot change now, but their next slot is stale:
// stale_fixup copies their row (cur -> next) afterwards.  Same bits as the
// full skip sweep (engine.hpp:173: an unmodified successor adds nothing).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream_u4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// Lists the task holding TOS row `row` (and every chunk of its hub).
__device__ __noinline__ void list_task_of_row(const TaskScanArgs& a, uint64_t row) {
  const uint64_t pos = row * 32;
  uint32_t lo = 0, hi = a.num_wtasks - 1;  // last t with wtasks[t].tos <= pos
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    if (a.wtasks[mid].tos <= pos) lo = mid; else hi = mid - 1;
  }
  HANF_DCHECK(a.wtasks[lo].tos <= pos && pos < a.wtasks[lo].tos + 32ull * a.wtasks[lo].trips);
  uint32_t first = lo, count = 1;
  if (a.wtasks[lo].nodes == 0) {  // hub chunk: every chunk of its hub
    const uint32_t h = a.chunk_hub[a.wtasks[lo].item];
    first = a.hub_first[h];
    count = a.hub_count[h];
  }
  for (uint32_t t = first; t < first + count; ++t)
    if (atomicExch(a.flags + t, 1u) == 0u) a.list[atomicAdd(a.count, 1u)] = t;
}

// Each warp streams 512-byte pieces (four TOS rows; lane l holds ids
// 4l..4l+3, so eight lanes share a row), four pieces in flight.
__global__ void __launch_bounds__(512) task_scan_kernel(const TaskScanArgs a) {
  extern __shared__ uint64_t summ_sm[];
  for (uint32_t i = threadIdx.x; i < a.summ_words; i += blockDim.x) summ_sm[i] = a.summ[i];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t pieces = a.tos_words / 128;  // (tos_words is a multiple of 32)
  const uint64_t tail_rows = (a.tos_words % 128) / 32;
  constexpr uint32_t R = 4;
  auto probe = [&](uint32_t w) -> bool {
    bool hit = (summ_sm[w >> (a.summ_shift + 6)] >> ((w >> a.summ_shift) & 63)) & 1;
    if (hit) hit = (__ldg(a.mod_cur + (w >> 6)) >> (w & 63)) & 1;
    return hit;
  };
  for (uint64_t p0 = ((blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5) * R;
       p0 < pieces; p0 += warps * R) {
    uint4 q[R];
#pragma unroll
    for (uint32_t k = 0; k < R; ++k)
      q[k] = p0 + k < pieces ? ld_stream_u4(a.tos + (p0 + k) * 128 + 4 * lane)
                             : make_uint4(a.zero_row, a.zero_row, a.zero_row, a.zero_row);
#pragma unroll
    for (uint32_t k = 0; k < R; ++k) {
      const bool hit = probe(q[k].x) | probe(q[k].y) | probe(q[k].z) | probe(q[k].w);
      uint32_t rows = __ballot_sync(0xffffffffu, hit);  // lane group l / 8 = row
      while (rows) {
        const uint32_t l = __ffs(rows) - 1;
        rows &= ~(0xffu << (l & ~7u));
        if (lane == 0) list_task_of_row(a, (p0 + k) * 4 + l / 8);
      }
    }
  }
  // the last < 4 rows: warp 0
  if (blockIdx.x == 0 && threadIdx.x < 32)
    for (uint64_t r = pieces * 4; r < pieces * 4 + tail_rows; ++r) {
      const bool hit = probe(a.tos[r * 32 + lane]);
      if (__any_sync(0xffffffffu, hit) && lane == 0) list_task_of_row(a, r);
    }
}

cudaError_t launch_task_scan(const TaskScanArgs& a, cudaStream_t s, uint64_t* launches) {
  if (a.num_wtasks == 0) return cudaSuccess;
  const size_t smem = sizeof(uint64_t) * a.summ_words;
  task_scan_kernel<<<148 * 3, 512, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError();
}

// next[v] = cur[v] for every row changed by the previous step (mod_cur)
// that did not change now (mod_next): their next slot held generation t-2.
__global__ void stale_fixup_kernel(const uint64_t* __restrict__ mod_cur,
                                   const uint64_t* __restrict__ mod_next, uint64_t words,
                                   uint64_t n, uint32_t pitch, const uint64_t* __restrict__ cur,
                                   uint64_t* __restrict__ next) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
       w += stride) {
    uint64_t bits = mod_cur[w] & ~mod_next[w];
    while (bits) {
      const uint64_t v = w * 64 + __ffsll(static_cast<long long>(bits)) - 1;
      bits &= bits - 1;
      if (v >= n) break;
      for (uint32_t k = 0; k < pitch; ++k) next[v * pitch + k] = cur[v * pitch + k];
    }
  }
}

cudaError_t launch_stale_fixup(const uint64_t* mod_cur, const uint64_t* mod_next, uint64_t n,
                               uint32_t pitch, const uint64_t* cur, uint64_t* next, cudaStream_t s,
                               uint64_t* launches) {
  const uint64_t words = (n + 63) / 64;
  if (words == 0) return cudaSuccess;
  uint64_t blocks = (words + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  stale_fixup_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(mod_cur, mod_next, words, n,
                                                                    pitch, cur, next);
  ++*launches;
  return cudaGetLastError();
}

// Needed-rows bitmap of a shard (peer-push filter): bit v is set iff row v
// is a successor id in the shard's TOS, i.e. one of its nodes can gather
// row v (hub chunks and the worklist step read the same successors).
// Padding ids (>= n) are skipped; a bit already set costs a read, not an
// atomic.
__global__ void need_rows_kernel(const uint32_t* __restrict__ tos, uint64_t count, uint32_t n,
                                 unsigned long long* __restrict__ need) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += stride) {
    const uint32_t v = tos[i];
    if (v >= n) continue;
    const unsigned long long bit = 1ull << (v & 63);
    if (!(need[v >> 6] & bit)) atomicOr(need + (v >> 6), bit);
  }
}

cudaError_t launch_need_rows(const uint32_t* tos, uint64_t count, uint64_t n, uint64_t* need,
                             cudaStream_t s, uint64_t* launches) {
  cudaError_t e = cudaMemsetAsync(need, 0, sizeof(uint64_t) * ((n + 63) / 64), s);
  if (e != cudaSuccess || count == 0) return e;
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  need_rows_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(
      tos, count, static_cast<uint32_t>(n), reinterpret_cast<unsigned long long*>(need));
  ++*launches;
  return cudaGetLastError();
}

// Rows of bitmap `rows` (words [0, words)) that peer p needs, summed over
// the peers: need[p] holds `words` words, peer after peer (the peer-push
// filter's copies); the total goes to *out (zeroed by the caller).
__global__ void count_pushes_kernel(const uint64_t* __restrict__ rows,
                                    const uint64_t* __restrict__ need, uint64_t words,
                                    uint32_t peers, unsigned long long* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  unsigned long long c = 0;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
       w += stride) {
    const uint64_t r = rows[w];
    for (uint32_t p = 0; p < peers; ++p) c += __popcll(r & need[p * words + w]);
  }
  for (int off = 16; off >= 1; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_count_pushes(const uint64_t* rows, const uint64_t* need, uint64_t words,
                                uint32_t peers, uint64_t* out, cudaStream_t s, uint64_t* launches) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
  if (e != cudaSuccess || words == 0) return e;
  uint64_t blocks = (words + 255) / 256;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  count_pushes_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(
      rows, need, words, peers, reinterpret_cast<unsigned long long*>(out));
  ++*launches;
  return cudaGetLastError();
}

// Peer-push exchange, end of a sharded compute: the shard's bitmap words
// and block sums into every peer's arena, block sums into the local inbox
// too (whole words: no clearing or atomics on the receiving side).
__global__ void publish_kernel(const PublishArgs a) {
  const uint64_t words = a.w1 - a.w0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < words;
       i += stride) {
    const uint64_t w = a.w0 + i;
    if (a.mod_next) {
      const uint64_t bits = a.mod_next[w];
      for (uint32_t p = 0; p < a.count; ++p) a.peer_mod[p][w] = bits;
    }
    if (a.block_sums) {
      const double sum = a.block_sums[w];
      for (uint32_t p = 0; p < a.count; ++p) a.peer_sums[p][w] = sum;
      a.peer_sums[a.count][w] = sum;
    }
  }
}

cudaError_t launch_publish(const PublishArgs& a, cudaStream_t s, uint64_t* launches) {
  if (a.w1 <= a.w0) return cudaSuccess;
  uint64_t ctas = (a.w1 - a.w0 + 255) / 256;
  if (ctas > 148ull * 8) ctas = 148ull * 8;
  publish_kernel<<<static_cast<uint32_t>(ctas), 256, 0, s>>>(a);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_finish(const FinishArgs& a, cudaStream_t s, uint64_t* launches) {
  if (a.blocks == 0) return cudaSuccess;
  const uint64_t ctas = (a.blocks + kFinishBlocks - 1) / kFinishBlocks;
  finish_kernel<<<static_cast<uint32_t>(ctas), kFinishThreads, 0, s>>>(a);
  ++*launches;
  return cudaGetLastError();
}

// Reference packing of a byte-layout row: word w of the dense W-word row
// holds bits [64w, 64w + 64) of register j at bit 5j (hll.hpp:183-240).
__device__ __forceinline__ uint64_t pack_word(const uint8_t* row, uint32_t registers, uint64_t w) {
  uint64_t word = 0;
  const uint32_t j0 = static_cast<uint32_t>(64 * w / 5);
  const uint32_t j1 = static_cast<uint32_t>((64 * w + 63) / 5);
  for (uint32_t j = j0; j <= j1 && j < registers; ++j) {
    const int64_t sh = static_cast<int64_t>(5 * j) - static_cast<int64_t>(64 * w);
    const uint64_t r = row[j] & 31u;
    word |= sh >= 0 ? r << sh : r >> -sh;
  }
  return word;
}

__global__ void gather_rows_bytes_kernel(const uint64_t* __restrict__ counters,
                                         const uint32_t* __restrict__ perm, uint64_t first,
                                         uint64_t count, uint32_t pitch, uint32_t words,
                                         uint32_t registers, uint64_t* __restrict__ dst) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       k < count * words; k += stride) {
    const uint64_t i = k / words, w = k % words;
    const uint64_t row = perm ? perm[first + i] : first + i;
    dst[k] = pack_word(reinterpret_cast<const uint8_t*>(counters + row * pitch), registers, w);
  }
}

// Restore into the byte layout: limb q (registers 4q..4q+3) of a row from
// the reference packing.
__global__ void scatter_rows_bytes_kernel(const uint64_t* __restrict__ src,
                                          const uint32_t* __restrict__ perm, uint64_t count,
                                          uint32_t pitch, uint32_t words, uint32_t registers,
                                          uint64_t* __restrict__ counters) {
  const uint64_t limbs = 2ull * pitch;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       k < count * limbs; k += stride) {
    const uint64_t i = k / limbs, q = k % limbs;
    const uint64_t row = perm ? perm[i] : i;
    const uint64_t* in = src + i * words;
    uint32_t limb = 0;
    for (uint32_t b = 0; b < 4; ++b) {
      const uint32_t j = static_cast<uint32_t>(4 * q + b);
      if (j >= registers) break;
      const uint32_t bit = 5 * j, wi = bit >> 6, off = bit & 63;
      uint64_t v = in[wi] >> off;
      if (off + 5 > 64 && wi + 1 < words) v |= in[wi + 1] << (64 - off);
      limb |= static_cast<uint32_t>(v & 31u) << (8 * b);
    }
    reinterpret_cast<uint32_t*>(counters + row * pitch)[q] = limb;
  }
}

// Counter read-back under relabelling: row perm[first + i] -> dst row i.
__global__ void gather_rows_kernel(const uint64_t* __restrict__ counters,
                                   const uint32_t* __restrict__ perm, uint64_t first,
                                   uint64_t count, uint32_t pitch, uint32_t words,
                                   uint64_t* __restrict__ dst) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       k < count * words; k += stride) {
    const uint64_t i = k / words, w = k % words;
    const uint64_t row = perm ? perm[first + i] : first + i;
    dst[k] = counters[row * pitch + w];
  }
}

// bits [0, n) of a bitmap set, the rest of its words cleared
__global__ void all_bits_kernel(uint64_t* __restrict__ bits, uint64_t n) {
  const uint64_t words = (n + 63) / 64;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < words;
       w += stride)
    bits[w] = (w + 1) * 64 <= n ? ~0ull : (~0ull >> ((w + 1) * 64 - n));
}

// summ bit i = OR of the bitmap's rows [i << shift, (i + 1) << shift)
__global__ void summary_kernel(const uint64_t* __restrict__ bits, uint64_t words, uint32_t shift,
                               uint64_t summ_bits, uint32_t* __restrict__ summ32) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  uint64_t any = 0;
  if (i < summ_bits) {
    const uint64_t w0 = (i << shift) >> 6, w1 = ((i + 1) << shift) >> 6;
    for (uint64_t w = w0; w < w1 && w < words; ++w) any |= bits[w];
  }
  const uint32_t b = __ballot_sync(0xffffffffu, any != 0);
  if ((threadIdx.x & 31) == 0 && i < summ_bits) summ32[i >> 5] = b;
}

cudaError_t launch_summary(const uint64_t* bits, uint64_t words, uint32_t shift, uint64_t summ_bits,
                           uint64_t* summ, cudaStream_t s, uint64_t* launches) {
  summary_kernel<<<static_cast<uint32_t>((summ_bits + 255) / 256), 256, 0, s>>>(
      bits, words, shift, summ_bits, reinterpret_cast<uint32_t*>(summ));
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_seed_bitmap(uint64_t* bits, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t blocks = ((n + 63) / 64 + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  all_bits_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(bits, n);
  return cudaGetLastError();
}

// Snapshot restore: dense row i -> counter row perm[i] (or i), W words.
__global__ void scatter_rows_kernel(const uint64_t* __restrict__ src,
                                    const uint32_t* __restrict__ perm, uint64_t count,
                                    uint32_t pitch, uint32_t words,
                                    uint64_t* __restrict__ counters) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       k < count * pitch; k += stride) {
    const uint64_t i = k / pitch, w = k % pitch;
    const uint64_t row = perm ? perm[i] : i;
    counters[row * pitch + w] = w < words ? src[i * words + w] : 0ull;  // padding stays 0
  }
}

cudaError_t launch_scatter_rows(const uint64_t* src, const uint32_t* perm, uint64_t count,
                                uint32_t pitch, uint32_t words, uint64_t* counters, bool bytes,
                                uint32_t registers, cudaStream_t s, uint64_t* launches) {
  if (count == 0) return cudaSuccess;
  if (bytes) {
    uint64_t blocks = (count * 2 * pitch + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    scatter_rows_bytes_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(
        src, perm, count, pitch, words, registers, counters);
    ++*launches;
    return cudaGetLastError();
  }
  uint64_t blocks = (count * pitch + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  scatter_rows_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(src, perm, count, pitch,
                                                                    words, counters);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const uint64_t* counters, const uint32_t* perm, uint64_t first,
                               uint64_t count, uint32_t pitch, uint32_t words, uint64_t* dst,
                               bool bytes, uint32_t registers, cudaStream_t s, uint64_t* launches) {
  if (count == 0) return cudaSuccess;
  uint64_t blocks = (count * words + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (bytes) {
    gather_rows_bytes_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(
        counters, perm, first, count, pitch, words, registers, dst);
    ++*launches;
    return cudaGetLastError();
  }
  gather_rows_kernel<<<static_cast<uint32_t>(blocks), 256, 0, s>>>(counters, perm, first, count,
                                                                   pitch, words, dst);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace hanf
