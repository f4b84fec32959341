// Micro-benchmark (dev aid): is splitting each 40-byte counter over a lane
// pair (each lane: 2 x LDG.128 + the SWAR max on its 5 limbs) faster than
// one lane per counter (3 x LDG.128 + 10 limbs), L2-resident, same ALU work
// per counter?  Uses the engine's own swar_max/Layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I../../paper_1011_5599_b200/csrc -o pair_bench pair_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "hanf_device.cuh"

using namespace hanf;

constexpr int W = 5;  // words per counter (m = 64, r = 5)

template <int U>
__global__ void __launch_bounds__(256, 4) k_full(const uint64_t* __restrict__ cnt,
                                                 const uint32_t* __restrict__ ids, uint32_t per_lane,
                                                 uint32_t* out) {
  using Lay = Layout<5, 64>;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  uint32_t acc[Lay::kLimbs] = {};
  for (uint32_t i = 0; i < per_lane; i += U) {
    uint32_t w[U];
#pragma unroll
    for (int j = 0; j < U; ++j) w[j] = __ldg(ids + (uint64_t)(i + j) * nt + t);
    uint4 raw[U][3];
#pragma unroll
    for (int j = 0; j < U; ++j) window128_load<W, 0>(raw[j], cnt, w[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint32_t y[Lay::kLimbs];
      window128_extract<Lay, W>(y, raw[j], w[j]);
      swar_max<Lay>(acc, y);
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < Lay::kLimbs; ++k) x ^= acc[k];
  if (x == 0x9e3779b9u) out[0] = x;
}

// lane pair (2p, 2p+1) folds the same successor: lane h holds limbs
// [5h, 5h+5) (registers 32h..32h+31, a register boundary at bit 160)
template <int U>
__global__ void __launch_bounds__(256, 4) k_pair(const uint64_t* __restrict__ cnt,
                                                 const uint32_t* __restrict__ ids, uint32_t per_pair,
                                                 uint32_t* out) {
  using Half = Layout<5, 32>;  // 5 limbs, same mask pattern for both halves
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t np = gridDim.x * blockDim.x / 2;
  const uint32_t p = t >> 1, h = t & 1;
  uint32_t acc[Half::kLimbs] = {};
  for (uint32_t i = 0; i < per_pair; i += U) {
    uint32_t w[U];
#pragma unroll
    for (int j = 0; j < U; ++j) w[j] = __ldg(ids + (uint64_t)(i + j) * np + p);
    uint4 raw[U][2];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint64_t word = (uint64_t)w[j] * W;
      const uint4* q = reinterpret_cast<const uint4*>(cnt + (word & ~1ull)) + h;
      raw[j][0] = __ldg(q);
      raw[j][1] = __ldg(q + 1);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t off = h + 2 * ((w[j] * W) & 1u);  // first limb within the 8 loaded
      auto at = [&](int i2) -> uint32_t {
        const uint4& q = raw[j][i2 / 4];
        switch (i2 % 4) {
          case 0: return q.x;
          case 1: return q.y;
          case 2: return q.z;
          default: return q.w;
        }
      };
      uint32_t y[Half::kLimbs];
#pragma unroll
      for (int k = 0; k < Half::kLimbs; ++k) {
        const uint32_t a0 = (off & 1) ? at(k + 1) : at(k);
        const uint32_t a2 = (off & 1) ? at(k + 3) : at(k + 2);
        y[k] = (off & 2) ? a2 : a0;
      }
      swar_max<Half>(acc, y);
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < Half::kLimbs; ++k) x ^= acc[k];
  if (x == 0x9e3779b9u) out[0] = x;
}

int main() {
  const uint64_t n = 1 << 20;
  const uint32_t ctas = 148 * 4, threads = 256, nt = ctas * threads;
  const uint32_t per_lane = 120;  // ~18 M counters per launch (full)
  std::vector<uint64_t> h(n * W + 8);
  uint64_t s = 0x1234567;
  for (auto& x : h) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = s; }
  std::vector<uint32_t> ids((uint64_t)per_lane * nt);
  for (auto& x : ids) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = (uint32_t)(s % n); }
  uint64_t* dc; uint32_t *di, *dout;
  cudaMalloc(&dc, h.size() * 8); cudaMalloc(&di, ids.size() * 4); cudaMalloc(&dout, 64);
  cudaMemcpy(dc, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(di, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, uint64_t counters, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    std::printf("%-24s %8.3f ms  %6.1f G counters/s  (%s)\n", name, ms, counters / ms / 1e6,
                cudaGetErrorString(cudaGetLastError()));
  };
  const uint64_t cf = (uint64_t)per_lane * nt;
  run("full U=3", cf, [&] { k_full<3><<<ctas, threads>>>(dc, di, per_lane, dout); });
  run("full U=2", cf, [&] { k_full<2><<<ctas, threads>>>(dc, di, per_lane, dout); });
  // pairs: same number of counters = per_lane * nt ids over nt/2 pairs
  const uint32_t per_pair = 2 * per_lane;
  run("pair U=3", cf, [&] { k_pair<3><<<ctas, threads>>>(dc, di, per_pair - per_pair % 3, dout); });
  run("pair U=4", cf, [&] { k_pair<4><<<ctas, threads>>>(dc, di, per_pair, dout); });
  run("pair U=2", cf, [&] { k_pair<2><<<ctas, threads>>>(dc, di, per_pair, dout); });
  return 0;
}
