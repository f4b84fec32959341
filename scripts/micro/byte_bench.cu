// Micro-benchmark (dev aid): gather + register-wise max of 64-register
// HLL counters, reference packing (40-byte rows, one lane per counter,
// 3 x LDG.128 + PackedMax on 10 limbs) against a byte-per-register layout
// (64-byte rows: a quad of lanes per counter, one LDG.128 each, and the
// guard-bit byte max: IADD3 + PRMT sign-replicate + LOP3 per 4 registers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I../../paper_1011_5599_b200/csrc -o byte_bench byte_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "hanf_device.cuh"

using namespace hanf;

constexpr int W = 5;

template <int U>
__global__ void __launch_bounds__(256, 5) k_packed(const uint64_t* __restrict__ cnt,
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

__device__ __forceinline__ uint32_t bmax(uint32_t x, uint32_t y) {
  const uint32_t d = x + 0x80808080u - y;   // bit 7 of each byte: x >= y
  const uint32_t m = __byte_perm(d, 0, 0xba98);  // sign-replicate each byte
  return lop3<0xE4>(x, y, m);               // m ? x : y
}

// quad q = lanes 4q..4q+3 folds one successor per trip; lane k holds
// registers [16k, 16k + 16) as bytes
template <int U>
__global__ void __launch_bounds__(256, 5) k_quad(const uint4* __restrict__ cnt,
                                                 const uint32_t* __restrict__ ids, uint32_t per_quad,
                                                 uint32_t* out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nq = gridDim.x * blockDim.x / 4;
  const uint32_t q = t >> 2, k = t & 3;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint32_t i = 0; i < per_quad; i += U) {
    uint32_t w[U];
#pragma unroll
    for (int j = 0; j < U; ++j) w[j] = __ldg(ids + (uint64_t)(i + j) * nq + q);
    uint4 y[U];
#pragma unroll
    for (int j = 0; j < U; ++j) y[j] = __ldg(cnt + (uint64_t)w[j] * 4 + k);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      acc.x = bmax(acc.x, y[j].x);
      acc.y = bmax(acc.y, y[j].y);
      acc.z = bmax(acc.z, y[j].z);
      acc.w = bmax(acc.w, y[j].w);
    }
  }
  const uint32_t x = acc.x ^ acc.y ^ acc.z ^ acc.w;
  if (x == 0x9e3779b9u) out[0] = x;
}

// one lane per counter, byte rows: 4 x LDG.128, 16 limbs
template <int U>
__global__ void __launch_bounds__(256, 4) k_lane_bytes(const uint4* __restrict__ cnt,
                                                       const uint32_t* __restrict__ ids,
                                                       uint32_t per_lane, uint32_t* out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  uint32_t acc[16] = {};
  for (uint32_t i = 0; i < per_lane; i += U) {
    uint32_t w[U];
#pragma unroll
    for (int j = 0; j < U; ++j) w[j] = __ldg(ids + (uint64_t)(i + j) * nt + t);
    uint4 y[U][4];
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) y[j][c] = __ldg(cnt + (uint64_t)w[j] * 4 + c);
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[4 * c + 0] = bmax(acc[4 * c + 0], y[j][c].x);
        acc[4 * c + 1] = bmax(acc[4 * c + 1], y[j][c].y);
        acc[4 * c + 2] = bmax(acc[4 * c + 2], y[j][c].z);
        acc[4 * c + 3] = bmax(acc[4 * c + 3], y[j][c].w);
      }
  }
  uint32_t x = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) x ^= acc[c];
  if (x == 0x9e3779b9u) out[0] = x;
}

int main() {
  const uint32_t ctas = 148 * 5, threads = 256, nt = ctas * threads;
  const uint32_t per_lane = 96;  // gathers per lane (packed / lane-bytes)
  const uint64_t total = (uint64_t)per_lane * nt;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  uint32_t* dout; cudaMalloc(&dout, 64);
  uint32_t* di; cudaMalloc(&di, total * 4);
  std::vector<uint32_t> ids(total);
  const uint64_t sizes[3] = {1ull << 20, 1ull << 22, 1ull << 26};
  for (int mix = 0; mix < 2; ++mix)
  for (uint64_t n : sizes) {
    uint64_t s = 0x1234567 + n;
    for (auto& x : ids) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      // mix 1: 2/3 of the gathers from the first 2^21 rows (config 5's hot share)
      const uint64_t lim = (mix == 1 && (s >> 40) % 3 != 0) ? (n < (1u << 21) ? n : (1u << 21)) : n;
      x = (uint32_t)((s >> 7) % lim);
    }
    cudaMemcpy(di, ids.data(), total * 4, cudaMemcpyHostToDevice);
    uint64_t *packed; uint4* bytes;
    cudaMalloc(&packed, (n * W + 8) * 8);
    cudaMalloc(&bytes, n * 64);
    cudaMemset(packed, 0x11, (n * W + 8) * 8);
    cudaMemset(bytes, 0x11, n * 64);
    auto run = [&](const char* name, auto launch) {
      for (int i = 0; i < 2; ++i) launch();
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) launch();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
      std::printf("rows 2^%-2d %-6s %-22s %8.3f ms  %6.1f G gathers/s  (%s)\n", __builtin_ctzll(n),
                  mix ? "hot2/3" : "unif", name, ms, total / ms / 1e6,
                  cudaGetErrorString(cudaGetLastError()));
    };
    run("packed lane U=3", [&] { k_packed<3><<<ctas, threads>>>(packed, di, per_lane, dout); });
    run("packed lane U=2", [&] { k_packed<2><<<ctas, threads>>>(packed, di, per_lane, dout); });
    run("bytes lane U=2", [&] { k_lane_bytes<2><<<ctas, threads>>>(bytes, di, per_lane, dout); });
    // quads: nt/4 quads, 4x the gathers each for the same total
    run("bytes quad U=4", [&] { k_quad<4><<<ctas, threads>>>(bytes, di, per_lane * 4, dout); });
    run("bytes quad U=8", [&] { k_quad<8><<<ctas, threads>>>(bytes, di, per_lane * 4, dout); });
    run("bytes quad U=2", [&] { k_quad<2><<<ctas, threads>>>(bytes, di, per_lane * 4, dout); });
    cudaFree(packed); cudaFree(bytes);
  }
  return 0;
}
