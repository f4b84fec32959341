// Micro-benchmark (dev aid): DRAM traffic and time of random gathers of
// W-word records from an array much larger than L2, by load shape.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ldg256(uint32_t (&v)[8], const void* p) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7]) : "l"(p));
}

template <int W, int MODE>
__global__ void gather(const uint64_t* __restrict__ a, const uint32_t* __restrict__ idx, uint64_t m,
                       uint64_t* out) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w = idx[i];
    const uint64_t word = w * W;
    if constexpr (MODE == 0) {  // W x 8-byte loads
#pragma unroll
      for (int k = 0; k < W; ++k) acc ^= __ldg(a + word + k);
    } else if constexpr (MODE == 1) {  // 16-byte window (W odd)
      const uint4* p = reinterpret_cast<const uint4*>(a + (word & ~1ull));
#pragma unroll
      for (int k = 0; k < (W + 2) / 2; ++k) { uint4 q = __ldg(p + k); acc ^= q.x ^ q.y ^ q.z ^ q.w; }
    } else if constexpr (MODE == 2) {  // 32-byte aligned window, only needed pieces
      const uint64_t first = word & ~3ull, last = (word + W - 1) & ~3ull;
      for (uint64_t b = first; b <= last; b += 4) {
        uint32_t v[8];
        ldg256(v, a + b);
        acc ^= v[0] ^ v[7];
      }
    } else {  // 64-byte block(s) containing the record, 2 x 32 bytes each
      const uint64_t first = word & ~7ull, last = (word + W - 1) & ~7ull;
      for (uint64_t b = first; b <= last; b += 8) {
        uint32_t v[8], u[8];
        ldg256(v, a + b);
        ldg256(u, a + b + 4);
        acc ^= v[0] ^ u[7];
      }
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  const uint64_t n = 1ull << 25;  // records
  const uint64_t m = 1ull << 28;  // gathers
  uint64_t *a, *out;
  uint32_t* idx;
  cudaMalloc(&a, sizeof(uint64_t) * (n * 10 + 32));
  cudaMalloc(&idx, sizeof(uint32_t) * m);
  cudaMalloc(&out, 8);
  cudaMemset(a, 1, sizeof(uint64_t) * (n * 10 + 32));
  // random indices: hash on device via a simple kernel
  uint32_t* h = (uint32_t*)malloc(sizeof(uint32_t) * m);
  uint64_t x = 88172645463325252ull;
  for (uint64_t i = 0; i < m; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)(x % n); }
  cudaMemcpy(idx, h, sizeof(uint32_t) * m, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(const uint64_t*, const uint32_t*, uint64_t, uint64_t*), int W) {
    k<<<148 * 16, 256>>>(a, idx, m, out);
    cudaEventRecord(e0);
    k<<<148 * 16, 256>>>(a, idx, m, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s W=%2d  %8.3f ms  %6.2f G gathers/s  %7.1f GB/s useful\n", name, W, ms, m / ms / 1e6,
           m * 8.0 * W / ms / 1e6);
  };
  run("3 x LDG.64", gather<3, 0>, 3);
  run("16B window", gather<3, 1>, 3);
  run("32B pieces", gather<3, 2>, 3);
  run("64B blocks", gather<3, 3>, 3);
  run("5 x LDG.64", gather<5, 0>, 5);
  run("16B window", gather<5, 1>, 5);
  run("32B pieces", gather<5, 2>, 5);
  run("64B blocks", gather<5, 3>, 5);
  run("10 x LDG.64", gather<10, 0>, 10);
  run("32B pieces", gather<10, 2>, 10);
  run("64B blocks", gather<10, 3>, 10);
  return 0;
}
