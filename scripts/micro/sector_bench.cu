// Dev aid: random gathers of 32-byte rows (config 4's padded m = 32 rows)
// out of a 1 GiB array under the cache policies a 256-bit load can carry.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sector_bench scripts/micro/sector_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

template <int POL>
__device__ __forceinline__ void ld256(uint32_t (&v)[8], const uint64_t* q) {
  if constexpr (POL == 0)
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(q));
  else if constexpr (POL == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(q));
  else if constexpr (POL == 2)
    asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(q));
  else
    asm volatile("ld.global.L1::no_allocate.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]) : "l"(q));
}

template <int POL>
__global__ void __launch_bounds__(256) gather(const uint64_t* __restrict__ rows, uint32_t mask,
                                              uint64_t per_thread, uint32_t* __restrict__ out) {
  uint64_t x = (blockIdx.x * 256ull + threadIdx.x) * 0x9e3779b97f4a7c15ull + 12345;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < per_thread; i += 4) {
    uint32_t v[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      ld256<POL>(v[j], rows + 4ull * (static_cast<uint32_t>(x >> 20) & mask));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= v[j][k];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int POL>
void run(const uint64_t* rows, uint32_t mask, uint32_t* out, const char* name) {
  const uint64_t total = 1ull << 28, threads = 148ull * 16 * 256, per = total / threads / 4 * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  gather<POL><<<148 * 16, 256>>>(rows, mask, per, out);
  cudaEventRecord(a);
  gather<POL><<<148 * 16, 256>>>(rows, mask, per, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-44s %8.3f ms  %6.1f G gathers/s\n", name, ms, per * threads / ms / 1e6);
}

int main() {
  const uint32_t rows_n = 1u << 25;  // 1 GiB of 32-byte rows
  uint64_t* rows; uint32_t* out;
  cudaMalloc(&rows, 32ull * rows_n); cudaMalloc(&out, 4);
  cudaMemset(rows, 1, 32ull * rows_n);
  run<0>(rows, rows_n - 1, out, "ld.global.nc.v8 (default)");
  run<1>(rows, rows_n - 1, out, "ld.global.nc.L1::no_allocate.v8");
  run<2>(rows, rows_n - 1, out, "ld.global.cg.v8");
  run<3>(rows, rows_n - 1, out, "ld.global.L1::no_allocate.L2::64B.v8");
  return 0;
}
