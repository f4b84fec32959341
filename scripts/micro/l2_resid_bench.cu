// Micro-benchmark (dev aid): can the B200 L2 keep a hot set of 40-byte
// counters resident under a stream of cold random gathers?  Gathers are
// 16-byte windows (3 x LDG.128, as union_kernel), a fraction p from the
// first H records (hot), the rest uniform over 2^28 records (10.7 GB).
// Policies: 0 = default (L1-allocating __ldg), 1 = hot evict_last + cold
// evict_first (createpolicy), with or without the persisting L2 set-aside.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z ^= z >> 33; z *= 0xff51afd7ed558ccdULL; z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ULL; z ^= z >> 33;
  return z;
}

template <int POL>
__global__ void gather(const uint64_t* __restrict__ a, uint64_t m, uint64_t hot, uint64_t n,
                       uint32_t p16, uint64_t seed, uint64_t* out) {
  uint64_t acc = 0;
  uint64_t pl, pf;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix(i ^ seed);
    const bool is_hot = (h & 0xffff) < p16;
    const uint64_t w = is_hot ? (h >> 16) % hot : (h >> 16) % n;
    const uint4* p = reinterpret_cast<const uint4*>(a + ((w * 5) & ~1ull));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      uint4 q;
      if (POL == 0) {
        q = __ldg(p + k);
      } else {
        const uint64_t pol = is_hot ? pl : pf;
        asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(p + k), "l"(pol));
      }
      acc ^= q.x ^ q.w;
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  const uint64_t n = 1ull << 28, m = 1ull << 28;
  uint64_t *a, *out;
  cudaMalloc(&a, sizeof(uint64_t) * (n * 5 + 32));
  cudaMalloc(&out, 8);
  cudaMemset(a, 1, sizeof(uint64_t) * (n * 5 + 32));
  int maxp = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](int pol, uint64_t hot, double p, size_t persist) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
    const uint32_t p16 = (uint32_t)(p * 65536);
    auto k = pol ? gather<1> : gather<0>;
    k<<<148 * 16, 256>>>(a, m, hot, n, p16, 1, out);
    cudaEventRecord(e0);
    k<<<148 * 16, 256>>>(a, m, hot, n, p16, 2, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pol %d hot %6.1f MB p_hot %.2f persist %5.1f MB: %8.3f ms  %6.2f G gathers/s\n", pol,
           hot * 40.0 / 1e6, p, persist / 1e6, ms, m / ms / 1e6);
  };
  for (uint64_t hot : {1ull << 19, 1ull << 20, 1ull << 21, 3ull << 20})
    run(0, hot, 1.0, 0);  // hot set alone: L2 capacity for random 40-B rows
  for (uint64_t hot : {1ull << 20, 1ull << 21}) {
    run(0, hot, 0.66, 0);
    run(1, hot, 0.66, 0);
    run(1, hot, 0.66, (size_t)maxp);
  }
  run(0, 1, 0.0, 0);  // all cold
  printf("max persisting %d\n", maxp);
  return 0;
}
