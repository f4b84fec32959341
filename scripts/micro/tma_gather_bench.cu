// Micro-benchmark (dev aid): random row gathers of 48-byte rows (a 40-byte
// counter padded to 6 words) through three paths, L2-resident and not:
//   ldg    3 x LDG.128 per lane (one lane per row) - the L1 data pipe path
//   g4     TMA tile::gather4 into a per-warp shared-memory ring, rows read
//          back with LDS.128 (bypasses the LSU wavefronts for the gather)
//   bulk   one cp.async.bulk (non-tensor) per row into the same ring
// Each gathered row is folded with XOR so the loads cannot be elided.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_bench tma_gather_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

constexpr int kRowWords = 6;  // 48 bytes
constexpr int kRowBytes = kRowWords * 8;
constexpr int kStage = 2048;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int col, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(256) k_ldg(const uint64_t* __restrict__ a,
                                             const uint32_t* __restrict__ idx, uint64_t m,
                                             uint64_t* out) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4* p = reinterpret_cast<const uint4*>(a + (uint64_t)idx[i] * kRowWords);
    const uint4 x = __ldg(p), y = __ldg(p + 1), z = __ldg(p + 2);
    acc ^= x.x ^ x.y ^ x.z ^ x.w ^ y.x ^ y.y ^ y.z ^ y.w ^ z.x ^ z.y ^ z.z ^ z.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// One warp = one pipeline of S stages x 32 rows; a warp owns contiguous
// 32-id groups [g0, g1).
template <int S, int MODE>
__global__ void __launch_bounds__(256) k_ring(const __grid_constant__ CUtensorMap map,
                                              const uint64_t* __restrict__ a,
                                              const uint32_t* __restrict__ idx, uint64_t groups,
                                              uint64_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // stage = 8 slots of 256 bytes (4 rows of 48 each: gather4 needs a
  // 128-byte aligned destination)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * S;
  uint8_t* ring = smem + 1024 + warp * S * kStage;
  const uint32_t my_row = (lane >> 2) * 256 + (lane & 3) * kRowBytes;
  if (lane < S) mbar_init(bars + lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint64_t g0 = groups * gw / nw, g1 = groups * (gw + 1) / nw;
  auto fill = [&](uint64_t g, int st) {
    const uint32_t id = __ldg(idx + g * 32 + lane);
    uint8_t* buf = ring + st * kStage;
    if (lane == 0) mbar_expect_tx(bars + st, 32 * kRowBytes);
    __syncwarp();
    if constexpr (MODE == 0) {
      const int r0 = __shfl_sync(~0u, id, (lane * 4 + 0) & 31);
      const int r1 = __shfl_sync(~0u, id, (lane * 4 + 1) & 31);
      const int r2 = __shfl_sync(~0u, id, (lane * 4 + 2) & 31);
      const int r3 = __shfl_sync(~0u, id, (lane * 4 + 3) & 31);
      if (lane < 8) tma_gather4(buf + lane * 256, &map, bars + st, 0, r0, r1, r2, r3);
    } else {
      bulk_copy(buf + my_row, a + (uint64_t)id * kRowWords, kRowBytes, bars + st);
    }
  };
  uint32_t acc = 0;
  const uint64_t cnt = g1 - g0;
  for (uint64_t k = 0; k < (cnt < S - 1 ? cnt : S - 1); ++k) fill(g0 + k, (int)k);
  for (uint64_t k = 0; k < cnt; ++k) {
    if (k + S - 1 < cnt) fill(g0 + k + S - 1, (int)((k + S - 1) % S));
    const int st = (int)(k % S);
    mbar_wait(bars + st, (uint32_t)((k / S) & 1));
    const uint4* p = reinterpret_cast<const uint4*>(ring + st * kStage + my_row);
    const uint4 x = p[0], y = p[1], z = p[2];
    acc ^= x.x ^ x.y ^ x.z ^ x.w ^ y.x ^ y.y ^ y.z ^ y.w ^ z.x ^ z.y ^ z.z ^ z.w;
    __syncwarp();
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
  const uint64_t rows_small = 1ull << 20, rows_big = 1ull << 26;
  const uint64_t m = 1ull << 24;  // gathers per launch
  uint64_t* a;
  uint32_t* idx;
  uint64_t* out;
  CK(cudaMalloc(&a, (rows_big + 1) * kRowBytes));
  CK(cudaMemset(a, 1, (rows_big + 1) * kRowBytes));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&out, 64));
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode),
                             cudaEnableDefault, &q));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (uint64_t rows : {rows_small, rows_big}) {
    std::vector<uint32_t> h(m);
    uint64_t s = 88172645463325252ull;
    for (auto& x : h) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      x = static_cast<uint32_t>(s % rows);
    }
    CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
    CUtensorMap map;
    cuuint64_t gdim[2] = {kRowWords, rows + 1};
    cuuint64_t gstride[1] = {kRowBytes};
    cuuint32_t box[2] = {kRowWords, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, a, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { std::printf("encode failed %d\n", (int)r); return 1; }
    auto run = [&](const char* name, auto launch) {
      for (int it = 0; it < 3; ++it) launch();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      const int reps = 10;
      for (int it = 0; it < reps; ++it) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= reps;
      std::printf("rows=2^%d %-22s %8.3f ms  %6.2f G rows/s\n", rows == rows_small ? 20 : 26, name,
                  ms, m / ms / 1e6);
    };
    for (int ctas : {4, 8}) {
      char nm[64];
      std::snprintf(nm, sizeof nm, "ldg x%d", ctas);
      run(nm, [&] { k_ldg<<<sms * ctas, 256>>>(a, idx, m, out); });
    }
    const uint64_t groups = m / 32;
#define RING(S, MODE, CTAS)                                                                   \
  {                                                                                           \
    const int sm = 1024 + 8 * S * kStage;                                          \
    CK(cudaFuncSetAttribute(k_ring<S, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    char nm[64];                                                                              \
    std::snprintf(nm, sizeof nm, "%s S=%d x%d", MODE == 0 ? "g4" : "bulk", S, CTAS);          \
    run(nm, [&] { k_ring<S, MODE><<<sms * CTAS, 256, sm>>>(map, a, idx, groups, out); });    \
  }
    RING(2, 0, 2) RING(4, 0, 2) RING(4, 0, 3) RING(3, 0, 4) RING(6, 0, 2)
    RING(2, 1, 2) RING(4, 1, 2) RING(3, 1, 4)
  }
  return 0;
}
