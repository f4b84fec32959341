// hanf_rng.h -- the counter-based streams of the synthetic generators,
// shared by the host builders (hanf_host.cpp) and the device builders
// (hanf_graphgen.cu) so both produce the same graphs bit for bit.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define HANF_HD __host__ __device__ __forceinline__
#else
#define HANF_HD inline
#endif

namespace hanf_rng {

// hash.hpp:8-15 (the reference's finaliser)
HANF_HD constexpr uint64_t mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}

// Counter-based stream: value k of stream (seed, key).  Every arc of the
// synthetic configs is a pure function of its index, so generation is
// parallel and identical on any thread count or device.
HANF_HD uint64_t hash3(uint64_t seed, uint64_t key, uint64_t k) {
  return mix64(mix64(seed ^ 0x5851f42d4c957f2dULL) ^ mix64(key * 0x9e3779b97f4a7c15ULL + k));
}
HANF_HD double u01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

// Random bijection on [0, 2^bits) (4-round unbalanced Feistel network keyed
// by seed), bits >= 2.  Used to permute node ids.
struct Feistel {
  uint32_t lbits, rbits;
  uint64_t keys[4];
  HANF_HD Feistel(uint32_t b, uint64_t seed) : lbits(b / 2), rbits(b - b / 2), keys{} {
    for (int i = 0; i < 4; ++i) keys[i] = mix64(seed * 4 + i + 0x7f4a7c15ULL);
  }
  HANF_HD uint64_t operator()(uint64_t x) const {
    uint64_t l = x >> rbits, r = x & ((1ull << rbits) - 1);
    uint32_t lb = lbits, rb = rbits;
    for (int i = 0; i < 4; ++i) {
      const uint64_t f = mix64(r ^ keys[i]) & ((1ull << lb) - 1);
      const uint64_t nl = r, nr = l ^ f;
      l = nl;  // the new left half has rb bits, the new right half lb bits
      r = nr;
      const uint32_t t = lb;
      lb = rb;
      rb = t;
    }
    return (l << rb) | r;
  }
};

// R-MAT draw i (configs 2 and 5): `scale` levels, 16 bits of the stream
// (seed, i) per level; thresholds ta < tb < tc are a, a+b, a+b+c in 1/65536.
HANF_HD void rmat_draw(uint64_t seed, uint64_t i, uint32_t scale, uint32_t ta, uint32_t tb,
                       uint32_t tc, uint64_t* u_out, uint64_t* v_out) {
  uint64_t u = 0, v = 0, h = 0;
  for (uint32_t level = 0; level < scale; ++level) {
    if ((level & 3) == 0) h = hash3(seed, i, level >> 2);
    const uint32_t r = static_cast<uint32_t>(h >> (16 * (level & 3))) & 0xffff;
    const uint64_t bu = r >= tb, bv = (r >= ta && r < tb) || r >= tc;
    u = (u << 1) | bu;
    v = (v << 1) | bv;
  }
  *u_out = u;
  *v_out = v;
}

}  // namespace hanf_rng
