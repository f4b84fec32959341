// hanf_device.cuh -- register layout, broadword max and estimator for sm_100a.
//
// Counters keep the reference packing bit for bit (hll.hpp:19-22, 183-240;
// FORMATS.md:25-41): counter i = u64 words [i*W, (i+1)*W), register j =
// bits [j*r, (j+1)*r) from the LSB of word 0, straddling words, padding 0.
//
// On the GPU the words are handled as 32-bit limbs (the native ALU width).
// A counter is processed in "chunks": a chunk is a whole lcm(64, r)-bit
// period of the packing (or the whole counter when it is shorter), so the
// per-limb high/low register masks are compile-time immediates and chunks
// are independent of each other.
#pragma once

#include <cstdint>
#include <cstdio>
#include <type_traits>

// Checked builds (make checked -> libhanf_checked.so, HANF_LIB=checked):
// every row, bitmap word and task index a kernel derives from device data
// is bounds-checked and a violation traps with its source line.  The
// default build compiles the checks out.
#ifdef HANF_CHECKED
#define HANF_DCHECK(c)                                                            \
  do {                                                                            \
    if (!(c)) {                                                                   \
      printf("hanf check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);          \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define HANF_DCHECK(c) \
  do {                 \
  } while (0)
#endif

namespace hanf {

template <int I>
using ic = std::integral_constant<int, I>;

// Compile-time loop: f(ic<B>{}), ..., f(ic<E-1>{}).
template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(ic<B>{});
    sfor<B + 1, E>(f);
  }
}

// d = LUT(a, b, c) with the PTX lop3 truth-table convention (a=0xF0,
// b=0xCC, c=0xAA).
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

// Register layout of one chunk: NREG registers of R bits.
template <int R, int NREG>
struct Layout {
  static constexpr bool kBytes = false;
  static constexpr int kR = R;
  static constexpr int kNReg = NREG;
  static constexpr int kBits = NREG * R;
  static constexpr int kLimbs = (kBits + 31) / 32;  // limbs holding register bits
  static constexpr int kWords = (kBits + 63) / 64;  // storage words of the chunk
  static constexpr uint32_t kMul = (1u << R) - 1;   // lane spread multiplier

  // High bit of every register that falls in limb i (PackedMax's H,
  // broadword.hpp:81-86, restated per 32-bit limb).
  __host__ __device__ static constexpr uint32_t high(int i) {
    uint32_t m = 0;
    for (int j = 0; j < NREG; ++j) {
      const int hb = j * R + R - 1;
      if (hb >= 32 * i && hb < 32 * i + 32) m |= 1u << (hb - 32 * i);
    }
    return m;
  }
  // Does a register straddle the boundary between limb i-1 and limb i?
  // Only there can a borrow cross limbs: every other register has its
  // minuend high bit forced (broadword.hpp:23-25).
  __host__ __device__ static constexpr bool straddle(int i) {
    return i > 0 && i < kLimbs && (32 * i) % R != 0;
  }
  // End (exclusive) of the borrow chain starting at limb s.
  __host__ __device__ static constexpr int chain_end(int s) {
    int e = s + 1;
    while (e < kLimbs && straddle(e)) ++e;
    return e;
  }
};

// Byte layout (the engine's default counter store for r = 5): register j of
// a counter is byte j of its row, value in the low 5 bits.  A row of M
// registers is M bytes, 16-byte aligned (M >= 16), so a quad of lanes reads
// a 64-register counter as one coalesced 64-byte access and the register-
// wise max is three instructions per four registers (byte_max).  Every
// exchange with the caller (read-back, snapshots, restore) converts to or
// from the reference packing (hll.hpp:183-240), so the bits a caller sees
// are the reference's.
template <int M>
struct ByteLayout {
  static constexpr bool kBytes = true;
  static constexpr int kR = 5;
  static constexpr int kNReg = M;
  static constexpr int kLimbs = M / 4;  // four registers per 32-bit limb
  static constexpr int kWords = M / 8;
};

// Byte-wise max of four registers (each < 128): bit 7 of byte k of
// x + 0x80 - y is set iff x_k >= y_k (no borrow leaves a byte), PRMT's
// sign-replicate selector turns it into a whole-byte mask, one LOP3
// selects.  This is PackedMax::max_into (broadword.hpp:94-130) on
// byte-aligned lanes, where no register straddles a limb.
__device__ __forceinline__ uint32_t byte_max(uint32_t x, uint32_t y) {
  const uint32_t d = x + 0x80808080u - y;
  uint32_t m;  // 0xff where x_k >= y_k (PRMT selector nibble 8 + k: byte k, sign-replicated)
  asm("prmt.b32 %0, %1, 0, 0xba98;" : "=r"(m) : "r"(d));
  return lop3<0xE4>(x, y, m);  // m ? x : y
}

__device__ __forceinline__ uint4 byte_max4(const uint4& x, const uint4& y) {
  return make_uint4(byte_max(x.x, y.x), byte_max(x.y, y.y), byte_max(x.z, y.z),
                    byte_max(x.w, y.w));
}

// sum of 2^(31 - M_j) over the 16 byte registers of v (M_j <= 31) and the
// number of zero registers: the r = 5 estimator's exact integer terms
__device__ __forceinline__ void byte_terms(const uint4& v, uint64_t& s, uint32_t& zeros) {
  const uint32_t l[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t term = 0x80000000u >> ((l[i] >> (8 * b)) & 31u);
      s += term;
      zeros += term >> 31;
    }
}

// d[S..S+N) = a[S..S+N) - b[S..S+N) as one multi-precision number (borrow
// chain in the carry flag).  One asm statement per chain so nothing can
// clobber the flag between links.
template <int S, int N, int L>
__device__ __forceinline__ void sub_chain(uint32_t (&d)[L], const uint32_t (&a)[L],
                                          const uint32_t (&b)[L]) {
  static_assert(N >= 1 && N <= 7, "chain length");
  if constexpr (N == 1) {
    d[S] = a[S] - b[S];
  } else if constexpr (N == 2) {
    asm("sub.cc.u32 %0, %2, %4;\n\tsubc.u32 %1, %3, %5;"
        : "=r"(d[S]), "=r"(d[S + 1])
        : "r"(a[S]), "r"(a[S + 1]), "r"(b[S]), "r"(b[S + 1]));
  } else if constexpr (N == 3) {
    asm("sub.cc.u32 %0, %3, %6;\n\tsubc.cc.u32 %1, %4, %7;\n\tsubc.u32 %2, %5, %8;"
        : "=r"(d[S]), "=r"(d[S + 1]), "=r"(d[S + 2])
        : "r"(a[S]), "r"(a[S + 1]), "r"(a[S + 2]), "r"(b[S]), "r"(b[S + 1]),
          "r"(b[S + 2]));
  } else if constexpr (N == 4) {
    asm("sub.cc.u32 %0, %4, %8;\n\tsubc.cc.u32 %1, %5, %9;\n\t"
        "subc.cc.u32 %2, %6, %10;\n\tsubc.u32 %3, %7, %11;"
        : "=r"(d[S]), "=r"(d[S + 1]), "=r"(d[S + 2]), "=r"(d[S + 3])
        : "r"(a[S]), "r"(a[S + 1]), "r"(a[S + 2]), "r"(a[S + 3]), "r"(b[S]),
          "r"(b[S + 1]), "r"(b[S + 2]), "r"(b[S + 3]));
  } else if constexpr (N == 5) {
    asm("sub.cc.u32 %0, %5, %10;\n\tsubc.cc.u32 %1, %6, %11;\n\t"
        "subc.cc.u32 %2, %7, %12;\n\tsubc.cc.u32 %3, %8, %13;\n\t"
        "subc.u32 %4, %9, %14;"
        : "=r"(d[S]), "=r"(d[S + 1]), "=r"(d[S + 2]), "=r"(d[S + 3]), "=r"(d[S + 4])
        : "r"(a[S]), "r"(a[S + 1]), "r"(a[S + 2]), "r"(a[S + 3]), "r"(a[S + 4]),
          "r"(b[S]), "r"(b[S + 1]), "r"(b[S + 2]), "r"(b[S + 3]), "r"(b[S + 4]));
  } else if constexpr (N == 6) {
    asm("sub.cc.u32 %0, %6, %12;\n\tsubc.cc.u32 %1, %7, %13;\n\t"
        "subc.cc.u32 %2, %8, %14;\n\tsubc.cc.u32 %3, %9, %15;\n\t"
        "subc.cc.u32 %4, %10, %16;\n\tsubc.u32 %5, %11, %17;"
        : "=r"(d[S]), "=r"(d[S + 1]), "=r"(d[S + 2]), "=r"(d[S + 3]), "=r"(d[S + 4]),
          "=r"(d[S + 5])
        : "r"(a[S]), "r"(a[S + 1]), "r"(a[S + 2]), "r"(a[S + 3]), "r"(a[S + 4]),
          "r"(a[S + 5]), "r"(b[S]), "r"(b[S + 1]), "r"(b[S + 2]), "r"(b[S + 3]),
          "r"(b[S + 4]), "r"(b[S + 5]));
  } else {
    asm("sub.cc.u32 %0, %7, %14;\n\tsubc.cc.u32 %1, %8, %15;\n\t"
        "subc.cc.u32 %2, %9, %16;\n\tsubc.cc.u32 %3, %10, %17;\n\t"
        "subc.cc.u32 %4, %11, %18;\n\tsubc.cc.u32 %5, %12, %19;\n\t"
        "subc.u32 %6, %13, %20;"
        : "=r"(d[S]), "=r"(d[S + 1]), "=r"(d[S + 2]), "=r"(d[S + 3]), "=r"(d[S + 4]),
          "=r"(d[S + 5]), "=r"(d[S + 6])
        : "r"(a[S]), "r"(a[S + 1]), "r"(a[S + 2]), "r"(a[S + 3]), "r"(a[S + 4]),
          "r"(a[S + 5]), "r"(a[S + 6]), "r"(b[S]), "r"(b[S + 1]), "r"(b[S + 2]),
          "r"(b[S + 3]), "r"(b[S + 4]), "r"(b[S + 5]), "r"(b[S + 6]));
  }
}

template <class Lay, int S, int L>
__device__ __forceinline__ void sub_chains(uint32_t (&d)[L], const uint32_t (&a)[L],
                                           const uint32_t (&b)[L]) {
  if constexpr (S < Lay::kLimbs) {
    constexpr int E = Lay::chain_end(S);
    sub_chain<S, E - S>(d, a, b);
    sub_chains<Lay, E>(d, a, b);
  }
}

// x <- register-wise max(x, y) over one chunk (the semantics of
// PackedMax::max_into, broadword.hpp:94-130).
//
// Pass 1 is the reference's comparison: lt = high bit of every lane where
// x < y, from d = (x|H) - (y&~H) with the borrow rippling only through
// straddling registers.  Pass 2 spreads each lt bit over its r-bit lane
// with one 32x32->64 multiply by (2^r - 1) of the lane's low bit (the high
// half carries straddling lanes into the next limb), replacing the
// reference's second borrow chain; the select is one LOP3.
//
// The chunk is processed one borrow chain at a time (limbs [S, E) joined by
// straddling registers).  At a chain end the next limb starts with a whole
// register, so no lt bit needs to cross (funnel input 0) and the spread
// carry is 0: chains are independent, which keeps the live temporaries to
// one chain's worth.
template <class Lay, int S>
__device__ __forceinline__ void swar_chain(uint32_t (&x)[Lay::kLimbs],
                                           const uint32_t (&y)[Lay::kLimbs]) {
  constexpr int NL = Lay::kLimbs;
  constexpr int R = Lay::kR;
  if constexpr (S < NL) {
    constexpr int E = Lay::chain_end(S);
    uint32_t a[NL], b[NL], d[NL], lt[NL];
    sfor<S, E>([&](auto I) {
      constexpr int i = decltype(I)::value;
      constexpr uint32_t H = Lay::high(i);
      a[i] = x[i] | H;
      b[i] = y[i] & ~H;
    });
    sub_chain<S, E - S>(d, a, b);
    sfor<S, E>([&](auto I) {
      constexpr int i = decltype(I)::value;
      constexpr uint32_t H = Lay::high(i);
      lt[i] = lop3<0x2B>(d[i], x[i], y[i]) & H;  // ((d | (x^y)) ^ (x | ~y)) & H
    });
    // spread_i = low(u_i * (2^r - 1)) | high(u_{i-1} * (2^r - 1)).  The two
    // never overlap, so the low word is one 32-bit multiply-add with the
    // carry as addend (it cannot overflow) and the next carry is the high
    // word alone: IMAD + IMAD.HI on the FMA pipe, no OR and no register
    // pair (an IMAD.WIDE with a 64-bit addend costs two moves per limb)
    uint32_t carry = 0;
    sfor<S, E>([&](auto I) {
      constexpr int i = decltype(I)::value;
      uint32_t u;
      if constexpr (i + 1 < E)
        u = __funnelshift_r(lt[i], lt[i + 1], R - 1);
      else
        u = lt[i] >> (R - 1);
      const uint32_t spread = u * Lay::kMul + carry;
      if constexpr (i + 1 < E) carry = __umulhi(u, Lay::kMul);
      x[i] = lop3<0xD8>(x[i], y[i], spread);  // (x & ~spread) | (y & spread)
    });
    swar_chain<Lay, E>(x, y);
  }
}

template <class Lay>
__device__ __forceinline__ void swar_max(uint32_t (&x)[Lay::kLimbs],
                                         const uint32_t (&y)[Lay::kLimbs]) {
  if constexpr (Lay::kBytes) {
    sfor<0, Lay::kLimbs>([&](auto I) {
      constexpr int i = decltype(I)::value;
      x[i] = byte_max(x[i], y[i]);
    });
  } else {
    swar_chain<Lay, 0>(x, y);
  }
}

// Counter loads with a cache policy: 0 = read-only path (L1 allocating, a
// miss fills the whole 128-byte line), 1 = ld.cg (L2 only, sector
// granular), 2 = ld.nc with L1::no_allocate.
template <int kPol>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  if constexpr (kPol == 0) {
    v = __ldg(p);
  } else if constexpr (kPol == 1) {
    asm("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  }
  return v;
}
template <int kPol>
__device__ __forceinline__ uint2 ld8(const uint2* p) {
  uint2 v;
  if constexpr (kPol == 0) {
    v = __ldg(p);
  } else if constexpr (kPol == 1) {
    asm("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  }
  return v;
}

// Loads one chunk (Lay::kWords u64 words at p) into limbs; padding limbs
// beyond kLimbs are dropped (they are zero by the layout contract).
template <class Lay, bool kVec16, int kPol = 0>
__device__ __forceinline__ void load_chunk(uint32_t (&v)[Lay::kLimbs], const uint64_t* p) {
  constexpr int NW = Lay::kWords;
  constexpr int NL = Lay::kLimbs;
  if constexpr (kVec16 && NW % 2 == 0) {
    sfor<0, NW / 2>([&](auto I) {
      constexpr int k = decltype(I)::value;
      const uint4 q = ld16<kPol>(reinterpret_cast<const uint4*>(p) + k);
      if constexpr (4 * k + 0 < NL) v[4 * k + 0] = q.x;
      if constexpr (4 * k + 1 < NL) v[4 * k + 1] = q.y;
      if constexpr (4 * k + 2 < NL) v[4 * k + 2] = q.z;
      if constexpr (4 * k + 3 < NL) v[4 * k + 3] = q.w;
    });
  } else {
    sfor<0, NW>([&](auto I) {
      constexpr int k = decltype(I)::value;
      const uint2 q = ld8<kPol>(reinterpret_cast<const uint2*>(p) + k);
      if constexpr (2 * k + 0 < NL) v[2 * k + 0] = q.x;
      if constexpr (2 * k + 1 < NL) v[2 * k + 1] = q.y;
    });
  }
}

// Same, through the coherent path (data written earlier in this kernel).
template <class Lay>
__device__ __forceinline__ void load_chunk_coherent(uint32_t (&v)[Lay::kLimbs],
                                                    const uint64_t* p) {
  constexpr int NW = Lay::kWords;
  constexpr int NL = Lay::kLimbs;
  sfor<0, NW>([&](auto I) {
    constexpr int k = decltype(I)::value;
    const uint64_t q = __ldcg(p + k);
    if constexpr (2 * k + 0 < NL) v[2 * k + 0] = static_cast<uint32_t>(q);
    if constexpr (2 * k + 1 < NL) v[2 * k + 1] = static_cast<uint32_t>(q >> 32);
  });
}

template <class Lay, bool kVec16>
__device__ __forceinline__ void store_chunk(uint64_t* p, const uint32_t (&v)[Lay::kLimbs]) {
  constexpr int NW = Lay::kWords;
  constexpr int NL = Lay::kLimbs;
  auto limb = [&](auto I) -> uint32_t {
    constexpr int i = decltype(I)::value;
    if constexpr (i < NL) return v[i]; else return 0u;
  };
  if constexpr (kVec16 && NW % 2 == 0) {
    sfor<0, NW / 2>([&](auto I) {
      constexpr int k = decltype(I)::value;
      uint4 q;
      q.x = limb(ic<4 * k + 0>{});
      q.y = limb(ic<4 * k + 1>{});
      q.z = limb(ic<4 * k + 2>{});
      q.w = limb(ic<4 * k + 3>{});
      reinterpret_cast<uint4*>(p)[k] = q;
    });
  } else {
    sfor<0, NW>([&](auto I) {
      constexpr int k = decltype(I)::value;
      uint2 q;
      q.x = limb(ic<2 * k + 0>{});
      q.y = limb(ic<2 * k + 1>{});
      reinterpret_cast<uint2*>(p)[k] = q;
    });
  }
}

// Stores a whole counter (Lay::kWords words, 8-byte aligned) with 16-byte
// stores where the address allows: NW = 5 costs 3 stores (one L1 wavefront
// each) instead of 5.  The alignment is per lane (runtime).
template <class Lay>
__device__ __forceinline__ void store_counter(uint64_t* p, const uint32_t (&v)[Lay::kLimbs]) {
  constexpr int NW = Lay::kWords;
  constexpr int NL = Lay::kLimbs;
  auto limb = [&](auto I) -> uint32_t {
    constexpr int i = decltype(I)::value;
    if constexpr (i < NL) return v[i]; else return 0u;
  };
  auto st16 = [&](auto K, int word) {  // limbs 2K .. 2K+3 at word `word`
    constexpr int k = decltype(K)::value;
    uint4 q;
    q.x = limb(ic<2 * k + 0>{});
    q.y = limb(ic<2 * k + 1>{});
    q.z = limb(ic<2 * k + 2>{});
    q.w = limb(ic<2 * k + 3>{});
    *reinterpret_cast<uint4*>(p + word) = q;
  };
  auto st8 = [&](auto K, int word) {  // limbs 2K, 2K+1 at word `word`
    constexpr int k = decltype(K)::value;
    uint2 q;
    q.x = limb(ic<2 * k + 0>{});
    q.y = limb(ic<2 * k + 1>{});
    *reinterpret_cast<uint2*>(p + word) = q;
  };
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    sfor<0, NW / 2>([&](auto I) {
      constexpr int k = decltype(I)::value;
      st16(ic<2 * k>{}, 2 * k);
    });
    if constexpr (NW % 2) st8(ic<NW - 1>{}, NW - 1);
  } else {
    st8(ic<0>{}, 0);
    sfor<0, (NW - 1) / 2>([&](auto I) {
      constexpr int k = decltype(I)::value;
      st16(ic<2 * k + 1>{}, 2 * k + 1);
    });
    if constexpr (NW % 2 == 0) st8(ic<NW - 1>{}, NW - 1);
  }
}

template <class Lay>
__device__ __forceinline__ bool limbs_nonzero(const uint32_t (&x)[Lay::kLimbs]) {
  uint32_t any = 0;
  sfor<0, Lay::kLimbs>([&](auto I) { any |= x[decltype(I)::value]; });
  return any != 0;
}

template <class Lay>
__device__ __forceinline__ bool limbs_differ(const uint32_t (&x)[Lay::kLimbs],
                                             const uint32_t (&y)[Lay::kLimbs]) {
  uint32_t diff = 0;
  sfor<0, Lay::kLimbs>([&](auto I) {
    constexpr int i = decltype(I)::value;
    diff |= x[i] ^ y[i];
  });
  return diff != 0;
}

template <class Lay>
__device__ __forceinline__ void shfl_max(uint32_t (&x)[Lay::kLimbs], int offset) {
  uint32_t y[Lay::kLimbs];
  sfor<0, Lay::kLimbs>([&](auto I) {
    constexpr int i = decltype(I)::value;
    y[i] = __shfl_xor_sync(0xffffffffu, x[i], offset);
  });
  swar_max<Lay>(x, y);
}

// ---------------------------------------------------------------------------
// Estimator (counter_estimate, hll.hpp:122-141), bit-exact.
//
// r = 5: every term 2^-M of the reference's harmonic sum is a multiple of
// 2^-31 and there are at most 2^20 of them, so the sequential double sum is
// exact and equals S * 2^-31 with the integer S = sum 2^(31-M) (< 2^51).
// r >= 6: terms go down to 2^-61, so the reference's rounding sequence is
// replayed with sequential double adds in register order.
// raw = ((alpha*m)*m)/harmonic with IEEE round-to-nearest operations, and
// linear counting m*log(m/z) comes from a host table built with the same
// libm call as the reference (log_table[z], z = 1..m).
// ---------------------------------------------------------------------------
// Peer-push exchange of sharded steps (hanf_shard_attach): generation t+1
// of every peer rank, same row layout as the local one.  Each row a step
// writes locally is stored there too (NVLink peer memory), so no counter
// collective follows the sweep.
constexpr int kMaxPeers = 7;
struct PeerRows {
  uint64_t* next[kMaxPeers];
  double* est[kMaxPeers];  // relabelled shards: estimates of changed rows too
  // needed-rows filter: bit v of need[p] (word (v >> 6) - need_base) is set
  // iff some node of peer p's range has row v as a successor, i.e. peer p
  // can ever gather it; rows a peer never gathers are not pushed to it.
  // null = push every written row (filter off)
  const uint64_t* need[kMaxPeers];
  uint32_t need_base;  // first bitmap word of this shard's range (lo >> 6)
  uint32_t count;
  uint32_t push_est;
};

// Does peer p gather row v (a row of this shard's range)?
__device__ __forceinline__ bool peer_wants(const PeerRows& p, uint32_t i, uint32_t v) {
  const uint64_t* nd = p.need[i];
  return !nd || ((nd[(v >> 6) - p.need_base] >> (v & 63)) & 1);
}

struct EstimateParams {
  double alpha;
  double m;       // registers, as double
  uint32_t registers;
  uint32_t register_bits;
  uint32_t words;
  const double* log_table;  // [m+1]
};

__device__ __forceinline__ uint32_t read_register(const uint64_t* c, uint32_t r, uint32_t j) {
  const uint32_t bit = j * r;
  const uint32_t word = bit >> 6;
  const uint32_t off = bit & 63;
  uint64_t v = c[word] >> off;
  if (off + r > 64) v |= c[word + 1] << (64 - off);
  return static_cast<uint32_t>(v) & ((1u << r) - 1);
}

__device__ __forceinline__ double finish_estimate(const EstimateParams& p, double harmonic,
                                                  uint32_t zeros) {
  const double raw = __ddiv_rn(__dmul_rn(__dmul_rn(p.alpha, p.m), p.m), harmonic);
  if (raw <= __dmul_rn(2.5, p.m) && zeros > 0) return p.log_table[zeros];
  return raw;
}

// Generic path: any (m, r) the reference accepts.
__device__ inline double estimate_counter_generic(const uint64_t* c, const EstimateParams& p) {
  uint32_t zeros = 0;
  if (p.register_bits == 5) {
    uint64_t s = 0;
    for (uint32_t j = 0; j < p.registers; ++j) {
      const uint32_t reg = read_register(c, 5, j);
      s += 1ull << (31 - reg);
      zeros += reg == 0;
    }
    return finish_estimate(p, __dmul_rn(static_cast<double>(s), 0x1p-31), zeros);
  }
  double harmonic = 0.0;
  for (uint32_t j = 0; j < p.registers; ++j) {
    const uint32_t reg = read_register(c, p.register_bits, j);
    harmonic = __dadd_rn(harmonic, __longlong_as_double(static_cast<long long>(1023 - reg) << 52));
    zeros += reg == 0;
  }
  return finish_estimate(p, harmonic, zeros);
}

// Byte layout: M registers as M bytes at c (16-byte aligned).
template <int M>
__device__ __forceinline__ double estimate_counter_bytes(const uint64_t* c, const EstimateParams& p) {
  uint64_t s = 0;
  uint32_t zeros = 0;
  const uint4* q = reinterpret_cast<const uint4*>(c);
  sfor<0, M / 16>([&](auto I) { byte_terms(q[decltype(I)::value], s, zeros); });
  return finish_estimate(p, __dmul_rn(static_cast<double>(s), 0x1p-31), zeros);
}

// Fast path for r = 5 with a compile-time register count: the counter is
// read as 32-bit limbs and every register is extracted with one funnel
// shift; 2^(31-M) is one wrapping funnel shift of 0x80000000.
template <int M>
__device__ __forceinline__ double estimate_counter_r5(const uint64_t* c, const EstimateParams& p) {
  constexpr int kLimbs = (M * 5 + 31) / 32;
  constexpr int kWords = (M * 5 + 63) / 64;
  uint32_t v[kLimbs + 1];
  sfor<0, kWords>([&](auto I) {
    constexpr int k = decltype(I)::value;
    const uint64_t q = c[k];
    if constexpr (2 * k < kLimbs + 1) v[2 * k] = static_cast<uint32_t>(q);
    if constexpr (2 * k + 1 < kLimbs + 1) v[2 * k + 1] = static_cast<uint32_t>(q >> 32);
  });
  if constexpr (2 * kWords < kLimbs + 1) v[kLimbs] = 0;
  uint64_t s = 0;
  uint32_t zeros = 0;
  sfor<0, M>([&](auto J) {
    constexpr int j = decltype(J)::value;
    constexpr int bit = j * 5;
    constexpr int limb = bit / 32;
    constexpr int off = bit % 32;
    const uint32_t raw = __funnelshift_r(v[limb], v[limb + 1], off);  // low 5 bits = M_j
    const uint32_t term = __funnelshift_r(0x80000000u, 0u, raw);  // 2^(31 - M_j), shift mod 32
    s += term;
    zeros += term >> 31;
  });
  return finish_estimate(p, __dmul_rn(static_cast<double>(s), 0x1p-31), zeros);
}

// ---------------------------------------------------------------------------
// 256-bit window gathers (sm_100 LDG.E.ENL2.256).  Counter w of a layout
// with a W-word stride starts at byte 8*W*w, i.e. q = (W*w) mod 4 words into
// its 32-byte block.  The counter is read as K aligned 32-byte loads (one
// L1 wavefront each; the 8-byte loads they replace cost one per word) and
// shifted down by q words with selects.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ldg256(uint32_t (&v)[8], const uint64_t* p) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}

// 128-bit windows: counter w (W words, W odd) starts q = (W*w) mod 2 words
// into its 16-byte block; ceil((W+1)/2) aligned 16-byte loads, one select.
template <int NW>
struct Window128 {
  static_assert(NW % 2 == 1, "even strides are 16-byte aligned already");
  static constexpr int kLoads = (NW + 2) / 2;
};

template <int NW, int kPol = 0>
__device__ __forceinline__ void window128_load(uint4 (&raw)[Window128<NW>::kLoads],
                                               const uint64_t* base, uint32_t w) {
  const uint64_t word = static_cast<uint64_t>(w) * NW;
  const uint4* p = reinterpret_cast<const uint4*>(base + (word & ~1ull));
  sfor<0, Window128<NW>::kLoads>([&](auto I) {
    constexpr int k = decltype(I)::value;
    raw[k] = ld16<kPol>(p + k);
  });
}

template <class Lay, int NW>
__device__ __forceinline__ void window128_extract(uint32_t (&x)[Lay::kLimbs],
                                                  const uint4 (&raw)[Window128<NW>::kLoads],
                                                  uint32_t w) {
  const bool s1 = (w * NW) & 1u;
  auto at = [&](int i) -> uint32_t {
    const uint4& q = raw[i / 4];
    switch (i % 4) {
      case 0: return q.x;
      case 1: return q.y;
      case 2: return q.z;
      default: return q.w;
    }
  };
  sfor<0, Lay::kLimbs>([&](auto I) {
    constexpr int i = decltype(I)::value;
    x[i] = s1 ? at(i + 2) : at(i);
  });
}

// ---------------------------------------------------------------------------
// Estimator from a counter held in limbs (single-chunk layouts), same
// arithmetic as estimate_counter_* above.
// ---------------------------------------------------------------------------
template <class Lay>
__device__ __forceinline__ double estimate_limbs(const uint32_t (&x)[Lay::kLimbs],
                                                 const EstimateParams& p) {
  if constexpr (Lay::kBytes) {
    uint64_t s = 0;
    uint32_t zeros = 0;
    sfor<0, Lay::kLimbs / 4>([&](auto I) {
      constexpr int i = decltype(I)::value;
      byte_terms(make_uint4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]), s, zeros);
    });
    return finish_estimate(p, __dmul_rn(static_cast<double>(s), 0x1p-31), zeros);
  }
  constexpr int R = Lay::kR;
  constexpr int NL = Lay::kLimbs;
  auto limb = [&](int i) -> uint32_t { return i < NL ? x[i] : 0u; };
  uint32_t zeros = 0;
  if constexpr (R == 5) {
    uint64_t s = 0;
    sfor<0, Lay::kNReg>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int bit = j * 5;
      const uint32_t raw = __funnelshift_r(limb(bit / 32), limb(bit / 32 + 1), bit % 32);
      const uint32_t term = __funnelshift_r(0x80000000u, 0u, raw);  // 2^(31 - M_j)
      s += term;
      zeros += term >> 31;
    });
    return finish_estimate(p, __dmul_rn(static_cast<double>(s), 0x1p-31), zeros);
  } else {
    double harmonic = 0.0;
    sfor<0, Lay::kNReg>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int bit = j * R;
      const uint32_t reg =
          __funnelshift_r(limb(bit / 32), limb(bit / 32 + 1), bit % 32) & ((1u << R) - 1);
      harmonic = __dadd_rn(harmonic,
                           __longlong_as_double(static_cast<long long>(1023 - reg) << 52));
      zeros += reg == 0;
    });
    return finish_estimate(p, harmonic, zeros);
  }
}

}  // namespace hanf
