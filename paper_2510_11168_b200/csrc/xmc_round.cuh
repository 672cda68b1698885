// Device-side number formats, keyed RNG and rounding.
//
// Semantics follow the reference exactly where a bit-exact answer exists:
//   * grids, RTN ties-to-even, saturation    formats.py:164-206
//   * SR neighbours / probability / compare  formats.py:180-194, 209-225
//   * splitmix64 keyed uniforms              rng.py:15-57
// The "fast" SR mode replaces splitmix64 by keyed hash (or Philox4x32-7)
// words and the hardware cvt.rs stochastic-rounding conversion
// (distributional parity).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cstdint>

#include "xmc_ptx.cuh"

namespace xmc {

enum Fmt : int32_t { FMT_FP32 = 0, FMT_BF16 = 1, FMT_FP16 = 2, FMT_E4M3 = 3, FMT_E5M2 = 4 };
enum Rounding : int32_t { ROUND_NEAREST = 0, ROUND_SR_EXACT = 1, ROUND_SR_FAST = 2 };

// latched device error bits (the handle status word; xmc_head.h error convention)
enum StatusBits : int32_t {
  ST_NONFINITE_X = 1,
  ST_BAD_SAMPLE = 2,
  ST_NONFINITE_GRAD = 4,
  ST_LABEL_OUTSIDE = 8,
  ST_CAPACITY = 16,
  ST_NONFINITE_MOMENTS = 32,
  ST_PEER_TIMEOUT = 128,  // peer grad_X all-reduce: a peer's tile never arrived
};

// Grid parameters of an emulated (E, M) format (formats.py:49-137).
struct GridFmt {
  int32_t man_bits;
  int32_t min_normal_exp;
  int32_t max_exp;
  int32_t pad;
  double max_finite;
};

XMC_DEV float fast_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
XMC_DEV float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------- splitmix64
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {  // rng.py:22-25
  z = (z ^ (z >> 30)) * kM1;
  z = (z ^ (z >> 27)) * kM2;
  return z ^ (z >> 31);
}

// RoundingRng._base (rng.py:42-46)
__host__ __device__ __forceinline__ uint64_t sm64_base(uint64_t seed, uint64_t step,
                                                       uint64_t tensor_id) {
  uint64_t h = sm64_mix(seed + kGamma);
  h = sm64_mix(h + step * kGamma);
  return sm64_mix(h + tensor_id * kGamma);
}

// uniform in [0,1) as float64, rng.py:48-57
XMC_DEV double sm64_uniform(uint64_t base, uint64_t idx) {
  const uint64_t b = sm64_mix(base + idx * kGamma);
  return static_cast<double>(b >> 11) * (1.0 / 9007199254740992.0);
}

// -------------------------------------------------------- Philox4x32-10
struct U4 {
  uint32_t x, y, z, w;
};

// Philox4x32-R (Salmon et al., SC'11).  The update epilogue uses R = 7, the
// smallest round count the Random123 authors report as BigCrush-clean for
// Philox4x32 ("Philox4x32-7"); R = 10 is their default safety margin.
template <int ROUNDS>
XMC_DEV U4 philox4x32(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < ROUNDS; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}
constexpr int kPhiloxRounds = 7;

// Philox4x32-7 with the round keys computed once (k_i = k + i * W): the key
// schedule is the same for every counter of a launch
struct PhiloxKeys {
  uint32_t k0[kPhiloxRounds], k1[kPhiloxRounds];
  uint32_t hk0, hk1;   // 64-bit key of the hash generator (see sr_hash_word)
};
XMC_DEV PhiloxKeys philox_keys(uint64_t key) {
  PhiloxKeys ks;
  uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
  ks.hk0 = k0;
  ks.hk1 = k1;
#pragma unroll
  for (int i = 0; i < kPhiloxRounds; ++i) {
    ks.k0[i] = k0;
    ks.k1[i] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ks;
}
XMC_DEV U4 philox4x32_keys(U4 c, const PhiloxKeys& ks) {
#pragma unroll
  for (int i = 0; i < kPhiloxRounds; ++i) {
    // one 32x32->64 multiply each (IMAD.WIDE.U32), not a lo/hi pair
    const uint64_t m0 = static_cast<uint64_t>(0xD2511F53u) * c.x;
    const uint64_t m1 = static_cast<uint64_t>(0xCD9E8D57u) * c.z;
    c = U4{static_cast<uint32_t>(m1 >> 32) ^ c.y ^ ks.k0[i], static_cast<uint32_t>(m1),
           static_cast<uint32_t>(m0 >> 32) ^ c.w ^ ks.k1[i], static_cast<uint32_t>(m0)};
  }
  return c;
}

// Keyed hash generator of the SR_FAST words (the default sr_impl "hash").
// Word i (a 40-bit word index: element / 4 for e4m3x4, element / 2 for
// bf16x2) of the step keyed by key = splitmix64(seed, step, tensor_id)
// (rng.py:42-46) = RXS-M-XS(((lo32(i) ^ ka) * 747796405 + k1)), the PCG output
// permutation applied to a keyed affine image of the index, with
// ka = k0 ^ (hi32(i) * 0x9E3779B9).  Both key halves enter (XOR before the
// multiply, add after it), so two steps' word streams are unrelated
// permutations of the index space instead of shifted windows of one
// sequence, and indexes past 2^32 words get their own key.  Within a step the
// map i -> word is a bijection on each 2^32 block (no repeats).
XMC_DEV uint32_t sr_hash_word(uint32_t ilo, uint32_t ka, uint32_t k1) {
  const uint32_t st = (ilo ^ ka) * 747796405u + k1;
  const uint32_t w = ((st >> ((st >> 28u) + 4u)) ^ st) * 277803737u;
  return (w >> 22u) ^ w;
}
XMC_DEV uint32_t sr_hash_ka(const PhiloxKeys& ks, uint64_t word_index) {
  return ks.hk0 ^ (static_cast<uint32_t>(word_index >> 32) * 0x9E3779B9u);
}

XMC_DEV U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// ------------------------------------------------- generic exact rounding
XMC_DEV double grid_ulp(const GridFmt& f, double x) {  // formats.py:164-168
  int e;
  frexp(x, &e);
  int ex = e - 1;
  ex = ex < f.min_normal_exp ? f.min_normal_exp : (ex > f.max_exp ? f.max_exp : ex);
  return ldexp(1.0, ex - f.man_bits);
}

XMC_DEV double grid_saturate(const GridFmt& f, double q, double x) {  // formats.py:171-177
  return fabs(q) > f.max_finite ? copysign(f.max_finite, x) : q;
}

XMC_DEV float grid_round_nearest(const GridFmt& f, float xf) {  // formats.py:197-206
  const double x = static_cast<double>(xf);
  const double ulp = grid_ulp(f, x);
  return static_cast<float>(grid_saturate(f, rint(x / ulp) * ulp, x));
}

// formats.py:180-194 (neighbors) + 209-225 (round_stochastic); u from splitmix64.
XMC_DEV float grid_round_stochastic(const GridFmt& f, float xf, double u) {
  const double x = static_cast<double>(xf);
  const double ulp = grid_ulp(f, x);
  const double fq = x / ulp;
  double lo = grid_saturate(f, floor(fq) * ulp, x);
  double hi = grid_saturate(f, ceil(fq) * ulp, x);
  if (fabs(x) > f.max_finite) lo = hi = copysign(f.max_finite, x);
  const float lo32 = static_cast<float>(lo), hi32 = static_cast<float>(hi);
  const double width = static_cast<double>(hi32) - static_cast<double>(lo32);
  const double p = width > 0.0 ? (x - static_cast<double>(lo32)) / width : 0.0;
  return u < p ? hi32 : lo32;
}

__host__ __device__ inline GridFmt grid_of(int32_t fmt) {
  switch (fmt) {
    case FMT_BF16: return GridFmt{7, -126, 127, 0, 3.3895313892515355e38};
    case FMT_FP16: return GridFmt{10, -14, 15, 0, 65504.0};
    case FMT_E4M3: return GridFmt{3, -6, 8, 0, 448.0};
    case FMT_E5M2: return GridFmt{2, -14, 15, 0, 57344.0};
    default: return GridFmt{23, -126, 127, 0, 3.4028234663852886e38};
  }
}

// ------------------------------------------------------ native encodings
// e4m3 pair: hi byte <- a, lo byte <- b
XMC_DEV uint16_t cvt_e4m3x2_rn(float a, float b) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(a), "f"(b));
  return r;
}
XMC_DEV uint16_t cvt_e5m2x2_rn(float a, float b) {
  uint16_t r;
  asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(a), "f"(b));
  return r;
}
// bf16 pair, RTN with saturation to +-max_finite (the oracle never produces inf)
XMC_DEV uint32_t cvt_bf16x2_rn(float a, float b) {
  uint32_t r;
  asm("cvt.rn.satfinite.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
// hardware stochastic rounding (sm_100a), rbits supplies the random bits
XMC_DEV uint32_t cvt_e4m3x4_rs(float a, float b, float c, float d, uint32_t rbits) {
  uint32_t r;
  asm("cvt.rs.satfinite.e4m3x4.f32 %0, {%1, %2, %3, %4}, %5;"
      : "=r"(r)
      : "f"(a), "f"(b), "f"(c), "f"(d), "r"(rbits));
  return r;
}
XMC_DEV uint32_t cvt_bf16x2_rs(float a, float b, uint32_t rbits) {
  uint32_t r;
  asm("cvt.rs.satfinite.bf16x2.f32 %0, %1, %2, %3;" : "=r"(r) : "f"(a), "f"(b), "r"(rbits));
  return r;
}

XMC_DEV uint8_t enc_e4m3(float v) { return static_cast<uint8_t>(cvt_e4m3x2_rn(0.f, v) & 0xFF); }
XMC_DEV uint8_t enc_e5m2(float v) { return static_cast<uint8_t>(cvt_e5m2x2_rn(0.f, v) & 0xFF); }
XMC_DEV uint16_t enc_bf16(float v) { return static_cast<uint16_t>(cvt_bf16x2_rn(0.f, v) & 0xFFFF); }

XMC_DEV float dec_e4m3(uint8_t b) {
  __nv_fp8_e4m3 t;
  t.__x = b;
  return static_cast<float>(t);
}
XMC_DEV float dec_e5m2(uint8_t b) {
  __nv_fp8_e5m2 t;
  t.__x = b;
  return static_cast<float>(t);
}
XMC_DEV float dec_bf16(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }

// two e4m3 bytes (lo, hi of a 16-bit word) -> two floats
// keep a value in a register at this program point: volatile asms keep their
// order, so work feeding `pin` cannot sink past a later barrier wait
XMC_DEV void pin(uint32_t& v) { asm volatile("" : "+r"(v)); }
XMC_DEV void pin(float& v) { asm volatile("" : "+f"(v)); }

XMC_DEV float2 dec_e4m3x2(uint16_t v) {
  uint32_t h2;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(v));
  __half2 h = *reinterpret_cast<__half2*>(&h2);
  return __half22float2(h);  // .x <- low byte, .y <- high byte
}

}  // namespace xmc
