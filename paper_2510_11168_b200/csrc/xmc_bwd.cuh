// Kernel 2 of a head chunk: input-gradient accumulation and the gradient-fused
// SGD update, both on tcgen05, reading the chunk's G once per d-tile.
//
//   grad_X^T[j] += W_old[t, j]^T . G[t]         (M = 128 d, N = samples, K = 128 labels)
//   dW[t, j]     = G[t] . Xq[:, j]               (M = 128 labels, N = 128 d, K = samples)
//   W[t, j]      = ROUND(W_old - lr (dW + wd W_old))   in place, RTN / SR
//
// Reference: input_gradient_accumulate head.py:199-209 (pre-update W, called
// before the update head.py:290-291), fused_weight_update head.py:212-251,
// sgd_sr_step optimizers.py:51-74, round_nearest / round_stochastic
// formats.py:197-225, keys = global flat index r*d + c (head.py:244-247).
//
// Work decomposition: CTA c owns d-tile j = c % dtiles and walks label tiles
// t = c / dtiles + k * R.  Its grad_X^T[j] partial stays in TMEM for the whole
// launch and is flushed once to a workspace (deterministic reduce afterwards).
// The dW accumulator is double-buffered in TMEM so the update epilogue of tile
// i overlaps the MMAs of tile i+1.  dW never leaves TMEM/registers.
//
// Warp roles: warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warps 2..17 update epilogue: 4 warps per TMEM sub-partition, each owning 32
// of the tile's 128 d-columns for its 32 label rows.  Per tile the epilogue
// reads W_old and draws its random bits while the MMA is still running,
// releases the dW buffer right after tcgen05.ld, writes W_new into a swizzled
// smem tile and one thread per sub-partition TMA-stores its 32-row slab.
//
// Operand precision.  EB is the MMA operand / W storage width (1: e4m3 with
// kind::f8f6f4, 2: bf16 with kind::f16); GE is the grid the update rounds
// onto (GE = EB normally).  The reference-precision mode of an e4m3 head runs
// this kernel with EB = 2 on a bf16 copy of the W chunk (exact: every e4m3
// value is a bf16 value) and GE = 1, so the rounding still lands on the e4m3
// grid, while G arrives as three bf16 planes hi + mid + lo = fp32 g (a 3x
// longer K; BwdParams::xt_kc maps a G k-chunk onto its Xq^T k-chunk).
#pragma once

#include "xmc_ptx.cuh"
#include "xmc_round.cuh"

namespace xmc {

// Epilogue warps: 16, i.e. 4 per TMEM sub-partition.  The general path gives
// each warp 32 of the tile's 128 columns on every tile.  The FAST path runs
// them as two ping-pong groups of 8 warps (2 per sub-partition, 64 columns
// each) that take alternate tiles, so one tile's update may take two tiles'
// worth of MMA time without stalling the tensor pipe (each group owns one of
// the two dW accumulator buffers).
constexpr int kBwdEpiWarps = 16;
constexpr int kBwdThreads = 64 + kBwdEpiWarps * 32;


struct BwdParams {
  int32_t rows;          // labels in this chunk
  int32_t d;             // feature dim
  int32_t num_tiles;     // ceil(rows / 128)
  int32_t dtiles;        // ceil(d / 128); the last d-tile may be partial (d % 32 == 0)
  int32_t kc_count;      // sample k-chunks of G (Bp * EB / 128, x3 for the reference-precision planes)
  int32_t xt_kc;         // k-chunks of one Xq^T plane: G k-chunk kc multiplies Xq^T k-chunk kc % xt_kc
  int32_t do_update;     // dW + SGD + rounding, W written in place
  int32_t gx_kc0;        // first G k-chunk accumulated into grad_X
  int32_t gx_kc_count;   // 0 = no grad_X
  int32_t gx_group;      // G k-chunks per grad_X MMA group (N = gx_group x 128 / EB samples): gx_kc_count for one
                         // column group, xt_kc for the reference-precision planes, which accumulate into the
                         // same TMEM columns (grad_X^T = sum over planes of W^T G_plane)
  int32_t g_e5m2;        // EB = 1: G is e5m2 (x 2^8) instead of e4m3 (x 2^8)
  int32_t gx_cols;       // TMEM columns of the grad_X accumulator (samples of one column group / plane)
  int32_t g_prefetch;    // 1: the producer prefetches the next tile's G boxes into L2 (slot-by-slot path)
  int32_t gx_flush;      // > 0 (general path): drain the grad_X accumulator into the partial slot every
                         // gx_flush tiles, bounding the length of the tensor core's fp32 accumulation chain
  uint8_t* W;            // chunk base (row-major rows x d, EB bytes/elem), written in place
  uint8_t* comp;         // Kahan compensation, chunk base (comp_rows x d, CE bytes/elem) or null
  int32_t comp_rows;     // leading chunk rows that carry a compensation (top-p% head-Kahan)
  int64_t row0_global;   // global label of chunk row 0 (RNG key)
  float lr, wd, dw_scale;
  int32_t rounding;      // ROUND_NEAREST / ROUND_SR_EXACT / ROUND_SR_FAST
  uint64_t rng_base;     // splitmix64 base(seed, step, tensor_id); Philox / hash key
  int32_t sr_bits;       // ROUND_SR_FAST bits: 0 keyed hash, 1 Philox4x32-7
  float* gx_ws;          // [R][d][gx_ld] fp32 partials (gx_ld = padded batch x planes)
  int32_t gx_ld;
  int32_t gx_accumulate; // 1: add into the partial slot, 0: overwrite it
  const uint32_t* keep;  // keyed dropout keep bits [rows][d / 32] (chunk-local) or null
  float drop_scale;      // f32(1) / f32(1 - p) applied to kept dW (head.py:239-242)
  int32_t* status;
  // Adam-style head (ADAMW instantiation): fp32 moments [rows][d] at the chunk
  // base, comp (CE = 4) fp32, constants as kahan_adamw_step forms them
  float* adam_m;
  float* adam_v;
  float b1, b2, omb1, omb2, bc1, bc2, eps;
};

// SB: bytes per stored W element (the HBM tile, the update epilogue, W_new).
// SB < EB (reference precision of an e4m3 head): the epilogue converts each
// e4m3 W tile into a bf16 operand tile (kOpBytes) for the grad_X MMAs.
// CS: bytes per element of a compensation tile staged by TMA next to each W
// stage (2: the bf16 head-Kahan compensation of the fast path; 0: none)
template <int EB, bool XT_RES, int KCMAX, int SB = EB, int CS = 0>
struct BwdCfg {
  static_assert(SB == EB || (SB == 1 && EB == 2), "bf16 operands of an e4m3 head only");
  static constexpr bool kW8 = SB != EB;              // W stored e4m3, MMA operands bf16
  static constexpr int kBoxK = 128 / EB;             // elements per 128-B atom row (operands)
  static constexpr int kWBoxK = 128 / SB;            // elements per 128-B atom row (stored W)
  static constexpr int kBox = 128 * 128;             // one [128 rows x 128 B] box
  static constexpr int kWBoxes = SB;                 // d-tile of 128 stored elements
  static constexpr int kWBytes = kWBoxes * kBox;
  static constexpr int kOpBytes = kW8 ? EB * kBox : 0;   // bf16 W^T operand tile (kW8)
  // e4m3: W_new is staged in its own smem tile (kOutBytes), so the W_old slot
  // is released right after the epilogue has read it and the update never
  // waits for the grad_X MMAs still reading W_old; bf16 (no smem left for a
  // second tile) writes W_new in place after the grad_X MMAs completed.
  // (measured equal within box noise: in place / 1 / 2 staging tiles with
  // 5 / 4 / 3 W stages; two staging tiles need one named barrier per tile)
  // (kW8: the MMAs read the converted operand tile, never the W stage, so
  // W_new goes in place and the freed 32 KB deepen the G ring to 1.5 tiles:
  // the next tile's first G boxes load while this tile's grad_X runs)
  static constexpr int kOutTiles = (SB == 1 && !kW8) ? 2 : 0;   // W_new staging tiles (0 = in place)
  static constexpr bool kOutBuf = kOutTiles > 0;
  // e4m3: 4 W stages (224 KB with the staging tiles; 3 -> 4 measured -1.5 %
  // bwd); the G ring (6 slots = 3 tiles) must not get shallower (4 slots: +10 %)
  // (staged compensation: 2 stages of W + comp and a 4-slot G ring fit 227 KB)
  // (bf16 head, batch 256: 2 W stages free room for a 6-slot G ring, 1.5 tiles)
  static constexpr bool kBf16Deep = EB == 2 && !kW8 && XT_RES && KCMAX == 4;
  static constexpr int kWStages = CS ? 2 : (kW8 ? (KCMAX > 2 ? 2 : 4) : (EB == 1 ? 4 : (kBf16Deep ? 2 : 3)));
  static constexpr int kCompBytes = CS * kBox;        // [128 rows x 128 cols] comp tile (CS = 2: two boxes)
  static constexpr int kWStride = kWBytes + kCompBytes;
  static constexpr int kOutBytes = kOutTiles * kWBytes;
  static constexpr int kKSlot = kBox + (XT_RES ? 0 : kBox);
  // e4m3: 6 G slots (3 tiles at batch 256); batch 512 / 1024 (4 / 8 k-chunks
  // per tile) 4 slots to stay within the 227 KB
  // KCMAX = 0: the grad_X-only pass of a batch > 256 (no Xq^T, no update):
  // the freed space deepens the G ring to two tiles
  static constexpr int kKStages = KCMAX == 0 ? (EB == 1 ? 6 : 8)
                                             : (kW8 ? (XT_RES ? 6 : 4)
                                                    : (kBf16Deep ? 6 : (EB == 1 ? ((KCMAX > 2 || CS) ? 4 : 6) : 4)));
  static constexpr int kXtBytes = XT_RES ? KCMAX * kBox : 0;
  static constexpr int kBarBytes = 8 * (2 * kWStages + 2 * kKStages + 4 + 2 + 2 + 2) + 16;
  static constexpr int kSmemBytes =
      1024 + kXtBytes + kWStages * kWStride + kOpBytes + kOutBytes + kKStages * kKSlot + kBarBytes;
  static constexpr int kKmma = 32 / EB;              // K per MMA instruction (elements)
  static constexpr int kChunks16 = 2 * SB;           // 16-B smem chunks per thread (32 stored elements)
};

// byte offset of 16-B chunk `h` of this thread's 32 columns [c0, c0+32) in the
// 128-B-swizzled W tile (one [128 x 128 B] box per 128 / EB columns)
template <int EB>
XMC_DEV uint32_t w_chunk_off(int row, int c0, int h) {
  if constexpr (EB == 1) {
    const int cidx = (c0 >> 4) + h;
    return row * 128 + ((cidx ^ (row & 7)) << 4);
  } else {
    const int cidx = ((c0 & 63) >> 3) + h;
    return (c0 >> 6) * (128 * 128) + row * 128 + ((cidx ^ (row & 7)) << 4);
  }
}

template <int EB>
XMC_DEV void w_decode(const uint4 (&raw)[2 * EB], float (&w)[32]) {
  if constexpr (EB == 1) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t wv[4] = {raw[h].x, raw[h].y, raw[h].z, raw[h].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 a = dec_e4m3x2(static_cast<uint16_t>(wv[k] & 0xFFFF));
        const float2 b = dec_e4m3x2(static_cast<uint16_t>(wv[k] >> 16));
        w[h * 16 + 4 * k + 0] = a.x;
        w[h * 16 + 4 * k + 1] = a.y;
        w[h * 16 + 4 * k + 2] = b.x;
        w[h * 16 + 4 * k + 3] = b.y;
      }
    }
  } else {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint32_t wv[4] = {raw[h].x, raw[h].y, raw[h].z, raw[h].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[h * 8 + 2 * k + 0] = __uint_as_float(wv[k] << 16);
        w[h * 8 + 2 * k + 1] = __uint_as_float(wv[k] & 0xFFFF0000u);
      }
    }
  }
}

// SR_FAST random words for the 32 elements [flat0, flat0 + 32) (flat0 a
// multiple of 32): one word per cvt.rs instruction of the grid GE -- e4m3x4
// (4 elements; lanes (c,d) / (a,b) draw their 16 bits from rbits[15:0] /
// [31:16], profiles/r1_probe_cvt_rs.txt) or bf16x2 (2 elements).  Word w of
// the step is hash(w, key) (sr_hash_word) or Philox4x32-7 at counter w / 4;
// consecutive threads' word ranges are disjoint.
template <int GE>
XMC_DEV void sr_words(const PhiloxKeys& ks, int64_t flat0, uint32_t (&rw)[8 * GE], bool philox) {
  const uint64_t w0 = static_cast<uint64_t>(flat0) >> (GE == 1 ? 2 : 1);   // multiple of 8 * GE
  if (!philox) {
    const uint32_t ka = sr_hash_ka(ks, w0);
    const uint32_t lo = static_cast<uint32_t>(w0);
#pragma unroll
    for (int k = 0; k < 8 * GE; ++k) rw[k] = sr_hash_word(lo + k, ka, ks.hk1);
    return;
  }
#pragma unroll
  for (int h = 0; h < 2 * GE; ++h) {
    const uint64_t ctr = (w0 >> 2) + h;
    const U4 r = philox4x32_keys(U4{static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), GE - 1u, 0u}, ks);
    rw[4 * h + 0] = r.x;
    rw[4 * h + 1] = r.y;
    rw[4 * h + 2] = r.z;
    rw[4 * h + 3] = r.w;
  }
}

// bf16x2 word of two e4m3 values (exact: every e4m3 value is a bf16 value)
XMC_DEV uint32_t e4m3x2_to_bf16x2(uint16_t v) {
  const float2 f = dec_e4m3x2(v);
  return (__float_as_uint(f.x) >> 16) | (__float_as_uint(f.y) & 0xFFFF0000u);
}

// Round 4 consecutive fp32 values x[0..3] onto the GE grid (RTN, exact SR or
// hardware SR with word rw4[0] (GE = 1) / rw4[0..1] (GE = 2)), write the
// rounded values back into x and the EB storage words into out (1 word for
// EB = 1, 2 words for EB = 2).
template <int EB, int GE>
XMC_DEV void round4(const BwdParams& p, int rounding, float (&x)[4], const uint32_t* rw4, int64_t flat,
                    uint32_t* out) {
  static_assert(GE <= EB, "the storage holds the grid");
  if (rounding == ROUND_SR_EXACT) {
    const GridFmt gf = grid_of(GE == 1 ? FMT_E4M3 : FMT_BF16);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      x[e] = grid_round_stochastic(gf, x[e], sm64_uniform(p.rng_base, static_cast<uint64_t>(flat + e)));
  }
  if constexpr (GE == 1) {
    const uint32_t w4 = rounding == ROUND_SR_FAST
                            ? cvt_e4m3x4_rs(x[3], x[2], x[1], x[0], rw4[0])
                            : (cvt_e4m3x2_rn(x[1], x[0]) | (static_cast<uint32_t>(cvt_e4m3x2_rn(x[3], x[2])) << 16));
    const float2 lo = dec_e4m3x2(static_cast<uint16_t>(w4 & 0xFFFF));
    const float2 hi = dec_e4m3x2(static_cast<uint16_t>(w4 >> 16));
    x[0] = lo.x; x[1] = lo.y; x[2] = hi.x; x[3] = hi.y;
    if constexpr (EB == 1) {
      out[0] = w4;
    } else {
      out[0] = (__float_as_uint(x[0]) >> 16) | (__float_as_uint(x[1]) & 0xFFFF0000u);
      out[1] = (__float_as_uint(x[2]) >> 16) | (__float_as_uint(x[3]) & 0xFFFF0000u);
    }
  } else {
    const uint32_t w0 = rounding == ROUND_SR_FAST ? cvt_bf16x2_rs(x[1], x[0], rw4[0]) : cvt_bf16x2_rn(x[1], x[0]);
    const uint32_t w1 = rounding == ROUND_SR_FAST ? cvt_bf16x2_rs(x[3], x[2], rw4[1]) : cvt_bf16x2_rn(x[3], x[2]);
    out[0] = w0;
    out[1] = w1;
    x[0] = __uint_as_float(w0 << 16); x[1] = __uint_as_float(w0 & 0xFFFF0000u);
    x[2] = __uint_as_float(w1 << 16); x[3] = __uint_as_float(w1 & 0xFFFF0000u);
  }
}

// updated = w (1 - lr wd) - (lr * dw_scale) acc  (SGD with wd folded,
// optimizers.py:71-73, one rounding), rounded onto the GE grid and packed
// into the tile's EB storage bytes.  FMA contraction moves the fp32 update by
// <= 1 fp32 ulp, far below the tensor-core accumulation noise of acc.
template <int EB, int GE>
XMC_DEV void w_update_pack(const BwdParams& p, int rounding, const uint32_t (&acc)[32], const float (&w)[32],
                           const uint32_t (&rw)[8 * GE], int64_t flat0, uint4 (&out)[2 * EB]) {
  const float a_lr = -p.lr * p.dw_scale;
  const float c_wd = 1.0f - p.lr * p.wd;
  const uint64_t A2 = f2pack(a_lr, a_lr), C2 = f2pack(c_wd, c_wd);
  float u[32];
  if (p.wd != 0.0f) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint64_t r = ffma2(f2pack(__uint_as_float(acc[2 * k]), __uint_as_float(acc[2 * k + 1])), A2,
                               fmul2(f2pack(w[2 * k], w[2 * k + 1]), C2));
      f2unpack(r, u[2 * k], u[2 * k + 1]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint64_t r = ffma2(f2pack(__uint_as_float(acc[2 * k]), __uint_as_float(acc[2 * k + 1])), A2,
                               f2pack(w[2 * k], w[2 * k + 1]));
      f2unpack(r, u[2 * k], u[2 * k + 1]);
    }
  }
  uint32_t pk[8 * EB];
  if constexpr (EB == GE) {
    if (rounding == ROUND_SR_EXACT) {
      const GridFmt gf = grid_of(EB == 1 ? FMT_E4M3 : FMT_BF16);
#pragma unroll
      for (int k = 0; k < 32; ++k)
        u[k] = grid_round_stochastic(gf, u[k], sm64_uniform(p.rng_base, static_cast<uint64_t>(flat0 + k)));
    }
    if constexpr (EB == 1) {
      if (rounding == ROUND_SR_FAST) {
#pragma unroll
        for (int k = 0; k < 8; ++k) pk[k] = cvt_e4m3x4_rs(u[4 * k + 3], u[4 * k + 2], u[4 * k + 1], u[4 * k], rw[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          pk[k] = cvt_e4m3x2_rn(u[4 * k + 1], u[4 * k]) | (static_cast<uint32_t>(cvt_e4m3x2_rn(u[4 * k + 3], u[4 * k + 2])) << 16);
      }
    } else {
      if (rounding == ROUND_SR_FAST) {
#pragma unroll
        for (int k = 0; k < 16; ++k) pk[k] = cvt_bf16x2_rs(u[2 * k + 1], u[2 * k], rw[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) pk[k] = cvt_bf16x2_rn(u[2 * k + 1], u[2 * k]);
      }
    }
  } else {
    // e4m3 grid in bf16 storage (reference-precision mode of an e4m3 head)
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      float x[4] = {u[4 * g], u[4 * g + 1], u[4 * g + 2], u[4 * g + 3]};
      round4<EB, GE>(p, rounding, x, &rw[g], flat0 + 4 * g, &pk[2 * g]);
    }
  }
#pragma unroll
  for (int h = 0; h < 2 * EB; ++h) out[h] = make_uint4(pk[4 * h], pk[4 * h + 1], pk[4 * h + 2], pk[4 * h + 3]);
}

// 32-bit word `i` of a packed 16-B-chunk array (compile-time index)
template <int N>
XMC_DEV uint32_t word_of(const uint4 (&v)[N], int i) {
  const uint4 q = v[i >> 2];
  return (i & 3) == 0 ? q.x : ((i & 3) == 1 ? q.y : ((i & 3) == 2 ? q.z : q.w));
}

// elements 4g .. 4g+3 of a thread's 32 storage elements -> floats
template <int EB>
XMC_DEV void decode4(const uint4 (&raw)[2 * EB], int g, float (&w)[4]) {
  if constexpr (EB == 1) {
    const uint32_t wv = word_of(raw, g);
    const float2 lo = dec_e4m3x2(static_cast<uint16_t>(wv & 0xFFFF));
    const float2 hi = dec_e4m3x2(static_cast<uint16_t>(wv >> 16));
    w[0] = lo.x; w[1] = lo.y; w[2] = hi.x; w[3] = hi.y;
  } else {
    const uint32_t w0 = word_of(raw, 2 * g), w1 = word_of(raw, 2 * g + 1);
    w[0] = __uint_as_float(w0 << 16); w[1] = __uint_as_float(w0 & 0xFFFF0000u);
    w[2] = __uint_as_float(w1 << 16); w[3] = __uint_as_float(w1 & 0xFFFF0000u);
  }
}

// Head-Kahan variant (kahan_add formats.py:246-263 composed
// with the SGD update optimizers.py:51-74; PAPER.md:795 keeps the
// compensation in BF16):
//   v = -lr (g + wd s);  y = v - c;  t = ROUND(s + y);  c' = (t - s) - y;  s' = t
// Works 4 elements at a time straight from the packed W (`raw`) and comp
// (`craw`) registers so only acc[32] is live at full width.  comp (CE = 2:
// bf16, CE = 4: fp32) is read/written from/to HBM by the owning thread; rows
// without compensation (top-p% head-Kahan) pass craw = 0 and
// drop cout.
template <int EB, int CE, int GE>
XMC_DEV void w_update_pack_kahan(const BwdParams& p, int rounding, const uint32_t (&acc)[32], const uint4 (&raw)[2 * EB],
                                 const uint32_t (&rw)[8 * GE], int64_t flat0, const uint4 (&craw)[CE * 2],
                                 uint4 (&out)[2 * EB], uint4* cdst, uint64_t pol) {
  const float a_lr = -p.lr * p.dw_scale;
  const float b_wd = -p.lr * p.wd;
  uint32_t pk[8 * EB];
  uint32_t cw[4];   // one 16-B chunk of new compensation, stored as soon as it is complete
#pragma unroll
  for (int g = 0; g < 8; ++g) {   // elements 4g .. 4g+3
    float w[4], c[4];
    decode4<EB>(raw, g, w);
    if constexpr (CE == 2) {
      const uint32_t c0 = word_of(craw, 2 * g), c1 = word_of(craw, 2 * g + 1);
      c[0] = __uint_as_float(c0 << 16); c[1] = __uint_as_float(c0 & 0xFFFF0000u);
      c[2] = __uint_as_float(c1 << 16); c[3] = __uint_as_float(c1 & 0xFFFF0000u);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) c[e] = __uint_as_float(word_of(craw, 4 * g + e));
    }
    float y[4], t[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float v = fmaf(a_lr, __uint_as_float(acc[4 * g + e]), b_wd * w[e]);
      y[e] = v - c[e];
      t[e] = w[e] + y[e];
    }
    round4<EB, GE>(p, rounding, t, &rw[GE == 1 ? g : 2 * g], flat0 + 4 * g, &pk[EB == 1 ? g : 2 * g]);
    float cn[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) cn[e] = (t[e] - w[e]) - y[e];
    if constexpr (CE == 2) {
      cw[2 * (g & 1)] = cvt_bf16x2_rn(cn[1], cn[0]);
      cw[2 * (g & 1) + 1] = cvt_bf16x2_rn(cn[3], cn[2]);
      if ((g & 1) && cdst) st_global_v4_hint(cdst + (g >> 1), make_uint4(cw[0], cw[1], cw[2], cw[3]), pol);
    } else {
      if (cdst)
        st_global_v4_hint(cdst + g, make_uint4(__float_as_uint(cn[0]), __float_as_uint(cn[1]), __float_as_uint(cn[2]),
                                               __float_as_uint(cn[3])), pol);
    }
  }
#pragma unroll
  for (int h = 0; h < 2 * EB; ++h) out[h] = make_uint4(pk[4 * h], pk[4 * h + 1], pk[4 * h + 2], pk[4 * h + 3]);
}

// Adam-style head update (kahan_adamw_step optimizers.py:112-137 with the
// chunk gradient g = dW from TMEM, kahan_add formats.py:246-263 with RTN onto
// the grid), 4 elements at a time: m, v, comp fp32 read and written from/to
// HBM by the owning thread.  Every op explicitly rounded in the reference's
// order, so given the same dW the result is the reference's bit for bit.
template <int EB, int GE>
XMC_DEV void w_update_pack_adamw(const BwdParams& p, const uint32_t (&acc)[32], const uint4 (&raw)[2 * EB],
                                 int64_t eoff, bool row_ok, uint4 (&out)[2 * EB], uint64_t pol) {
  uint32_t pk[8 * EB];
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    float w[4];
    decode4<EB>(raw, g, w);
    float4* mp = reinterpret_cast<float4*>(p.adam_m + eoff) + g;
    float4* vp = reinterpret_cast<float4*>(p.adam_v + eoff) + g;
    float4* cp = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.comp) + eoff) + g;
    const float4 m4 = row_ok ? *mp : z4, v4 = row_ok ? *vp : z4, c4 = row_ok ? *cp : z4;
    const float mm[4] = {m4.x, m4.y, m4.z, m4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
    const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
    float m1[4], v1[4], y[4], t[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gg = __fmul_rn(__uint_as_float(acc[4 * g + e]), p.dw_scale);
      m1[e] = __fadd_rn(__fmul_rn(p.b1, mm[e]), __fmul_rn(p.omb1, gg));
      v1[e] = __fadd_rn(__fmul_rn(p.b2, vv[e]), __fmul_rn(__fmul_rn(p.omb2, gg), gg));
      const float mhat = __fdiv_rn(m1[e], p.bc1);
      const float vhat = __fdiv_rn(v1[e], p.bc2);
      const float upd = __fmul_rn(-p.lr, __fadd_rn(__fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), p.eps)),
                                                  __fmul_rn(p.wd, w[e])));
      y[e] = __fsub_rn(upd, cc[e]);
      t[e] = __fadd_rn(w[e], y[e]);
    }
    round4<EB, GE>(p, ROUND_NEAREST, t, nullptr, 0, &pk[EB == 1 ? g : 2 * g]);
    if (row_ok) {
      st_global_v4_hint(mp, make_uint4(__float_as_uint(m1[0]), __float_as_uint(m1[1]), __float_as_uint(m1[2]),
                                       __float_as_uint(m1[3])), pol);
      st_global_v4_hint(vp, make_uint4(__float_as_uint(v1[0]), __float_as_uint(v1[1]), __float_as_uint(v1[2]),
                                       __float_as_uint(v1[3])), pol);
      float cn[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) cn[e] = __fsub_rn(__fsub_rn(t[e], w[e]), y[e]);
      st_global_v4_hint(cp, make_uint4(__float_as_uint(cn[0]), __float_as_uint(cn[1]), __float_as_uint(cn[2]),
                                       __float_as_uint(cn[3])), pol);
    }
  }
#pragma unroll
  for (int h = 0; h < 2 * EB; ++h) out[h] = make_uint4(pk[4 * h], pk[4 * h + 1], pk[4 * h + 2], pk[4 * h + 3]);
}

// The kernel: CTA bid of the grid (d-tile bid % dtiles, row group bid / dtiles).
// FAST: the production specialisation (SR_FAST, e4m3, no compensation, no
// dropout mask) with every runtime mode switch folded away.
// the fast path stages a bf16 head-Kahan compensation by TMA
template <int CE, bool FAST>
__host__ __device__ constexpr int bwd_comp_staged() { return (FAST && CE == 2) ? 2 : 0; }

template <int EB, bool XT_RES, int KCMAX, int CE, bool FAST = false, bool ADAMW = false, int GE = EB, int SB = EB>
__global__ void __launch_bounds__(kBwdThreads, 1)
    xmc_bwd_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_g,
                   const __grid_constant__ CUtensorMap tm_xt, const __grid_constant__ CUtensorMap tm_ws,
                   const __grid_constant__ CUtensorMap tm_c, const BwdParams p_arg) {
  // a by-value copy: the compiler keeps launch-uniform fields in uniform
  // registers (a __grid_constant__ reference measured 17 % slower)
  BwdParams p = p_arg;
  constexpr int CS = bwd_comp_staged<CE, FAST>();
  using C = BwdCfg<EB, XT_RES, KCMAX, SB, CS>;
  static_assert(!ADAMW || (CE == 4 && !FAST), "the Adam-style head keeps an fp32 compensation");
  static_assert(!FAST || (EB == 1 && GE == 1 && (CE == 0 || CE == 2)),
                "the fast path is the e4m3 SR_FAST head (optionally with a bf16 Kahan compensation)");
  constexpr int WS = C::kWStages;
  constexpr int KS = C::kKStages;
  const int bid = static_cast<int>(blockIdx.x), nblk = static_cast<int>(gridDim.x);
  // FAST: SR_FAST or RTN (a warp-uniform branch at the rounding step)
  const int rounding = p.rounding;
  const bool fast_sr = !FAST || rounding == ROUND_SR_FAST;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xt_s = smem;
  uint8_t* w_s = smem + C::kXtBytes;
  uint8_t* op_s = w_s + WS * C::kWStride;      // bf16 W^T operand tile (kW8)
  uint8_t* out_s = op_s + C::kOpBytes;         // W_new staging tiles (kOutBuf)
  uint8_t* k_s = out_s + C::kOutBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(k_s + KS * C::kKSlot);
  uint64_t* w_full = bars;                 // [WS]
  uint64_t* w_empty = w_full + WS;         // [WS]
  uint64_t* k_full = w_empty + WS;         // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* t_full = k_empty + KS;         // [2]
  uint64_t* t_empty = t_full + 2;          // [2]
  uint64_t* xt_full = t_empty + 2;
  uint64_t* gx_full = xt_full + 1;
  uint64_t* op_full = gx_full + 1;         // kW8: operand tile converted (every epilogue warp)
  uint64_t* op_empty = op_full + 1;        // kW8: the tile's grad_X MMAs have read it
  uint64_t* gxw_full = op_empty + 1;       // a grad_X accumulation window is complete (gx_flush)
  uint64_t* gxw_empty = gxw_full + 1;      // ... and drained into the partial slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gxw_empty + 1);
  int32_t* status_s = reinterpret_cast<int32_t*>(tmem_slot + 1);

  const uint32_t warp = warp_id_sync();
  const int j = bid % p.dtiles;
  const int R = nblk / p.dtiles;
  const int r0 = bid / p.dtiles;
  const bool do_gx = p.gx_kc_count > 0;
  // kW8: the epilogue converts each e4m3 W tile to the bf16 operand tile
  const bool conv = C::kW8 && do_gx;
  // grad_X accumulation windows of gx_win tiles (general path only)
  const int gx_win = (!FAST && p.gx_flush > 0) ? p.gx_flush : 0x7fffffff;
  // this CTA's label tiles: r0, r0 + R, ... (the d-tile CTAs of a row group
  // walk them in step, so each G tile is requested by all six at once)
  const int ntl = r0 < p.num_tiles ? (p.num_tiles - r0 + R - 1) / R : 0;
  // label tiles in DESCENDING order: the forward walks them ascending, so
  // the first tiles here are the ones whose G (written evict_last) is still
  // in L2 when the backward starts
#ifdef XMC_BWD_ASCENDING
  auto tile_at = [&](int k) { return r0 + k * R; };
#else
  auto tile_at = [&](int k) { return p.num_tiles - 1 - (r0 + k * R); };
#endif
  // k-chunks (batch slices) a tile needs: all of them when the update runs
  // (dW sums over the whole batch), else only the grad_X column group's
  const int kb = p.do_update ? 0 : p.gx_kc0;
  const int ke = p.do_update ? p.kc_count : p.gx_kc0 + p.gx_kc_count;
  const int nk = ke - kb;
  // bytes a k slot receives: the G box, plus the streamed Xq^T box (dW only)
  const uint32_t kslot_bytes = (!XT_RES && p.do_update) ? C::kKSlot : C::kBox;

  if (warp == 0 && elect_one()) {
    prefetch_tmap(&tm_w);
    prefetch_tmap(&tm_g);
    prefetch_tmap(&tm_xt);
    if constexpr (CS > 0) prefetch_tmap(&tm_c);
    for (int s = 0; s < WS; ++s) {
      mbar_init(&w_full[s], 1);
      // MMA commit + (kOutBuf) every epilogue warp once it has read W_old, or
      // (in place) one store thread per TMEM sub-partition once W_new is stored
      // (kW8: the MMAs read the bf16 operand tile, not the stage: epilogue warps only)
      mbar_init(&w_empty[s], FAST ? 1 + kBwdEpiWarps / 2
                                  : (C::kOutBuf ? 1 + kBwdEpiWarps : (C::kW8 ? 4 : 5)));
    }
    for (int s = 0; s < KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&t_full[s], 1);
      mbar_init(&t_empty[s], FAST ? kBwdEpiWarps / 2 : kBwdEpiWarps);
    }
    mbar_init(xt_full, 1);
    mbar_init(gx_full, 1);
    mbar_init(op_full, kBwdEpiWarps);
    mbar_init(op_empty, 1);
    mbar_init(gxw_full, 1);
    mbar_init(gxw_empty, kBwdEpiWarps);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  // PDL: the prologue above (barriers, TMEM, tensor maps) overlapped the
  // previous kernel's tail; from here on its outputs are read
  griddep_wait();
  griddep_launch_dependents();
  ClkSpan::begin(1);
  // a latched error of an earlier kernel of the step turns this one into a
  // no-op; read once so every role of the CTA agrees
  if (threadIdx.x == 0) *status_s = *p.status;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_gx = tmem_base + 256;   // cols [256, 512): grad_X^T partial
  // cols [0,128) and [128,256): the two dW buffers
  // (shuffled from lane 0: provably warp-uniform, which keeps the role code
  // below on the uniform datapath -- a plain per-thread load cost ~17 %)
  const bool aborted = __shfl_sync(0xffffffffu, *status_s, 0) != 0;

  if (aborted) {
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    // A bulk-tensor copy instruction holds its thread for ~max(585, 1.8 x
    // 128-B lines of all its lanes) cycles (tools/probe_tma.cu), so a tile's
    // boxes go out together as ONE warp-wide instruction, lane l = box l.
    const int lane = static_cast<int>(lane_id());
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    if constexpr (XT_RES && KCMAX > 0) {
      if (lane == 0) mbar_arrive_expect_tx(xt_full, p.xt_kc * C::kBox);
      __syncwarp();
      if (lane < p.xt_kc)
        tma_load_2d_hint(xt_s + lane * C::kBox, &tm_xt, xt_full, lane * C::kBoxK, j * 128, pol_keep);
      __syncwarp();
    }
    int ws = 0, ks = 0;
    uint32_t wph = 0, kph = 0;
    // the tile's G slots are consecutive ring slots when the ring holds whole tiles
    const bool whole = nk > 0 && nk <= KS && KS % nk == 0;
    for (int it = 0; it < ntl; ++it) {
      const int tile = tile_at(it);
      mbar_wait_sleep(&w_empty[ws], wph ^ 1);
      if (whole) {
        for (int i = 0; i < nk; ++i) mbar_wait(&k_empty[ks + i], kph ^ 1);
        // staged compensation: the tile's comp boxes ride with its W stage
        // (only tiles with rows inside the compensated prefix)
        const int ncb = (CS > 0 && tile * 128 < p.comp_rows) ? CS : 0;
        if (lane == 0) {
#ifdef XMC_WHATIF_NO_WLOAD
          mbar_arrive_expect_tx(&w_full[ws], 0);
#else
          mbar_arrive_expect_tx(&w_full[ws], C::kWBytes + ncb * C::kBox);
#endif
          for (int i = 0; i < nk; ++i) mbar_arrive_expect_tx(&k_full[ks + i], kslot_bytes);
        }
        __syncwarp();
        // W boxes, then per k-chunk the G box (+ the Xq^T box when not resident)
        const int kGB = (!XT_RES && p.do_update) ? 2 : 1;
        const int gl = lane - C::kWBoxes;
        const int i = gl / kGB, sub = gl % kGB;
        const bool is_w = lane < C::kWBoxes;
        if constexpr (CS > 0) {   // comp box cb = lane - (W boxes + G boxes)
          const int cb = gl - nk * kGB;
          if (cb >= 0 && cb < ncb)
            tma_load_2d_hint(w_s + ws * C::kWStride + C::kWBytes + cb * C::kBox, &tm_c, &w_full[ws],
                             j * 128 + cb * 64, tile * 128, pol_stream);
        }
#ifdef XMC_WHATIF_NO_WLOAD
        const bool active = !is_w && (gl >= 0 && i < nk);
#else
        const bool active = is_w || (gl >= 0 && i < nk);
#endif
        const CUtensorMap* m = is_w ? &tm_w : (sub == 0 ? &tm_g : &tm_xt);
        uint8_t* dst = is_w ? w_s + ws * C::kWStride + lane * C::kBox : k_s + (ks + i) * C::kKSlot + sub * C::kBox;
        uint64_t* bar = is_w ? &w_full[ws] : &k_full[ks + i];
        const int kcg = kb + i;
        int xk = kcg;   // Xq^T k-chunk of G k-chunk kcg (kcg < 3 xt_kc)
        while (xk >= p.xt_kc) xk -= p.xt_kc;
        const int32_t c0 = is_w ? j * 128 + lane * C::kWBoxK : (sub == 0 ? kcg : xk) * C::kBoxK;
        const int32_t c1 = is_w ? tile * 128 : (sub == 0 ? tile * 128 : j * 128);
        if (active) tma_load_2d_hint(dst, m, bar, c0, c1, is_w ? pol_stream : pol_keep);
        __syncwarp();
        ks += nk;
        if (ks == KS) { ks = 0; kph ^= 1; }
      } else {
        // more k-chunks than ring slots (bf16 batch 512, reference-precision
        // planes): slot by slot
        if (lane == 0) mbar_arrive_expect_tx(&w_full[ws], C::kWBytes);
        __syncwarp();
        if (lane < C::kWBoxes)
          tma_load_2d_hint(w_s + ws * C::kWStride + lane * C::kBox, &tm_w, &w_full[ws], j * 128 + lane * C::kWBoxK,
                           tile * 128, pol_stream);
        __syncwarp();
        // the next tile's G boxes into L2 while this one streams from the ring
        // (the reference-precision planes: the ring holds only a plane or two)
        if (p.g_prefetch && it + 1 < ntl && lane < nk) tma_prefetch_2d(&tm_g, (kb + lane) * C::kBoxK, tile_at(it + 1) * 128);
        if constexpr (XT_RES) {
          // G boxes in batches of one grad_X group (one warp-wide instruction,
          // lane = box); groups never straddle the ring end (KS % bat == 0)
          const int bat = (KS % p.gx_group == 0 && nk % p.gx_group == 0) ? p.gx_group : 1;
          for (int kc = kb; kc < ke; kc += bat) {
            for (int i = 0; i < bat; ++i) mbar_wait(&k_empty[ks + i], kph ^ 1);
            if (lane < bat) {
              mbar_arrive_expect_tx(&k_full[ks + lane], kslot_bytes);
              tma_load_2d_hint(k_s + (ks + lane) * C::kKSlot, &tm_g, &k_full[ks + lane], (kc + lane) * C::kBoxK,
                               tile * 128, pol_keep);
            }
            __syncwarp();
            ks += bat;
            if (ks == KS) { ks = 0; kph ^= 1; }
          }
        } else {
          int xk = 0;   // Xq^T k-chunk of kc (kb = 0 whenever Xq^T is loaded)
          for (int kc = kb; kc < ke; ++kc) {
            mbar_wait(&k_empty[ks], kph ^ 1);
            uint8_t* slot = k_s + ks * C::kKSlot;
            if (lane == 0) mbar_arrive_expect_tx(&k_full[ks], kslot_bytes);
            __syncwarp();
            if (lane == 0) tma_load_2d_hint(slot, &tm_g, &k_full[ks], kc * C::kBoxK, tile * 128, pol_keep);
            if (lane == 1 && p.do_update)
              tma_load_2d_hint(slot + C::kBox, &tm_xt, &k_full[ks], xk * C::kBoxK, j * 128, pol_keep);
            __syncwarp();
            if (++xk == p.xt_kc) xk = 0;
            if (++ks == KS) { ks = 0; kph ^= 1; }
          }
        }
      }
      if (++ws == WS) { ws = 0; wph ^= 1; }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // e4m3 head: kind::f8f6f4 with G e4m3 or e5m2 (format code 1); bf16: kind::f16
    const uint32_t gf = EB == 1 ? (p.g_e5m2 ? 1u : 0u) : 1u;
    const uint32_t xf = EB == 1 ? 0u : 1u;
    const uint32_t idesc_dw = umma_idesc(gf, xf, false, false, 128, 128);                         // A = G, B = Xq
    const uint32_t idesc_gx = umma_idesc(xf, gf, true, true, 128, p.gx_group * C::kBoxK);         // A = W^T, B = G
    if constexpr (XT_RES && KCMAX > 0) mbar_wait(xt_full, 0);
    if constexpr (FAST) {
      // Production path, lean instruction stream (the MMA warp shares its
      // scheduler with 4 epilogue warps; with ~275 instructions per tile it
      // was itself the pipeline's critical path).  Descriptors are affine in
      // the smem address: built once, advanced by (byte offset >> 4).
      // Every tile's KCMAX G k-chunks are consecutive ring slots (KS % KCMAX == 0).
      static_assert(KS % KCMAX == 0, "whole tiles in the G ring");
      const uint64_t dG = umma_desc_sw128(smem_u32(k_s), 16, 1024);            // dW A: G, K-major
      const uint64_t dX = umma_desc_sw128(smem_u32(xt_s), 16, 1024);           // dW B: Xq^T, K-major
      const uint64_t dWt = umma_desc_sw128(smem_u32(w_s), C::kBox, 1024);      // grad_X A: W^T, MN-major
      static_assert(C::kWStride % 16 == 0, "stage stride in descriptor units");
      const uint64_t dGt = umma_desc_sw128(smem_u32(k_s), C::kKSlot, 1024);    // grad_X B: G, MN-major
      int ws = 0, ks = 0, ds = 0;
      uint32_t wph = 0, kph = 0, dph = 0;
      for (int it = 0; it < ntl; ++it) {
        mbar_wait(&w_full[ws], wph);
        mbar_wait(&t_empty[ds], dph ^ 1);
        tc_fence_after();
        const uint32_t d_dw = tmem_base + ds * 128;
#pragma unroll
        for (int kc = 0; kc < KCMAX; ++kc) {
          mbar_wait(&k_full[ks + kc], kph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ga = dG + ((static_cast<uint32_t>(ks + kc) * C::kKSlot) >> 4);
            const uint64_t xb = dX + ((kc * C::kBox) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_f8(d_dw, ga + 2 * k, xb + 2 * k, idesc_dw, (kc | k) != 0);
            if (kc == KCMAX - 1) mma_commit(&t_full[ds]);   // dW complete -> update epilogue
          }
          __syncwarp();
        }
        if (elect_one()) {
#ifdef XMC_WHATIF_NO_GX
          if (false) {
#else
          if (do_gx) {
#endif
            const uint64_t wa = dWt + ((static_cast<uint32_t>(ws) * C::kWStride) >> 4);
            const uint64_t gb = dGt + ((static_cast<uint32_t>(ks) * C::kKSlot) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_f8(tmem_gx, wa + 256 * k, gb + 256 * k, idesc_gx, (it | k) != 0);
          }
#pragma unroll
          for (int kc = 0; kc < KCMAX; ++kc) mma_commit(&k_empty[ks + kc]);
          mma_commit(&w_empty[ws]);
        }
        __syncwarp();
        ks += KCMAX;
        if (ks == KS) { ks = 0; kph ^= 1; }
        if (++ws == WS) { ws = 0; wph ^= 1; }
        if (++ds == 2) { ds = 0; dph ^= 1; }
      }
    }
    int ws = 0, ks = 0, ds = 0;
    uint32_t wph = 0, kph = 0, dph = 0;
    const int gsz = p.gx_group;   // k-chunks per grad_X MMA group
    // groups per accumulator: the column groups of one plane (reference
    // precision with N = 128 groups); group gi writes columns (gi % gpp) x N
    const int gpp = p.gx_cols / (gsz * C::kBoxK) > 0 ? p.gx_cols / (gsz * C::kBoxK) : 1;
    // Lean bookkeeping (the reference-precision backward issues 12 k-chunks a
    // tile and was bound by this warp's instruction stream, ~230 instructions
    // per k-chunk with runtime divisions): descriptors are affine in the smem
    // address (built once, advanced by byte offset >> 4) and the group /
    // window positions are running counters instead of % and /.
    const uint64_t dG0 = umma_desc_sw128(smem_u32(k_s), 16, 1024);                  // dW A: G, K-major
    const uint64_t dX0 = XT_RES ? umma_desc_sw128(smem_u32(xt_s), 16, 1024)         // dW B: Xq^T, K-major
                                : umma_desc_sw128(smem_u32(k_s) + C::kBox, 16, 1024);
    const uint64_t dGt0 = umma_desc_sw128(smem_u32(k_s), C::kKSlot, 1024);          // grad_X B: G, MN-major
    int win_pos = 0, win_idx = 0;   // it % gx_win, it / gx_win
    // groups of two k-chunks cover the whole tile from k-chunk 0, never wrap
    // the ring and never straddle an Xq^T plane boundary
    const bool pair_groups = gsz == 2 && do_gx && p.do_update && kb == 0 && p.gx_kc0 == 0 &&
                             p.gx_kc_count == ke && ke % 2 == 0 && KS % 2 == 0 && p.xt_kc % 2 == 0;
    for (int it = 0; it < (FAST ? 0 : ntl); ++it) {
      mbar_wait(&w_full[ws], wph);
      mbar_wait(&t_empty[ds], dph ^ 1);
      tc_fence_after();
      // grad_X A operand: the W stage, or (kW8) the bf16 tile the epilogue converted
      const uint32_t w_addr = C::kW8 ? smem_u32(op_s) : smem_u32(w_s + ws * C::kWStride);
      const uint64_t dA0 = umma_desc_sw128(w_addr, C::kBox, 1024);                  // grad_X A: W^T, MN-major
      const uint32_t d_dw = tmem_base + ds * 128;
      bool op_ready = !C::kW8;
      // a new accumulation window starts once the epilogue drained the last one
      const bool fresh = win_pos == 0;
      int gpos = 0, gi = 0, gcol = 0;   // gk % gsz, gk / gsz, (gk / gsz) % gpp
      bool gpast = false;               // gk / gsz >= gpp
      int xk = kb;   // Xq^T k-chunk of G k-chunk kc (the planes repeat it)
      while (xk >= p.xt_kc) xk -= p.xt_kc;
      if (pair_groups) {
        // every k-chunk in a grad_X group of two (reference-precision planes,
        // bf16 G of an e4m3 head): one pass per group, i.e. half the waits,
        // fences, elections and counter updates per MMA of the loop below;
        // same MMAs, same order per accumulator, same commits
        for (int kc = 0; kc < ke; kc += 2) {
          mbar_wait(&k_full[ks], kph);
          mbar_wait(&k_full[ks + 1], kph);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const uint64_t ad = dG0 + ((static_cast<uint32_t>(ks + b) * C::kKSlot) >> 4);
              const uint64_t bd = dX0 + (XT_RES ? ((static_cast<uint32_t>(xk + b) * C::kBox) >> 4)
                                                : ((static_cast<uint32_t>(ks + b) * C::kKSlot) >> 4));
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if constexpr (EB == 1) mma_f8(d_dw, ad + 2 * k, bd + 2 * k, idesc_dw, ((kc + b) | k) != 0);
                else mma_f16(d_dw, ad + 2 * k, bd + 2 * k, idesc_dw, ((kc + b) | k) != 0);
              }
            }
            if ((C::kOutBuf || C::kW8) && kc + 2 == ke) mma_commit(&t_full[ds]);
          }
          __syncwarp();
          // the grad_X group: the operand tile converted (kW8), the window's
          // accumulator drained (first group of a window)
          if (C::kW8 && !op_ready) {
            mbar_wait(op_full, static_cast<uint32_t>(it) & 1u);
            op_ready = true;
            tc_fence_after();
          }
          if (fresh && it > 0 && gi == 0) {
            mbar_wait(gxw_empty, static_cast<uint32_t>(win_idx - 1) & 1u);
            tc_fence_after();
          }
          if (elect_one()) {
            const bool acc0 = !fresh || gpast;
            const uint32_t d_gx = tmem_gx + gcol * 2 * C::kBoxK;
            const uint64_t bd0 = dGt0 + ((static_cast<uint32_t>(ks) * C::kKSlot) >> 4);
#pragma unroll
            for (int k = 0; k < 128 / C::kKmma; ++k) {
              constexpr uint32_t kStep = (C::kKmma * 128) >> 4;
              if constexpr (EB == 1) mma_f8(d_gx, dA0 + k * kStep, bd0 + k * kStep, idesc_gx, acc0 || k != 0);
              else mma_f16(d_gx, dA0 + k * kStep, bd0 + k * kStep, idesc_gx, acc0 || k != 0);
            }
            mma_commit(&k_empty[ks]);
            mma_commit(&k_empty[ks + 1]);
            if (!(C::kOutBuf || C::kW8) && kc + 2 == ke) mma_commit(&t_full[ds]);
          }
          __syncwarp();
          ++gi;
          if (++gcol == gpp) { gcol = 0; gpast = true; }
          xk += 2;
          if (xk == p.xt_kc) xk = 0;
          ks += 2;
          if (ks == KS) { ks = 0; kph ^= 1; }
        }
      }
      for (int kc = pair_groups ? ke : kb; kc < ke; ++kc) {
        mbar_wait(&k_full[ks], kph);
        const int gk = kc - p.gx_kc0;
        const bool in_gx = do_gx && gk >= 0 && gk < p.gx_kc_count;
        const bool gx_last = in_gx && gpos == gsz - 1;   // a grad_X group's G boxes are all in
        if (C::kW8 && gx_last && !op_ready) {
          mbar_wait(op_full, static_cast<uint32_t>(it) & 1u);
          op_ready = true;
        }
        if (gx_last && fresh && it > 0 && gi == 0)   // the window's first group
          mbar_wait(gxw_empty, static_cast<uint32_t>(win_idx - 1) & 1u);
        tc_fence_after();
        if (elect_one()) {
          if (p.do_update) {
            const uint64_t ad = dG0 + ((static_cast<uint32_t>(ks) * C::kKSlot) >> 4);
            const uint64_t bd = dX0 + (XT_RES ? ((static_cast<uint32_t>(xk) * C::kBox) >> 4)
                                              : ((static_cast<uint32_t>(ks) * C::kKSlot) >> 4));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if constexpr (EB == 1) mma_f8(d_dw, ad + 2 * k, bd + 2 * k, idesc_dw, (kc | k) != 0);
              else mma_f16(d_dw, ad + 2 * k, bd + 2 * k, idesc_dw, (kc | k) != 0);
            }
          }
          // dW complete -> hand it to the update epilogue before the grad_X
          // MMAs are queued (commit tracks only the MMAs issued so far)
          // (kW8: the grad_X MMAs read the operand tile, so W_new in place
          // does not have to wait for them either)
          if ((C::kOutBuf || C::kW8) && kc == ke - 1) mma_commit(&t_full[ds]);
          // grad_X^T: one MMA group with N = gsz k-chunks of samples, issued
          // once its G boxes (contiguous ring slots, LBO = slot pitch) landed;
          // W (A operand) is then read from smem once per group.  Groups of
          // the reference-precision planes accumulate into the same columns.
          if (gx_last) {
            const bool acc0 = !fresh || gpast;
            const uint32_t d_gx = tmem_gx + gcol * gsz * C::kBoxK;
            const int s0 = ks - gpos;   // ring slot of the group's first k-chunk
            if (s0 >= 0) {
              const uint64_t bd0 = dGt0 + ((static_cast<uint32_t>(s0) * C::kKSlot) >> 4);
#pragma unroll
              for (int k = 0; k < 128 / C::kKmma; ++k) {
                constexpr uint32_t kStep = (C::kKmma * 128) >> 4;   // K rows of one MMA, MN-major
                if constexpr (EB == 1) mma_f8(d_gx, dA0 + k * kStep, bd0 + k * kStep, idesc_gx, acc0 || k != 0);
                else mma_f16(d_gx, dA0 + k * kStep, bd0 + k * kStep, idesc_gx, acc0 || k != 0);
              }
              for (int s = s0; s <= ks; ++s) mma_commit(&k_empty[s]);
            } else {
              // the group wraps around the ring: one N = kBoxK MMA group per
              // k-chunk into its TMEM columns
              const uint32_t idesc_c = umma_idesc(xf, gf, true, true, 128, C::kBoxK);
              for (int c = 0; c <= gpos; ++c) {
                const int sc = s0 + c < 0 ? s0 + c + KS : s0 + c;
                const uint32_t gc = smem_u32(k_s + sc * C::kKSlot);
#pragma unroll
                for (int k = 0; k < 128 / C::kKmma; ++k) {
                  const uint64_t ad = umma_desc_sw128(w_addr + k * C::kKmma * 128, C::kBox, 1024);
                  const uint64_t bd = umma_desc_sw128(gc + k * C::kKmma * 128, C::kKSlot, 1024);
                  if constexpr (EB == 1) mma_f8(d_gx + c * C::kBoxK, ad, bd, idesc_c, acc0 || k != 0);
                  else mma_f16(d_gx + c * C::kBoxK, ad, bd, idesc_c, acc0 || k != 0);
                }
                mma_commit(&k_empty[sc]);
              }
            }
          } else if (!in_gx) {
            mma_commit(&k_empty[ks]);
          }
          // in place: dW is handed over only after the grad_X MMAs, which read
          // the W_old tile the epilogue overwrites with W_new
          if (!(C::kOutBuf || C::kW8) && kc == ke - 1) mma_commit(&t_full[ds]);
        }
        __syncwarp();
        if (in_gx && ++gpos == gsz) {
          gpos = 0;
          ++gi;
          if (++gcol == gpp) { gcol = 0; gpast = true; }
        }
        if (++xk == p.xt_kc) xk = 0;
        if (++ks == KS) { ks = 0; kph ^= 1; }
      }
      if (++win_pos == gx_win) { win_pos = 0; ++win_idx; }   // now (it + 1) % gx_win, (it + 1) / gx_win
      if (elect_one()) {
        if constexpr (C::kW8) {
          if (conv) mma_commit(op_empty);   // the stage itself is released by the epilogue
        } else {
          mma_commit(&w_empty[ws]);
        }
        if (do_gx && win_pos == 0 && it + 1 < ntl) mma_commit(gxw_full);
      }
      __syncwarp();
      if (++ws == WS) { ws = 0; wph ^= 1; }
      if (++ds == 2) { ds = 0; dph ^= 1; }
    }
    if (elect_one()) mma_commit(gx_full);
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;                 // 0 .. kBwdEpiWarps-1
    const int q = warp & 3;                  // TMEM sub-partition
    const int quarter = ew >> 2;             // which 32 of the 128 d-columns
    const int row = q * 32 + lane_id();
    const int c0 = quarter * 32;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    // the 4 warps of sub-partition q own rows [32q, 32q+32) of every tile;
    // they sync among themselves and one lane TMA-stores their 32-row slab
    const bool storer = (quarter == 0) && lane_id() == 0;
    const uint64_t pol_w_out = policy_evict_first();   // W_new streams out; keep L2 for G
    int ws = 0, ds = 0, prev_ws = -1;
    int ot_flip = 0;
    uint32_t wph = 0, dph = 0;
    const PhiloxKeys pk = philox_keys(p.rng_base);   // round keys, once per launch
    // grad_X^T accumulator (TMEM lane = d index) into this CTA's slot of the
    // [R][d][gx_ld] partial buffer; the chunks (and accumulation windows) of
    // one step add into it (stream-ordered, one owner per slot: deterministic)
    auto gx_drain = [&](bool accumulate) {
      const int nchunks = j * 128 + row < p.d ? p.gx_cols / 32 : 0;
      float* dst = p.gx_ws + (static_cast<int64_t>(r0) * p.d + j * 128 + row) * p.gx_ld + p.gx_kc0 * C::kBoxK;
#pragma unroll 1
      for (int cch = quarter; cch < nchunks; cch += 4) {
        uint32_t r[32];
        tmem_ld32(tmem_gx + lane_off + cch * 32, r);
        tmem_ld_wait();
        float4* o = reinterpret_cast<float4*>(dst + cch * 32);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float4 v = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                 __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
          if (accumulate) {
            const float4 old = o[k];
            v.x += old.x;
            v.y += old.y;
            v.z += old.z;
            v.w += old.w;
          }
          o[k] = v;
        }
      }
    };
    if constexpr (FAST) {
      // ---- production path (e4m3, SR_FAST, no compensation / dropout):
      // ping-pong groups.  Group g = ew / 8 takes tiles it = g, g + 2, ... and
      // owns dW buffer g; its warp (q, half) updates rows [32q, 32q+32) x
      // columns [64 half, 64 half + 64).  Per tile: W_old of both 32-column
      // groups and the first group's SR words / decoded, (1 - lr wd)-scaled
      // W_old are ready BEFORE the dW wait (they overlap the MMAs).
      const int g = ew >> 3;
      const int half = (ew >> 2) & 1;
      const int cw0 = half * 64;
      const bool gstorer = half == 0 && lane_id() == 0;
      const float c_wd = 1.0f - p.lr * p.wd;
      const float a_lr = -p.lr * p.dw_scale;
      uint8_t* ot = out_s + g * C::kWBytes;          // this group's W_new staging tile
      const uint32_t ot_s = smem_u32(ot);
      bool stored = false;
      if constexpr (CE == 2) {
        // ---- head-Kahan (bf16 compensation, formats.py:246-263 composed
        // with sgd_sr_step): the comp tile rides with the W
        // stage (TMA), both are read into registers before the stage is
        // released; dW is read 16 columns at a time to keep W_old, comp and
        // the SR words live; comp' goes out by st.global (rows inside the
        // compensated prefix only), W_new through the staging tile.
        const float b_wd = -p.lr * p.wd;
        const uint64_t pol_c = policy_evict_first();
        for (int it = g; it < ntl; it += 2) {
          const int tile = tile_at(it);
          const int wsi = it % WS;
          const uint32_t wphi = static_cast<uint32_t>(it / WS) & 1u;
          const uint32_t dphi = static_cast<uint32_t>(it >> 1) & 1u;
          const uint32_t wt_s = smem_u32(w_s + wsi * C::kWStride);
          const uint32_t ct_s = wt_s + C::kWBytes;
          mbar_wait(&w_full[wsi], wphi);
          const int64_t grow = static_cast<int64_t>(tile) * 128 + row;
          const int64_t flat0 = (p.row0_global + grow) * static_cast<int64_t>(p.d) + j * 128 + cw0;
          const bool tile_c = tile * 128 < p.comp_rows;           // the producer loaded its comp boxes
          const bool krow = grow < p.comp_rows && j * 128 + cw0 < p.d;   // this thread stores comp'
          uint4 raw[4], craw[8];
#pragma unroll
          for (int h = 0; h < 4; ++h) raw[h] = lds128(wt_s + w_chunk_off<EB>(row, cw0 + (h >> 1) * 32, h & 1));
#pragma unroll
          for (int h = 0; h < 8; ++h)
            craw[h] = tile_c ? lds128(ct_s + w_chunk_off<2>(row, cw0 + (h >> 2) * 32, h & 3)) : make_uint4(0, 0, 0, 0);
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&w_empty[wsi]);
          uint32_t rw[8];
          if (fast_sr) sr_words<1>(pk, flat0, rw, p.sr_bits != 0);
          if (gstorer && stored) bulk_wait_read<0>();
          named_bar_sync(1 + q + 4 * g, 64);
          mbar_wait_sleep(&t_full[g], dphi);
          tc_fence_after();
#pragma unroll
          for (int cg = 0; cg < 2; ++cg) {
            if (cg == 1 && fast_sr) sr_words<1>(pk, flat0 + 32, rw, p.sr_bits != 0);
            uint32_t pk8[8];
#pragma unroll
            for (int qt = 0; qt < 2; ++qt) {
              uint32_t acc[16];
              tmem_ld16(tmem_base + lane_off + g * 128 + cw0 + cg * 32 + qt * 16, acc);
              tmem_ld_wait();
              if (cg == 1 && qt == 1) {
                tc_fence_before();
                __syncwarp();
                if (lane_id() == 0) mbar_arrive(&t_empty[g]);
              }
              uint32_t cw[8];
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                const int e = cg * 32 + qt * 16 + 4 * k4;   // element of the thread's 64
                const uint32_t wv = word_of(raw, e >> 2);
                const float2 w01 = dec_e4m3x2(static_cast<uint16_t>(wv & 0xFFFF));
                const float2 w23 = dec_e4m3x2(static_cast<uint16_t>(wv >> 16));
                const float w[4] = {w01.x, w01.y, w23.x, w23.y};
                const uint32_t c0w = word_of(craw, e >> 1), c1w = word_of(craw, (e >> 1) + 1);
                const float c[4] = {__uint_as_float(c0w << 16), __uint_as_float(c0w & 0xFFFF0000u),
                                    __uint_as_float(c1w << 16), __uint_as_float(c1w & 0xFFFF0000u)};
                float y[4], t[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                  const float v = fmaf(a_lr, __uint_as_float(acc[4 * k4 + x]), b_wd * w[x]);
                  y[x] = v - c[x];
                  t[x] = w[x] + y[x];
                }
                const uint32_t w4 = fast_sr ? cvt_e4m3x4_rs(t[3], t[2], t[1], t[0], rw[qt * 4 + k4])
                                            : (cvt_e4m3x2_rn(t[1], t[0]) |
                                               (static_cast<uint32_t>(cvt_e4m3x2_rn(t[3], t[2])) << 16));
                pk8[qt * 4 + k4] = w4;
                const float2 r01 = dec_e4m3x2(static_cast<uint16_t>(w4 & 0xFFFF));
                const float2 r23 = dec_e4m3x2(static_cast<uint16_t>(w4 >> 16));
                const float tr[4] = {r01.x, r01.y, r23.x, r23.y};
                float cn[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) cn[x] = (tr[x] - w[x]) - y[x];
                cw[2 * k4] = cvt_bf16x2_rn(cn[1], cn[0]);
                cw[2 * k4 + 1] = cvt_bf16x2_rn(cn[3], cn[2]);
              }
              if (krow) {
                uint4* cdst = reinterpret_cast<uint4*>(p.comp + (grow * p.d + j * 128 + cw0 + cg * 32 + qt * 16) * 2);
                st_global_v4_hint(cdst, make_uint4(cw[0], cw[1], cw[2], cw[3]), pol_c);
                st_global_v4_hint(cdst + 1, make_uint4(cw[4], cw[5], cw[6], cw[7]), pol_c);
              }
            }
            const int cc = cw0 + cg * 32;
            sts128(ot_s + w_chunk_off<EB>(row, cc, 0), make_uint4(pk8[0], pk8[1], pk8[2], pk8[3]));
            sts128(ot_s + w_chunk_off<EB>(row, cc, 1), make_uint4(pk8[4], pk8[5], pk8[6], pk8[7]));
          }
          fence_proxy_async_smem();
          named_bar_sync(1 + q + 4 * g, 64);
          if (gstorer) {
            tma_store_2d_hint(&tm_ws, ot + q * 32 * 128, j * 128, tile * 128 + q * 32, pol_w_out);
            bulk_commit();
            stored = true;
          }
        }
      }
      for (int it = g; it < (CE == 2 ? 0 : ntl); it += 2) {
        const int tile = tile_at(it);
        const int wsi = it % WS;
        const uint32_t wphi = static_cast<uint32_t>(it / WS) & 1u;
        const uint32_t dphi = static_cast<uint32_t>(it >> 1) & 1u;
        const uint32_t wt_s = smem_u32(w_s + wsi * C::kWStride);
        mbar_wait(&w_full[wsi], wphi);
        const int64_t grow = static_cast<int64_t>(tile) * 128 + row;
        const int64_t flat0 = (p.row0_global + grow) * static_cast<int64_t>(p.d) + j * 128 + cw0;
        uint4 raw[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) raw[h] = lds128(wt_s + w_chunk_off<EB>(row, cw0 + (h >> 1) * 32, h & 1));
#ifdef XMC_WHATIF_NO_WLOAD
        for (int h = 0; h < 4; ++h) raw[h] = make_uint4(raw[h].x & 0x3F3F3F3Fu, raw[h].y & 0x3F3F3F3Fu, raw[h].z & 0x3F3F3F3Fu, raw[h].w & 0x3F3F3F3Fu);
#endif
        // W_old is in registers: the slot can be refilled once the MMAs are done too
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&w_empty[wsi]);
        auto prep = [&](int cg, uint32_t (&rw)[8], float (&wc)[32]) {
#ifdef XMC_WHATIF_NO_EPI_MATH
          for (int k = 0; k < 8; ++k) rw[k] = word_of(raw, 4 * cg + (k & 3)) ^ k;
          for (int k = 0; k < 32; ++k) wc[k] = 0.f;
          return;
#endif
          if (fast_sr) sr_words<1>(pk, flat0 + cg * 32, rw, p.sr_bits != 0);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 r4 = raw[2 * cg + h];
            const uint32_t wv[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 lo = dec_e4m3x2(static_cast<uint16_t>(wv[k] & 0xFFFF));
              const float2 hi = dec_e4m3x2(static_cast<uint16_t>(wv[k] >> 16));
              wc[h * 16 + 4 * k + 0] = lo.x;
              wc[h * 16 + 4 * k + 1] = lo.y;
              wc[h * 16 + 4 * k + 2] = hi.x;
              wc[h * 16 + 4 * k + 3] = hi.y;
            }
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) {   // w (1 - lr wd)  (optimizers.py:71-73, wd folded)
            const uint64_t r = fmul2(f2pack(wc[2 * k], wc[2 * k + 1]), f2pack(c_wd, c_wd));
            f2unpack(r, wc[2 * k], wc[2 * k + 1]);
          }
        };
        // updated = w (1 - lr wd) - lr dW, one SR rounding onto e4m3 (cvt.rs)
        auto finish = [&](int cg, const uint32_t (&acc)[32], const uint32_t (&rw)[8], const float (&wc)[32]) {
          uint32_t pk8[8];
#ifdef XMC_WHATIF_NO_EPI_MATH
          for (int k = 0; k < 8; ++k) pk8[k] = (acc[4 * k] ^ rw[k]) & 0x3F3F3F3Fu;
          if (false)
#endif
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float u[4];
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const uint64_t r = ffma2(f2pack(__uint_as_float(acc[4 * k + e]), __uint_as_float(acc[4 * k + e + 1])),
                                       f2pack(a_lr, a_lr), f2pack(wc[4 * k + e], wc[4 * k + e + 1]));
              f2unpack(r, u[e], u[e + 1]);
            }
            pk8[k] = fast_sr ? cvt_e4m3x4_rs(u[3], u[2], u[1], u[0], rw[k])
                             : (cvt_e4m3x2_rn(u[1], u[0]) | (static_cast<uint32_t>(cvt_e4m3x2_rn(u[3], u[2])) << 16));
          }
          const int cc = cw0 + cg * 32;
          sts128(ot_s + w_chunk_off<EB>(row, cc, 0), make_uint4(pk8[0], pk8[1], pk8[2], pk8[3]));
          sts128(ot_s + w_chunk_off<EB>(row, cc, 1), make_uint4(pk8[4], pk8[5], pk8[6], pk8[7]));
        };
        uint32_t rw[8];
        float wc[32];
        prep(0, rw, wc);
#pragma unroll
        for (int k = 0; k < 8; ++k) pin(rw[k]);
#pragma unroll
        for (int k = 0; k < 32; ++k) pin(wc[k]);
        // this group's previous W_new store must have read the staging tile
        if (gstorer && stored) bulk_wait_read<0>();
        named_bar_sync(1 + q + 4 * g, 64);
        mbar_wait_sleep(&t_full[g], dphi);   // off the critical path: do not steal issue slots
        tc_fence_after();
        {
          uint32_t acc[32];
          tmem_ld32(tmem_base + lane_off + g * 128 + cw0, acc);
          tmem_ld_wait();
          finish(0, acc, rw, wc);
        }
        {
          uint32_t acc[32];
          tmem_ld32(tmem_base + lane_off + g * 128 + cw0 + 32, acc);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&t_empty[g]);
          prep(1, rw, wc);
          finish(1, acc, rw, wc);
        }
        fence_proxy_async_smem();
        named_bar_sync(1 + q + 4 * g, 64);
#ifdef XMC_WHATIF_NO_WSTORE
        if (false) {
#else
        if (gstorer) {
#endif
          tma_store_2d_hint(&tm_ws, ot + q * 32 * 128, j * 128, tile * 128 + q * 32, pol_w_out);
          bulk_commit();
          stored = true;
        }
      }
      if (gstorer && stored) bulk_wait<0>();
    }
    for (int it = 0; it < (FAST ? 0 : ntl); ++it) {
      const int tile = tile_at(it);
      uint8_t* wt = w_s + ws * C::kWStride;
      mbar_wait(&w_full[ws], wph);
      const uint32_t wt_s = smem_u32(wt);
      uint4 raw[C::kChunks16];
      if (p.do_update || conv) {
#pragma unroll
        for (int h = 0; h < C::kChunks16; ++h) raw[h] = lds128(wt_s + w_chunk_off<SB>(row, c0, h));
      }
      if constexpr (C::kW8) {
        if (conv) {
          // e4m3 W_old -> the bf16 grad_X operand tile (exact), same swizzled
          // layout a bf16 TMA box would have; the MMA warp waits on op_full
          mbar_wait(op_empty, (static_cast<uint32_t>(it) & 1u) ^ 1u);
          const uint32_t op = smem_u32(op_s);
#pragma unroll
          for (int h = 0; h < 4; ++h) {   // bf16 16-B chunk h = e4m3 elements [8h, 8h + 8)
            const uint32_t w0 = word_of(raw, 2 * h), w1 = word_of(raw, 2 * h + 1);
            sts128(op + w_chunk_off<2>(row, c0, h),
                   make_uint4(e4m3x2_to_bf16x2(static_cast<uint16_t>(w0 & 0xFFFF)),
                              e4m3x2_to_bf16x2(static_cast<uint16_t>(w0 >> 16)),
                              e4m3x2_to_bf16x2(static_cast<uint16_t>(w1 & 0xFFFF)),
                              e4m3x2_to_bf16x2(static_cast<uint16_t>(w1 >> 16))));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(op_full);
        }
      }
      if (p.do_update) {
        const int64_t grow = static_cast<int64_t>(tile) * 128 + row;
        const int64_t flat0 = (p.row0_global + grow) * static_cast<int64_t>(p.d) + j * 128 + c0;
        // --- independent of dW: W_old and random bits, overlapping the MMAs
        if constexpr (C::kOutBuf) {
          // W_old is in registers: the slot can be refilled once the MMAs are done too
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&w_empty[ws]);
        } else if (storer && prev_ws >= 0) {
          // lazily release the previous tile's W slot: its TMA store has had a
          // tile's worth of time to read the smem, so this rarely waits
          bulk_wait_read<0>();
          mbar_arrive(&w_empty[prev_ws]);
          prev_ws = -1;
        }
        uint4 craw[CE > 0 ? CE * 2 : 1];
        // columns past d (partial last d-tile) are computed on TMA's zero fill
        // and clipped by the TMA store; per-thread side buffers skip them
        const bool col_ok = j * 128 + c0 < p.d;
        const bool krow = CE > 0 && grow < p.comp_rows && col_ok;   // this row carries a compensation
        if constexpr (CE > 0 && !ADAMW) {   // Kahan compensation of this thread's 32 elements (HBM)
          const uint4* csrc = reinterpret_cast<const uint4*>(p.comp + (grow * p.d + j * 128 + c0) * CE);
#pragma unroll
          for (int h = 0; h < CE * 2; ++h) craw[h] = krow ? __ldg(csrc + h) : make_uint4(0u, 0u, 0u, 0u);
        }
        uint32_t km = 0u;   // dropout keep bits of this thread's 32 columns
        if (p.keep != nullptr && grow < p.rows && col_ok)
          km = __ldg(p.keep + grow * (p.d >> 5) + ((j * 128 + c0) >> 5));
        uint32_t rw[8 * GE];
        if (rounding == ROUND_SR_FAST) sr_words<GE>(pk, flat0, rw, p.sr_bits != 0);
        float w[CE > 0 ? 1 : 32];
        if constexpr (CE == 0) w_decode<SB>(raw, w);
        // --- dW from TMEM, then release the accumulator buffer at once
        mbar_wait(&t_full[ds], dph);
        tc_fence_after();
        uint32_t acc[32];
        tmem_ld32(tmem_base + lane_off + ds * 128 + c0, acc);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&t_empty[ds]);
        if (p.keep != nullptr) {   // scratch *= mask / (1 - p)  (head.py:239-242)
#pragma unroll
          for (int k = 0; k < 32; ++k)
            acc[k] = __float_as_uint(__uint_as_float(acc[k]) * (((km >> k) & 1u) ? p.drop_scale : 0.0f));
        }
        uint4 out[C::kChunks16];
        if constexpr (ADAMW) {
          w_update_pack_adamw<SB, GE>(p, acc, raw, grow * p.d + j * 128 + c0, grow < p.rows && col_ok, out, pol_w_out);
        } else if constexpr (CE > 0) {
          uint4* cdst = krow ? reinterpret_cast<uint4*>(p.comp + (grow * p.d + j * 128 + c0) * CE) : nullptr;
          w_update_pack_kahan<SB, CE, GE>(p, rounding, acc, raw, rw, flat0, craw, out, cdst, pol_w_out);
        } else {
          w_update_pack<SB, GE>(p, rounding, acc, w, rw, flat0, out);
        }
        // W_new into a swizzled smem tile (the staging tile, or in place once
        // the grad_X MMAs have read W_old), then one TMA store per 32-row slab
        // (full 128-B lines to HBM, no LSU traffic)
        uint8_t* ot = wt;
        if constexpr (C::kOutTiles == 2) {
          ot = out_s + (ot_flip & 1) * C::kWBytes;
          ++ot_flip;
        }
        const uint32_t ot_s = smem_u32(ot);
#pragma unroll
        for (int h = 0; h < C::kChunks16; ++h) sts128(ot_s + w_chunk_off<SB>(row, c0, h), out[h]);
        fence_proxy_async_smem();
        // two staging tiles: before this barrier the storer waits until the
        // previous tile's store (the only one outstanding) has read its smem,
        // so after it every warp may overwrite that tile on the next tile
        if (C::kOutTiles == 2 && storer && prev_ws >= 0) bulk_wait_read<0>();
        named_bar_sync(1 + q, 128);
        if (storer) {
#pragma unroll
          for (int b = 0; b < C::kWBoxes; ++b)
            tma_store_2d_hint(&tm_ws, ot + b * C::kBox + q * 32 * 128, j * 128 + b * C::kWBoxK, tile * 128 + q * 32,
                              pol_w_out);
          bulk_commit();
        }
        prev_ws = ws;
      } else {
        mbar_wait(&t_full[ds], dph);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&t_empty[ds]);
        if (C::kOutBuf ? lane_id() == 0 : storer) mbar_arrive(&w_empty[ws]);
      }
      if (do_gx && (it + 1) % gx_win == 0 && it + 1 < ntl) {
        // drain a complete accumulation window; the MMA warp restarts the
        // accumulator after every epilogue warp has read its part
        const int w = it / gx_win;
        mbar_wait(gxw_full, static_cast<uint32_t>(w) & 1u);
        tc_fence_after();
        gx_drain(w > 0 || p.gx_accumulate != 0);
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(gxw_empty);
      }
      if (++ws == WS) { ws = 0; wph ^= 1; }
      if (++ds == 2) { ds = 0; dph ^= 1; }
    }
    if (!FAST && storer && p.do_update) {
      bulk_wait<0>();
      if (!C::kOutBuf && prev_ws >= 0) mbar_arrive(&w_empty[prev_ws]);
    }
    if (do_gx) {
      mbar_wait(gx_full, 0);
      tc_fence_after();
      gx_drain(ntl > gx_win || p.gx_accumulate != 0);
    }
  }

  tc_fence_before();
  __syncthreads();
  ClkSpan::end(1);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace xmc
