// Kernel 1 of a head chunk: logits S = W_c . Xq^T on tcgen05 (TMEM accumulator),
// fused epilogue G = clip(sigmoid(S), 2^-24, 1-2^-24) - Y (positives from the
// per-tile label-bucketed list), written once to the chunk's G buffer in the
// backward operand format.  Reference: head_forward_logits head.py:164-178 and
// logit_gradient head.py:181-196 (also the plain-logits mode used by
// ChunkedHead.scores head.py:109-112).
//
// Warp roles (persistent, one CTA per SM):
//   warp 0      TMA producer  (W k-chunk + Xq k-chunk per stage)
//   warp 1      MMA issuer    (one elected lane), owns the TMEM allocation
//   warps 2..   epilogue      (2 or 4 warps per TMEM sub-partition)
//
// PAIR = true: CTA pairs (cluster of 2, tcgen05 cta_group::2).  The pair
// computes M = 256 labels (128 per CTA) x N = B with ONE MMA stream issued by
// the leader; each CTA stages only its half of Xq (N/2 samples) and its own
// 128 W rows, so Xq traffic from L2 and shared-memory traffic per label halve.
// TMA completions of both CTAs land on the leader's full barrier; the
// leader's commits multicast to both CTAs' empty / tmem-full barriers; the
// peer's epilogue releases the accumulator on the leader's barrier.
//
// G output formats (template GOUT, mode 0):
//   G_OPERAND  e4m3 head: e4m3(256 g); bf16 head: bf16(g).  sigmoid =
//              1 / (1 + 2^(-z log2 e)): ex2 on MUFU; for e4m3 the 2^8 scale is
//              folded into the reciprocal, which runs on the FMA pipe (magic
//              seed + 3 Newton steps, rel. err < 2^-20), and the clip is
//              dropped because both clip edges round to the same e4m3 code.
//   G_E5M2     e4m3 head: e5m2(256 g) -- same scale, range down to the
//              reference's 2^-24 clip (e5m2 subnormals reach 2^-16 = 2^8 * 2^-24),
//              so trained heads' small sigmoids do not flush to zero.
//   G_REF      reference precision: g exactly as logit_gradient computes it
//              (IEEE expf, fp32 add and divide, clip, fp32 "-1" at positives),
//              split EXACTLY into three bf16 planes hi + mid + lo = g, written
//              as [hi | mid | lo] (row stride 3 Bp).  The backward consumes the
//              planes as a 3x longer K (bf16 x bf16 products are exact), so it
//              multiplies by the fp32 G of the reference (head.py:193-208, 236).
//              With g_planes = 1 only hi = bf16(g) is written.
//   G_BF16     e4m3 head, bf16(g) computed as a bf16 head computes it (fast
//              sigmoid, clip): the bf16-G operand mode (the paper's FP8
//              weights with BF16 logit gradients).
#pragma once

#include "xmc_ptx.cuh"
#include "xmc_round.cuh"

namespace xmc {

enum GOut : int { G_OPERAND = 0, G_E5M2 = 1, G_REF = 2, G_BF16 = 3 };

struct FwdParams {
  int32_t rows;        // labels in this chunk
  int32_t B;           // valid samples
  int32_t d;           // feature dim (multiple of 128 B / elem)
  int32_t num_tiles;   // ceil(rows / 128)
  int32_t mode;        // 0: write G; 1: write fp32 logits; 2: top-k (TOPK instantiation)
  const int32_t* tile_ptr;   // [num_tiles + 1] into entries (chunk-local tiles)
  const uint32_t* entries;   // (row_in_tile << 16) | sample
  void* out;                 // G [rows][ld] or logits fp32 [rows][ld]
  int64_t ld;                // leading dimension (elements) of out
  int64_t plane_ld;          // G_REF: elements between the hi / mid / lo planes of a row
  int32_t g_planes;          // G_REF: 3 (hi | mid | lo, reference precision) or 1 (hi = bf16(g) only)
  int32_t w_keep_units;      // training forward: the last units of each CTA load W with evict_last (the
                             // backward walks the tiles in reverse, so it finds them, and their G, in L2)
  float* stats;              // [0] += sum |G| over valid entries (optional)
  float logit_scale;         // z = logit_scale * acc (1, or 1/(1-p) under keyed dropout)
  // top-k scoring (TOPK instantiation): per (sample, CTA, sub-partition) the
  // kTopK best (score, global label) of that warp's rows, [Bp][nslots][kTopK]
  float* cand_s;
  int32_t* cand_l;
  int32_t unit_mul;          // TOPK prologue: only every unit_mul-th work unit (a strided label sample)
  const float* topk_bound;   // TOPK: [B][8] top-8 scores of that sample (slot 7 <= the final 8th), or null
  int32_t topk_max_only;     // TOPK prologue: each lane list keeps only the maximum score of its labels
  int64_t label0;            // global label of local row 0 of this launch
  int32_t* status;           // nonzero abort bits -> no-op; NaN logits latch ST 4
  int32_t sample0;           // first sample of this pass (batch split into BN-wide passes); entries of
                             // other samples are skipped, this pass's are shifted by -sample0
};

// XRES (CTA pairs only): this CTA's Xq rows stay resident in shared memory
// for the whole launch (loaded once, kXResChunks K-chunks max, i.e. d <= 768
// for e4m3), so a stage carries only its W box: half the TMA work and L2->SM
// traffic per tile.
template <int EB, int BN, bool PAIR, bool XRES = false>
struct FwdCfg {
  static_assert(!XRES || PAIR, "resident Xq runs on CTA pairs");
  static constexpr int kBoxK = 128 / EB;                  // K elements per 128-B swizzle atom
  static constexpr int kWBytes = 128 * 128;               // W box: 128 rows x 128 B
  static constexpr int kXRows = PAIR ? BN / 2 : BN;       // Xq rows staged by this CTA
  static constexpr int kXBoxRows = kXRows > 256 ? 256 : kXRows;
  static constexpr int kXBoxes = kXRows / kXBoxRows;
  static constexpr int kXBytes = kXRows * 128;
  static constexpr int kXResChunks = 6;
  static constexpr int kXResBytes = XRES ? kXResChunks * kXBytes : 0;
  static constexpr int kStageBytes = kWBytes + (XRES ? 0 : kXBytes);
  static constexpr int kStages = XRES ? 7 : ((200 * 1024) / kStageBytes > 6 ? 6 : (200 * 1024) / kStageBytes);
  static constexpr int kAccStages = (2 * BN <= 512) ? 2 : 1;
  static constexpr int kTmemCols = (BN * kAccStages) <= 128 ? 128 : ((BN * kAccStages) <= 256 ? 256 : 512);
  static constexpr int kWordsPerRow = BN / 32;
  static constexpr int kBitmapBytes = 128 * kWordsPerRow * 4;
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kXResBytes + kStages * kStageBytes + kBitmapBytes + 256;
  static constexpr int kMmaN = BN > 256 ? 256 : BN;
  // epilogue: 4 warps per TMEM sub-partition for wide tiles, 2 otherwise
  static constexpr int kEpiWarps = (BN >= 256 || XRES) ? 16 : 8;
  static constexpr int kThreads = 64 + kEpiWarps * 32;
  static constexpr int kColsPerWarp = BN / (kEpiWarps / 4);
  static constexpr int kChunks = kColsPerWarp / 32;
};

constexpr int kTopK = 8;   // candidates kept per (sample, warp list); user k <= kTopK

// (v, lv) ranks before (s, ls): higher score, ties toward the lower label
// (metrics.py:38-47 stable descending order)
XMC_DEV bool topk_better(float v, int32_t lv, float s, int32_t ls) { return v > s || (v == s && lv < ls); }

// insert into a descending list (registers, fully unrolled)
XMC_DEV void topk_insert(float (&s)[kTopK], int32_t (&l)[kTopK], float v, int32_t lv) {
  if (!topk_better(v, lv, s[kTopK - 1], l[kTopK - 1])) return;
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    if (topk_better(v, lv, s[i], l[i])) {
      const float ts = s[i];
      const int32_t tl = l[i];
      s[i] = v;
      l[i] = lv;
      v = ts;
      lv = tl;
    }
  }
}

// logit_gradient's sigmoid (head.py:193-195) in the reference's fp32 ops:
// clip(1 / (1 + exp(-z)), 2^-24, 1 - 2^-24) with IEEE expf / add / divide
XMC_DEV float ref_sigmoid_clip(float z) {
  float g = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
  g = g < 5.9604644775390625e-08f ? 5.9604644775390625e-08f : g;   // NaN propagates like np.clip
  return g > 0.99999994039535522461f ? 0.99999994039535522461f : g;
}

// The kernel body: work units unit0, unit0 + ustride, ... (tiles, or tile
// pairs for PAIR).
template <int EB, int BN, bool PAIR, bool TOPK, bool XRES, int GOUT>
XMC_DEV void fwd_body(const CUtensorMap& tm_w, const CUtensorMap& tm_x, const FwdParams p, const int unit0,
                      const int ustride) {
  using C = FwdCfg<EB, BN, PAIR, XRES>;
  static_assert(!PAIR || BN <= 256, "paired tiles use one N <= 256 accumulator");
  static_assert(GOUT != G_E5M2 || EB == 1, "e5m2 G is the e4m3 head's wide-range operand");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xres = smem;                           // [kXResChunks][kXRows x 128 B] (XRES)
  uint8_t* stage_base = smem + C::kXResBytes;
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(stage_base + C::kStages * C::kStageBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage_base + C::kStages * C::kStageBytes + C::kBitmapBytes);
  uint64_t* full = bars;                          // [kStages]   (leader's counts both CTAs)
  uint64_t* empty = bars + C::kStages;            // [kStages]
  uint64_t* tfull = bars + 2 * C::kStages;        // [kAccStages]
  uint64_t* tempty = tfull + C::kAccStages;       // [kAccStages] (leader's counts both CTAs)
  uint64_t* xfull = tempty + C::kAccStages;       // resident Xq landed (leader's counts both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + 1);
  int32_t* status_s = reinterpret_cast<int32_t*>(tmem_slot + 1);

  const uint32_t warp = warp_id_sync();
  const int kc_count = (p.d + C::kBoxK - 1) / C::kBoxK;   // a partial last K-chunk is zero-filled by TMA
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  // work units: single tiles, or tile pairs (2u, 2u+1) for a CTA pair
  // (unit_mul > 1: the top-k prologue visits units 0, unit_mul, 2 unit_mul, ...)
  const int umul = p.unit_mul > 1 ? p.unit_mul : 1;
  const int num_units = ((PAIR ? (p.num_tiles + 1) / 2 : p.num_tiles) + umul - 1) / umul;
  // Xq rows (samples) this CTA stages
  const int xrow0 = PAIR ? static_cast<int>(rank) * C::kXRows : 0;

  if (warp == 0 && elect_one()) {
    prefetch_tmap(&tm_w);
    prefetch_tmap(&tm_x);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], PAIR ? 2 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::kAccStages; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (PAIR ? 2 : 1) * C::kEpiWarps);
    }
    mbar_init(xfull, PAIR ? 2 : 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_2sm<C::kTmemCols>(tmem_slot);
    else tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  // PDL: the prologue above (barriers, TMEM, tensor maps) overlapped the
  // previous kernel's tail; from here on its outputs are read
  griddep_wait();
  griddep_launch_dependents();
  ClkSpan::begin(0);
  // A latched error of an earlier kernel of the step turns this one into a
  // no-op.  The status word is read ONCE (by the pair leader) and every warp of
  // both CTAs takes that value: the kernel itself may latch an error later, and
  // roles of one pair must never disagree about skipping (they would hang on
  // each other's barriers).
  if (threadIdx.x == 0 && leader) *status_s = *p.status;
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // (shuffled from lane 0: provably warp-uniform, which keeps the role code
  // below on the uniform datapath)
  int32_t st_word;
  if constexpr (PAIR) st_word = ld_shared_cluster_s32(mapa_shared(status_s, 0));
  else st_word = *status_s;
  const bool aborted = __shfl_sync(0xffffffffu, st_word, 0) != 0;

  if (aborted) {
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    // A bulk-tensor copy instruction occupies its warp for ~max(585, 1.8 x
    // 128-B lines of ALL its lanes) cycles (tools/probe_tma.cu), so one box
    // per instruction caps a CTA at ~28 B/clk.  The producer therefore issues
    // the boxes of kIPB consecutive stages as ONE warp-wide instruction, lane
    // l carrying box l (W or an Xq box of one stage).
    constexpr int kBPI = 1 + (XRES ? 0 : (PAIR ? 1 : C::kXBoxes));   // boxes per stage
    constexpr int kIPB = XRES ? 3 : 2;                                 // stages per instruction
    static_assert(kBPI * kIPB <= 32, "one lane per box");
    const int lane = static_cast<int>(lane_id());
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();   // (also W of the last w_keep_units units)
    if constexpr (XRES) {
      // this CTA's Xq rows, every K-chunk, once: one warp-wide instruction
      if (lane == 0) {
        if (leader) mbar_arrive_expect_tx(xfull, 2 * kc_count * C::kXBytes);
        else mbar_arrive_cluster(mapa_shared(xfull, 0));
      }
      __syncwarp();
      if (lane < kc_count)
        tma_load_2d_2sm(xres + lane * C::kXBytes, &tm_x, mapa_shared(xfull, 0), lane * C::kBoxK, xrow0, pol_x);
      __syncwarp();
    }
    const int my_units = unit0 < num_units ? (num_units - unit0 + ustride - 1) / ustride : 0;
    const int total = my_units * kc_count;   // stages this CTA fills
    for (int n0 = 0; n0 < total; n0 += kIPB) {
      const int cnt = min(kIPB, total - n0);
      // stage / phase of item n: ring position n mod kStages, lap n / kStages
      for (int i = 0; i < cnt; ++i) {
        const int n = n0 + i;
        mbar_wait(&empty[n % C::kStages], ((n / C::kStages) & 1) ^ 1);
      }
      const int it = lane / kBPI, b = lane % kBPI;
      const int n = n0 + it;
      const int st_i = n % C::kStages;
      const int u = unit0 + (n / kc_count) * ustride;
      const int kc = n % kc_count;
      const int tile = PAIR ? 2 * u * umul + static_cast<int>(rank) : u * umul;
      uint8_t* sb = stage_base + st_i * C::kStageBytes;
      const bool active = it < cnt;
      if (active && b == 0) {
        if constexpr (PAIR) {
          if (leader) mbar_arrive_expect_tx(&full[st_i], 2 * C::kStageBytes);
          else mbar_arrive_cluster(mapa_shared(&full[st_i], 0));
        } else {
          mbar_arrive_expect_tx(&full[st_i], C::kStageBytes);
        }
      }
      __syncwarp();
      const CUtensorMap* m = b == 0 ? &tm_w : &tm_x;
      uint8_t* dst = b == 0 ? sb : sb + C::kWBytes + (b - 1) * C::kXBoxRows * 128;
      const int32_t c1 = b == 0 ? tile * 128 : xrow0 + (b - 1) * C::kXBoxRows;
      const uint64_t pol = (b == 0 && n / kc_count < my_units - p.w_keep_units) ? pol_w : pol_x;
      if (active) {
        if constexpr (PAIR) tma_load_2d_2sm(dst, m, mapa_shared(&full[st_i], 0), kc * C::kBoxK, c1, pol);
        else tma_load_2d_hint(dst, m, &full[st_i], kc * C::kBoxK, c1, pol);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (leader) {
      constexpr uint32_t kM = PAIR ? 256 : 128;
      constexpr uint32_t idesc = (EB == 1) ? umma_idesc(0, 0, false, false, kM, C::kMmaN)
                                           : umma_idesc(1, 1, false, false, kM, C::kMmaN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      if constexpr (XRES) mbar_wait(xfull, 0);
      for (int u = unit0; u < num_units; u += ustride) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kc = 0; kc < kc_count; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(stage_base + stage * C::kStageBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = umma_desc_sw128(sa + k * 32, 16, 1024);
#pragma unroll
              for (int xb = 0; xb < (PAIR ? 1 : C::kXBoxes); ++xb) {
                const uint32_t xa = XRES ? smem_u32(xres + kc * C::kXBytes) : sa + C::kWBytes;
                const uint64_t bd = umma_desc_sw128(xa + xb * C::kXBoxRows * 128 + k * 32, 16, 1024);
                if constexpr (PAIR) {
                  if constexpr (EB == 1) mma_f8_2sm(d_tmem, ad, bd, idesc, (kc | k) != 0);
                  else mma_f16_2sm(d_tmem, ad, bd, idesc, (kc | k) != 0);
                } else {
                  if constexpr (EB == 1) mma_f8(d_tmem + xb * 256, ad, bd, idesc, (kc | k) != 0);
                  else mma_f16(d_tmem + xb * 256, ad, bd, idesc, (kc | k) != 0);
                }
              }
            }
            if constexpr (PAIR) {
              mma_commit_2sm_mc(&empty[stage], 0x3);
              if (kc == kc_count - 1) mma_commit_2sm_mc(&tfull[acc], 0x3);
            } else {
              mma_commit(&empty[stage]);
              if (kc == kc_count - 1) mma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        if (++acc == C::kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else if constexpr (TOPK) {
    // --------------------------------------------- streaming top-k epilogue
    // ChunkedHead.scores (head.py:109-112) + top_k_indices (metrics.py:38-47)
    // without materialising scores.  Per 32x32 block (32 rows of this warp's
    // sub-partition x 32 samples) a register transpose across the warp gives
    // lane c the 32 scores of sample col0 + c; each lane keeps a sorted
    // register list of the kTopK best (score, label) of its sample over every
    // row this warp sees.  Rows arrive in increasing label order, so strict
    // ">" keeps the reference's stable tie order (lower label first).
    const int ew = warp - 2;
    const int q = warp & 3;
    const int grp = ew >> 2;
    const int lane = lane_id();
    float ls[C::kChunks][kTopK];
    int32_t ll[C::kChunks][kTopK];
#pragma unroll
    for (int cc = 0; cc < C::kChunks; ++cc)
#pragma unroll
      for (int i = 0; i < kTopK; ++i) {
        ls[cc][i] = -INFINITY;
        ll[cc][i] = 0x7fffffff;
      }
    // Pre-filter without the transpose.  Each lane's sample threshold (its
    // list's k-th score, raised to just below the prologue's bound) is
    // mirrored in shared memory (the positives bitmap region, unused here:
    // 16 x BN bytes = warps x chunks x 32 floats), so a 32 x 32 block whose
    // scores are all <= the thresholds costs 8 broadcast LDS.128 and 32
    // compares instead of the 5-stage shuffle transpose.  Blocks with a
    // candidate take the exact transpose + insert path (same strict ">").
    // The bound: the prologue's 8th score over a strided label sample is <=
    // the final 8th score, so an item under it cannot reach the top-k; one
    // EQUAL to it still can (lower-label tie rule), hence nextafter(-inf).
    float* th_s = reinterpret_cast<float*>(bitmap) + ew * C::kChunks * 32;
#pragma unroll
    for (int cc = 0; cc < C::kChunks; ++cc) {
      const int sc = grp * C::kColsPerWarp + cc * 32 + lane;
      float t0 = INFINITY;
      if (sc < p.B) t0 = p.topk_bound ? nextafterf(p.topk_bound[sc * kTopK + kTopK - 1], -INFINITY) : -INFINITY;
      th_s[cc * 32 + lane] = t0;
    }
    __syncwarp();
    auto tile_of = [&](int u) { return PAIR ? 2 * u * umul + static_cast<int>(rank) : u * umul; };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = unit0; u < num_units; u += ustride) {
      const int tile = tile_of(u);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t r0w = static_cast<int64_t>(tile) * 128 + q * 32;   // first row of this warp
      const int64_t left = static_cast<int64_t>(p.rows) - r0w;
      const int vrows = left >= 32 ? 32 : (left <= 0 ? 0 : static_cast<int>(left));
      const uint32_t rowmask = vrows >= 32 ? 0xffffffffu : ((1u << vrows) - 1u);
      const int32_t lab0 = static_cast<int32_t>(p.label0 + r0w);
#pragma unroll
      for (int cc = 0; cc < C::kChunks; ++cc) {
        const int col0 = grp * C::kColsPerWarp + cc * 32;
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + col0, r);
        tmem_ld_wait();
        if (p.topk_max_only) {
          // prologue: only a lower bound is needed.  The maxima of disjoint
          // label groups are distinct scores, so the 8th largest of them
          // cannot exceed the final 8th score.  Column max over the warp's
          // 32 rows by a reduce-scatter butterfly (lane c ends with sample
          // col0 + c): 31 shuffles instead of the 80 of the transpose.
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = lane < vrows ? __uint_as_float(r[i]) : -INFINITY;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < o; ++i) {
              const float recv = __shfl_xor_sync(0xffffffffu, up ? v[i] : v[i + o], o);
              v[i] = fmaxf(up ? v[i + o] : v[i], recv);
            }
          }
          ls[cc][0] = fmaxf(ls[cc][0], v[0]);
          continue;
        }
        {
          // lane = row here: r[c] = score(row, sample col0 + c)
          bool cand = false;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 t = *reinterpret_cast<const float4*>(th_s + cc * 32 + 4 * c4);
            cand |= __uint_as_float(r[4 * c4 + 0]) > t.x;
            cand |= __uint_as_float(r[4 * c4 + 1]) > t.y;
            cand |= __uint_as_float(r[4 * c4 + 2]) > t.z;
            cand |= __uint_as_float(r[4 * c4 + 3]) > t.w;
          }
          if (!__any_sync(0xffffffffu, cand && lane < vrows)) continue;
        }
        // butterfly transpose: afterwards r[i] of lane c = score(row i, sample col0 + c)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (i & o) continue;
            const uint32_t a = r[i], b = r[i | o];
            const uint32_t recv = __shfl_xor_sync(0xffffffffu, up ? a : b, o);
            r[i] = up ? recv : a;
            r[i | o] = up ? b : recv;
          }
        }
        const float th = th_s[cc * 32 + lane];
        uint32_t pm = 0u;
#pragma unroll
        for (int i = 0; i < 32; ++i) pm |= (__uint_as_float(r[i]) > th ? 1u : 0u) << i;
        pm &= rowmask;
        if (col0 + lane >= p.B) pm = 0u;
        if (__any_sync(0xffffffffu, pm != 0u)) {   // rare once the lists are warm
          float rv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) rv[i] = __uint_as_float(r[i]);
#pragma unroll 1
          while (pm) {
            const int i = __ffs(pm) - 1;
            pm &= pm - 1;
            topk_insert(ls[cc], ll[cc], rv[i], lab0 + i);
          }
        }
        if (col0 + lane < p.B) th_s[cc * 32 + lane] = fmaxf(th, ls[cc][kTopK - 1]);
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && !leader) mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == C::kAccStages) { acc = 0; acc_phase ^= 1; }
    }
    const int nslots = gridDim.x * 4;
    const int slot = blockIdx.x * 4 + q;
#pragma unroll
    for (int cc = 0; cc < C::kChunks; ++cc) {
      const int s = grp * C::kColsPerWarp + cc * 32 + lane;
      if (s < p.B) {
        const size_t o = (static_cast<size_t>(s) * nslots + slot) * kTopK;
#pragma unroll
        for (int i = 0; i < kTopK; ++i) {
          p.cand_s[o + i] = ls[cc][i];
          p.cand_l[o + i] = ll[cc][i];
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    constexpr int NT = C::kEpiWarps * 32;
    const int ew = warp - 2;                 // 0 .. kEpiWarps-1
    const int q = warp & 3;                  // TMEM sub-partition of this warp
    const int grp = ew >> 2;                 // which column group of the tile
    const int row = q * 32 + lane_id();      // row within the 128-label tile
    const int etid = ew * 32 + lane_id();
    const bool want_stats = p.stats != nullptr && p.mode == 0;
    const int s0 = p.sample0;                    // first sample (positive entries)
    const int bvalid = p.B;                      // valid columns
    const bool pad_cols = bvalid < BN;
    const bool use_pos = p.mode == 0 && p.tile_ptr != nullptr;
    const uint64_t pol_g = policy_evict_last();   // G is re-read by the backward kernel
    float abs_sum = 0.f;
    bool nan_seen = false;
    const float zk = -1.4426950408889634f * p.logit_scale;   // -log2(e) * scale
    // operand G of an e4m3 head carries the 2^8 scale (e4m3 / e5m2 encodings)
    // FP8 G (2^8-scaled e4m3 / e5m2) of an e4m3 head; G_BF16 computes and
    // stores G exactly as a bf16 head does (unscaled, clipped, bf16)
    constexpr bool kScaled = EB == 1 && GOUT != G_REF && GOUT != G_BF16;
    int acc = 0;
    uint32_t acc_phase = 0;
    auto tile_of = [&](int u) { return PAIR ? 2 * u * umul + static_cast<int>(rank) : u * umul; };
    // tile_ptr bounds of the first tile; the next tile's are prefetched below
    int e0 = 0, e1 = 0;
    if (use_pos && unit0 < num_units && tile_of(unit0) < p.num_tiles) {
      e0 = p.tile_ptr[tile_of(unit0)];
      e1 = p.tile_ptr[tile_of(unit0) + 1];
    }
    for (int u = unit0; u < num_units; u += ustride) {
      const int tile = tile_of(u);
      int n0 = 0, n1 = 0;
      const int nt = tile_of(u + ustride);
      if (use_pos && u + ustride < num_units && nt < p.num_tiles) {
        n0 = p.tile_ptr[nt];
        n1 = p.tile_ptr[nt + 1];
      }
      // positives of this tile -> bitmap, only when the tile has any (uniform)
      const bool has_pos = e1 > e0;
      if (has_pos) {
        named_bar_sync(1, NT);   // previous users of the bitmap are done
        for (int w = etid; w < 128 * C::kWordsPerRow; w += NT) bitmap[w] = 0u;
        named_bar_sync(1, NT);
        for (int e = e0 + etid; e < e1; e += NT) {
          const uint32_t v = p.entries[e];
          const uint32_t r = v >> 16, s = (v & 0xFFFFu) - static_cast<uint32_t>(s0);
          if (s < static_cast<uint32_t>(BN)) atomicOr(&bitmap[r * C::kWordsPerRow + (s >> 5)], 1u << (s & 31));
        }
        named_bar_sync(1, NT);
      }
      e0 = n0;
      e1 = n1;

      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t grow = static_cast<int64_t>(tile) * 128 + row;
      const bool row_ok = grow < p.rows;
#pragma unroll 1
      for (int cc = 0; cc < C::kChunks; ++cc) {
        const int col0 = grp * C::kColsPerWarp + cc * 32;
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + col0, r);
        tmem_ld_wait();
        if (p.mode == 1) {
          if (row_ok) {
            float* o = reinterpret_cast<float*>(p.out) + grow * p.ld;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < bvalid) o[col0 + j] = __uint_as_float(r[j]) * p.logit_scale;
          }
          continue;
        }
        const uint32_t pos = has_pos ? bitmap[row * C::kWordsPerRow + (col0 >> 5)] : 0u;
        float g[32];
        if constexpr (GOUT == G_REF) {
          // the reference's fp32 sigmoid; positives get the fp32 "-1" (head.py:196)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float z = __uint_as_float(r[j]) * p.logit_scale;
            nan_seen |= (z != z);
            g[j] = ref_sigmoid_clip(z);
            if ((pos >> j) & 1u) g[j] = __fsub_rn(g[j], 1.0f);
          }
        } else if constexpr (kScaled) {
          // g256 = 256 sigmoid(z) = 1 / y, y = 2^-8 (1 + 2^(-z log2 e))
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float za, zb;
            f2unpack(fmul2(f2pack(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), f2pack(zk, zk)), za, zb);
            // e clamped to 2^100 keeps y finite (g then rounds to 0 in e4m3).
            // e5m2 needs no clamp: an infinite / huge e makes the Newton
            // iterate NaN or -inf, and the 2^-16 clip below (fmaxf returns
            // the non-NaN operand) yields exactly the clipped value 256 * 2^-24
            // that sigmoid(z) < 2^-100 has in the reference
            float ea = fast_ex2(za), eb = fast_ex2(zb);
            if constexpr (GOUT != G_E5M2) {
              ea = fminf(ea, 1.2676506e30f);
              eb = fminf(eb, 1.2676506e30f);
            }
            const uint64_t y = ffma2(f2pack(ea, eb), f2pack(0.00390625f, 0.00390625f),
                                     f2pack(0.00390625f, 0.00390625f));
            float y0, y1;
            f2unpack(y, y0, y1);
            uint64_t x = f2pack(__uint_as_float(0x7EF311C3u - __float_as_uint(y0)),
                                __uint_as_float(0x7EF311C3u - __float_as_uint(y1)));
            const uint64_t two = f2pack(2.0f, 2.0f);
            const uint64_t ny = f2pack(-y0, -y1);
#pragma unroll
            for (int it = 0; it < 3; ++it) x = fmul2(x, ffma2(ny, x, two));   // x (2 - y x)
            f2unpack(x, g[j], g[j + 1]);
          }
          if constexpr (GOUT == G_E5M2) {
            // the 2^-24 clip (head.py:47-48) is representable in e5m2 x 2^8
            // (2^-16, its smallest subnormal): keep it
#pragma unroll
            for (int j = 0; j < 32; ++j) g[j] = fmaxf(g[j], 1.52587890625e-05f);
          }
        } else {
          const float SIG_LO = 5.9604644775390625e-08f;   // 2^-24  (head.py:47-48)
          const float SIG_HI = 0.99999994039535522461f;   // 1 - 2^-24
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float z = __uint_as_float(r[j]);
            nan_seen |= (z != z);
            float sg = fast_rcp(1.0f + fast_ex2(z * zk));
            sg = sg < SIG_LO ? SIG_LO : sg;   // NaN propagates like np.clip
            g[j] = sg > SIG_HI ? SIG_HI : sg;
          }
        }
        if constexpr (GOUT != G_REF) {
          const float one = kScaled ? 256.0f : 1.0f;
          if (pos != 0u) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((pos >> j) & 1u) g[j] -= one;
          }
        }
        if (pad_cols) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j >= bvalid) g[j] = 0.0f;
        }
        if (want_stats && row_ok) {
#pragma unroll
          for (int j = 0; j < 32; ++j) abs_sum += fabsf(g[j]);
        }
        if (row_ok) {
          if constexpr (GOUT == G_REF) {
            // g = hi + mid + lo exactly: hi = bf16(g), mid = bf16(g - hi),
            // lo = bf16(g - hi - mid) (each residual is exact in fp32 and the
            // last one has <= 8 significant bits)
            uint32_t ph[16], pm[16], pl[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              ph[j] = cvt_bf16x2_rn(g[2 * j + 1], g[2 * j]);
              const float r0 = g[2 * j] - __uint_as_float(ph[j] << 16);
              const float r1 = g[2 * j + 1] - __uint_as_float(ph[j] & 0xFFFF0000u);
              pm[j] = cvt_bf16x2_rn(r1, r0);
              const float t0 = r0 - __uint_as_float(pm[j] << 16);
              const float t1 = r1 - __uint_as_float(pm[j] & 0xFFFF0000u);
              pl[j] = cvt_bf16x2_rn(t1, t0);
            }
            uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + grow * p.ld + col0;
            auto store_plane = [&](uint16_t* dst, const uint32_t (&v)[16]) {
              st_global_v8_hint(dst, *reinterpret_cast<const uint32_t(*)[8]>(&v[0]), pol_g);
              st_global_v8_hint(dst + 16, *reinterpret_cast<const uint32_t(*)[8]>(&v[8]), pol_g);
            };
            store_plane(o, ph);
            if (p.g_planes > 1) {
              store_plane(o + p.plane_ld, pm);
              store_plane(o + 2 * p.plane_ld, pl);
            }
          } else if constexpr (kScaled) {
            uint32_t pk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t lo = GOUT == G_E5M2 ? cvt_e5m2x2_rn(g[4 * j + 1], g[4 * j + 0])
                                                 : cvt_e4m3x2_rn(g[4 * j + 1], g[4 * j + 0]);
              const uint32_t hi = GOUT == G_E5M2 ? cvt_e5m2x2_rn(g[4 * j + 3], g[4 * j + 2])
                                                 : cvt_e4m3x2_rn(g[4 * j + 3], g[4 * j + 2]);
              pk[j] = lo | (hi << 16);
            }
            // one 256-bit store: the thread's 32 G bytes are one full sector
            st_global_v8_hint(reinterpret_cast<uint8_t*>(p.out) + grow * p.ld + col0, pk, pol_g);
          } else {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = cvt_bf16x2_rn(g[2 * j + 1], g[2 * j]);
            uint16_t* o = reinterpret_cast<uint16_t*>(p.out) + grow * p.ld + col0;
            const uint32_t (&pa)[8] = *reinterpret_cast<const uint32_t(*)[8]>(&pk[0]);
            const uint32_t (&pb)[8] = *reinterpret_cast<const uint32_t(*)[8]>(&pk[8]);
            st_global_v8_hint(o, pa, pol_g);        // two full 32-B sectors
            st_global_v8_hint(o + 16, pb, pol_g);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {
        if (PAIR && !leader) mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == C::kAccStages) { acc = 0; acc_phase ^= 1; }
    }
    if (want_stats) {
      abs_sum *= kScaled ? 0.00390625f : 1.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) abs_sum += __shfl_xor_sync(0xffffffffu, abs_sum, o);
      if (lane_id() == 0) atomicAdd(p.stats, abs_sum);
    }
    if (__any_sync(0xffffffffu, nan_seen) && lane_id() == 0) atomicOr(p.status, 4 /*ST_NONFINITE_GRAD*/);
  }

  tc_fence_before();
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  ClkSpan::end(0);
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_2sm<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <int EB, int BN, bool PAIR, bool TOPK = false, bool XRES = false, int GOUT = G_OPERAND>
__global__ void __launch_bounds__(FwdCfg<EB, BN, PAIR, XRES>::kThreads, 1)
    xmc_fwd_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                   const FwdParams p) {
  if constexpr (PAIR) {
    fwd_body<EB, BN, PAIR, TOPK, XRES, GOUT>(tm_w, tm_x, p, static_cast<int>(cluster_id_x()),
                                             static_cast<int>(num_clusters_x()));
  } else {
    fwd_body<EB, BN, PAIR, TOPK, XRES, GOUT>(tm_w, tm_x, p, static_cast<int>(blockIdx.x),
                                             static_cast<int>(gridDim.x));
  }
}

}  // namespace xmc
