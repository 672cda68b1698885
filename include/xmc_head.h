/*
 * xmc_head.h -- C ABI of the B200-native ELMO extreme-classification head.
 *
 * Drop-in boundary for the reference's hot path (lpxmc, pure Python/numpy):
 * every entry point below replaces one reference function, cited as
 * /root/reference/pkg/src/lpxmc/<file>:<line>.  Plain pointers and sizes only;
 * device pointers are CUDA global-memory addresses, `stream` is a cudaStream_t.
 * The library never frees caller memory; the caller (the Python host module,
 * via torch) owns W, X, positives, outputs and the workspace.
 *
 * Error convention (mirrors the reference's exceptions, head.py / formats.py /
 * optimizers.py): every call returns an xmc_status; xmc_last_error() gives a
 * message.  Device-detected errors (non-finite input/gradient, sample index
 * out of range) are latched in the handle's status word: every later kernel
 * (of this step and of later steps) becomes a no-op that leaves W untouched,
 * and grad_X comes back as NaN, until xmc_head_check() reports the error and
 * clears the latch.
 */
#ifndef XMC_HEAD_H_
#define XMC_HEAD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  XMC_OK = 0,
  XMC_ERR_ARG = 1,         /* ValueError: bad config / argument     */
  XMC_ERR_SHAPE = 2,       /* ValueError: dimension mismatch        */
  XMC_ERR_NONFINITE = 3,   /* ValueError: non-finite input/gradient */
  XMC_ERR_INDEX = 4,       /* IndexError: sample index out of range */
  XMC_ERR_LABEL = 5,       /* ValueError: label outside chunk range */
  XMC_ERR_CUDA = 6,        /* RuntimeError: CUDA failure            */
  XMC_ERR_UNSUPPORTED = 7, /* NotImplementedError                   */
  XMC_ERR_CAPACITY = 8     /* workspace too small for this call     */
} xmc_status;

/* Storage / grid formats (formats.py:139-143).  Native storage: fp32 = 4 B,
 * bf16 = 2 B (torch.bfloat16 bits), e4m3 = 1 B (float8_e4m3fn bits, identical
 * to encode_grid_bits, head.py:317-338), e5m2 = 1 B. */
typedef enum { XMC_FMT_FP32 = 0, XMC_FMT_BF16 = 1, XMC_FMT_FP16 = 2, XMC_FMT_E4M3 = 3, XMC_FMT_E5M2 = 4 } xmc_fmt;

/* SgdSrConfig.rounding (optimizers.py:28-41).  SR_EXACT draws u from the
 * reference's splitmix64 keyed generator (rng.py:36-57) and compares in fp64
 * exactly like round_stochastic (formats.py:209-225): bit-identical decisions.
 * SR_FAST feeds keyed random words to the hardware cvt.rs conversion: by
 * default a stateless keyed hash of the word index (one word per cvt.rs
 * instruction) under the 64-bit key splitmix64(seed, step, tensor_id), or
 * Philox4x32-7 (xmc_step_args.sr_bits = 1). */
typedef enum { XMC_ROUND_NEAREST = 0, XMC_ROUND_SR_EXACT = 1, XMC_ROUND_SR_FAST = 2 } xmc_rounding;

/* Head geometry: ChunkedHead (head.py:69-112) restricted to one rank's label
 * shard [label_offset, label_offset + num_labels_local) of num_labels_global. */
typedef struct {
  int64_t num_labels_global; /* L                                        */
  int64_t label_offset;      /* first global label owned by this rank     */
  int64_t num_labels_local;  /* labels owned by this rank                 */
  int32_t dim;               /* d, a multiple of 32 (partial last 128-column tile is zero-filled) */
  int32_t fmt;               /* xmc_fmt of W: XMC_FMT_E4M3 or XMC_FMT_BF16 */
  int32_t num_chunks;        /* k: chunks = partition(num_labels_local, k) (head.py:51-57) */
  int32_t max_batch;         /* B capacity of the workspace               */
  int64_t max_positives;     /* nnz capacity of the workspace             */
  int32_t num_sms;           /* persistent-grid size (0 = device SM count)*/
  int32_t comp_bytes;        /* Kahan compensation storage: 0 none, 2 bf16, 4 fp32 */
  int32_t dropout;           /* 1: reserve the keyed-dropout scratch (masked W chunk + keep bits),
                                needed for steps with dropout_p > 0 (head.py:138-161) */
  int32_t precision;         /* xmc_precision of the backward GEMMs (see below) */
  int64_t comp_labels;       /* with comp_bytes > 0: only GLOBAL labels < comp_labels carry a
                                compensation (top-p% head-Kahan over frequency-sorted labels,
                                PAPER.md:795); <= 0 = every label.  The comp buffer then holds the
                                shard's rows [0, clamp(comp_labels - label_offset, 0, local)). */
  int32_t g_format;          /* XMC_PRECISION_OPERAND only: the G operand format of an e4m3 head,
                                XMC_FMT_E5M2 (e5m2(2^8 g), the default for 0), XMC_FMT_E4M3
                                (e4m3(2^8 g)) or XMC_FMT_BF16 (bf16(g): FP8 weights with BF16 logit
                                gradients as in the paper; e4m3 W tiles become bf16 operands in
                                shared memory, batch <= 256); ignored for a bf16 head (always bf16(g)) */
  int32_t reserved;
} xmc_head_desc;

/* Precision of G in the two backward GEMMs (dW = G.Xq and grad_X += G^T.W).
 *  XMC_PRECISION_REFERENCE: G exactly as the reference's fp32 logit_gradient
 *    (head.py:181-196, accurate expf / divide), split exactly into three bf16
 *    planes g = hi + mid + lo; the backward runs kind::f16 MMAs over the 3x
 *    longer K, so every product G[l,b] Xq[b,c] and G[l,b] W[l,c] is exact and
 *    only the fp32 accumulation order differs from the reference's sgemm
 *    (head.py:193-208, 236; "update computed at working precision
 *    before the single rounding").  An e4m3 head's W tiles are converted to
 *    bf16 operand tiles in shared memory (exact) and the update still rounds
 *    onto the e4m3 grid.
 *  XMC_PRECISION_OPERAND: G is rounded once to a tensor-core operand format
 *    (desc.g_format): an e4m3 head uses e5m2 or e4m3 of 2^8 g with all three
 *    GEMMs on FP8 kind::f8f6f4 (the production fast path), or bf16(g) with
 *    bf16 operand tiles as for the reference precision (the paper's BF16 logit
 *    gradients); a bf16 head uses bf16(g). */
typedef enum { XMC_PRECISION_OPERAND = 0, XMC_PRECISION_REFERENCE = 1 } xmc_precision;

typedef struct xmc_head* xmc_head_t;

/* Per-step hyper-parameters (SgdSrConfig + RoundingRng + step). */
typedef struct {
  float lr;            /* > 0                                   */
  float weight_decay;  /* >= 0                                  */
  int32_t rounding;    /* xmc_rounding                          */
  int32_t sr_bits;     /* XMC_ROUND_SR_FAST bit source: 0 keyed hash (default), 1 Philox4x32-7 */
  uint64_t seed;       /* RoundingRng(seed)                     */
  uint64_t step;       /* step index keying the draws           */
  uint64_t tensor_id;  /* ChunkedHead.tensor_id (HEAD_WEIGHTS_TAG) */
  double dropout_p;    /* ChunkedHead.dropout_p in [0, 1): keyed weight dropout,
                          keep = u(seed, step, DROPOUT_TAG, r*d + c) >= p (head.py:138-161) */
} xmc_step_args;

const char* xmc_last_error(void);
const char* xmc_version(void);

/* Workspace bytes needed for `desc` (G chunk buffer, Xq/Xq^T, grad_X partials,
 * positive lists, status words). */
xmc_status xmc_head_workspace_size(const xmc_head_desc* desc, size_t* bytes);

/* Bind a handle to a device workspace of >= workspace_size bytes. */
xmc_status xmc_head_create(const xmc_head_desc* desc, void* workspace, size_t workspace_bytes,
                           xmc_head_t* out);
xmc_status xmc_head_destroy(xmc_head_t h);

/* head_update (head.py:254-298): one full step over all chunks of this shard.
 *   W          device, num_labels_local x dim in desc.fmt, updated in place
 *   X          device fp32, B x dim (rounded once to the head grid, head.py:265)
 *   pos_sample / pos_label: device int32 COO of positives, nnz entries, any
 *              order; labels are GLOBAL ids, those outside this shard are
 *              ignored (as the reference ignores labels outside every chunk)
 *   grad_x     device fp32 B x dim: the (shard-partial) input gradient,
 *              overwritten (head.py:266, 290)
 *   stats      device fp32[2] or NULL: [0] = sum |G| of the step, [1] unused
 */
xmc_status xmc_head_step(xmc_head_t h, void* W, const float* X, int32_t B, const int32_t* pos_sample,
                         const int32_t* pos_label, int64_t nnz, const xmc_step_args* args,
                         float* grad_x, float* stats, void* stream);

/* head_update with the head-Kahan extension: kahan_add
 * (formats.py:246-263) composed with the SGD update (optimizers.py:51-74),
 *   v = -lr (g + wd s); y = v - c; s' = ROUND(s + y); c' = (s' - s) - y,
 * with the compensation c stored per weight in `comp` (desc.comp_bytes: bf16
 * as in PAPER.md:795, or fp32 as in the reference's KahanState).  comp NULL
 * == xmc_head_step. */
xmc_status xmc_head_step_kahan(xmc_head_t h, void* W, void* comp, const float* X, int32_t B,
                               const int32_t* pos_sample, const int32_t* pos_label, int64_t nnz,
                               const xmc_step_args* args, float* grad_x, float* stats, void* stream);

/* Adam-style head (north_star: "the SGD or Adam-style update"): the chunk
 * gradient dW of every weight goes through kahan_adamw_step
 * (optimizers.py:112-137) -- fp32 moments m, v and an fp32 Kahan compensation
 * comp, all [L_local][d] -- inside the fused backward epilogue instead of the
 * SGD step.  beta1/beta2 are the config's Python floats (double) and t is the
 * 1-based AdamW step; args supplies seed/step/tensor_id/dropout (lr, wd and
 * rounding are taken from adam).  The handle needs comp_bytes 4 for every
 * label.  Everything else is xmc_head_step. */
typedef struct xmc_adamw_args {
  float lr, weight_decay, eps, reserved;
  double beta1, beta2;
  int64_t t;
} xmc_adamw_args;
xmc_status xmc_head_step_adamw(xmc_head_t h, void* W, float* comp, float* m, float* v, const float* X,
                               int32_t B, const int32_t* pos_sample, const int32_t* pos_label, int64_t nnz,
                               const xmc_adamw_args* adam, const xmc_step_args* args, float* grad_x,
                               float* stats, void* stream);

/* Synchronise `stream` and report a latched device error (and clear it). */
xmc_status xmc_head_check(xmc_head_t h, void* stream);

/* ---- unfused pieces, for parity isolation (same kernels as the step) ---- */

/* head_forward_logits (head.py:164-178): logits[r][s] = sum_c W_eff[row0+r][c] Xq[s][c],
 * for local rows [row0, row1), fp32 out with leading dimension ld (>= B).
 * W_eff = W * keep / (1 - p) when args && args->dropout_p > 0 (seed/step from
 * args; head.py:155-161), else W -- which is also ChunkedHead.scores
 * (head.py:109-112, dropout disabled) transposed.  args may be NULL. */
xmc_status xmc_head_logits(xmc_head_t h, const void* W, const float* X, int32_t B, int64_t row0,
                           int64_t row1, float* logits, int64_t ld, const xmc_step_args* args,
                           void* stream);

/* dropout_mask (head.py:138-152) for global rows [row0, row1) of a matrix with
 * num_cols columns: bit k of keep[(r - row0) * ceil(num_cols / 32) + c / 32]
 * (k = c % 32) = (u >= p), u = RoundingRng(seed).uniform(step, DROPOUT_TAG,
 * r * num_cols + c).  keep is caller device memory. */
xmc_status xmc_dropout_mask(int64_t row0, int64_t row1, int32_t num_cols, uint64_t seed, uint64_t step,
                            double p, uint32_t* keep, void* stream);

/* Streaming top-k scoring: ChunkedHead.scores (head.py:109-112, dropout off)
 * followed by metrics.top_k_indices (metrics.py:38-47) per sample, without
 * materialising the B x L score matrix.  top_scores / top_labels are B x k
 * (row-major), labels GLOBAL (desc.label_offset added), ordered by score
 * descending with ties toward the lower label.  1 <= k <= 8. */
xmc_status xmc_head_topk(xmc_head_t h, const void* W, const float* X, int32_t B, int32_t k,
                         float* top_scores, int64_t* top_labels, void* stream);

/* logit_gradient (head.py:181-196): G = clip(sigmoid(logits)) - Y, elementwise fp32.
 * Labels are chunk-relative GLOBAL ids in [chunk_start, chunk_start + rows). */
xmc_status xmc_logit_gradient(const float* logits, int64_t rows, int32_t B, int64_t ld,
                              const int32_t* pos_sample, const int32_t* pos_label, int64_t nnz,
                              int64_t chunk_start, float* G, void* stream);

/* input_gradient_accumulate (head.py:199-209) and/or fused_weight_update
 * (head.py:212-251) on local rows [row0, row1) from an fp32 G (rows x B, ld):
 * G is converted to the handle's backward operand format (desc.precision:
 * the exact three-plane bf16 split, or the operand rounding) and run through
 * the same tcgen05 kernel as the step.  acc (B x dim fp32) += when
 * accumulate_gx != 0; W updated in place when update != 0. */
xmc_status xmc_head_backward(xmc_head_t h, void* W, const float* G, int64_t ld, const float* X,
                             int32_t B, int64_t row0, int64_t row1, float* acc, int32_t accumulate_gx,
                             int32_t update, const xmc_step_args* args, void* stream);

/* ---- elementwise numeric core (formats.py / optimizers.py), bit-exact ---- */

/* Grid of an emulated (exp_bits, man_bits) format, formats.py:49-137.
 * extended_range < 0 selects the reference default (e4m3 only). */
typedef struct {
  int32_t exp_bits;
  int32_t man_bits;
  int32_t extended_range;
  int32_t reserved;
} xmc_grid;

/* round_nearest (formats.py:197-206): out[i] = RTN(x[i]) as fp32 on-grid values. */
xmc_status xmc_round_nearest(xmc_grid g, const float* x, float* out, int64_t n, void* stream);

/* round_stochastic (formats.py:209-225) with RoundingRng(seed).uniform(step,
 * tensor_id, index[i]) (rng.py:54-57); index may be NULL (then i). */
xmc_status xmc_round_stochastic(xmc_grid g, const float* x, float* out, int64_t n, uint64_t seed,
                                uint64_t step, uint64_t tensor_id, const uint64_t* index, void* stream);

/* sgd_sr_step (optimizers.py:51-74) on fp32 on-grid weights:
 * w[i] <- ROUND(w - lr*(grad + wd*w)), keys index[i] (NULL -> i). Sets a
 * latched non-finite error through the return of the NEXT xmc_sync_status. */
xmc_status xmc_sgd_sr_step(xmc_grid g, float* w, const float* grad, int64_t n, float lr, float wd,
                           int32_t rounding, uint64_t seed, uint64_t step, uint64_t tensor_id,
                           const uint64_t* index, int32_t* status, void* stream);

/* Kahan-compensated SGD on the head grid (kahan_add
 * formats.py:246-263 composed with sgd_sr_step): fp32 on-grid w, fp32 comp. */
xmc_status xmc_kahan_sgd_step(xmc_grid g, float* w, float* comp, const float* grad, int64_t n, float lr,
                              float wd, int32_t rounding, uint64_t seed, uint64_t step,
                              uint64_t tensor_id, const uint64_t* index, int32_t* status, void* stream);

/* kahan_adamw_step (optimizers.py:112-137, kahan_add formats.py:246-263):
 * AdamW with bias-corrected fp32 moments m, v and a Kahan-compensated
 * parameter w (fp32 on-grid values) / comp (fp32), n elements, step t >= 1.
 * beta1/beta2 are the config's Python floats (double): the bias corrections
 * f32(1 - beta^t) are formed in double as the reference does.  Bit-exact with
 * the reference; non-finite moments or updates return XMC_ERR_NONFINITE and
 * leave every buffer unchanged. */
xmc_status xmc_kahan_adamw_step(xmc_grid g, float* w, float* comp, float* m, float* v, const float* grad,
                                int64_t n, float lr, double beta1, double beta2, float eps, float wd,
                                int64_t t, void* stream);

/* Native-storage RTN cast, e.g. X -> e4m3 bytes (head.py:265). */
xmc_status xmc_cast_rn(const float* x, void* out, int64_t n, int32_t fmt, int32_t* status, void* stream);

/* ---- node-local grad_X all-reduce over peer memory ----
 * Replaces the per-step `ncclAllReduce(sum)` of the ranks' partial grad_X
 * (the sum head_update's callers need when W is label-sharded; head.py:254-298
 * returns one rank's partial) together with the step's own reduction of the
 * grad_X partial slots: ONE kernel pushes each 32x32 tile of the rank's
 * partial into every peer's exchange buffer over NVLink (CUDA IPC mapping),
 * waits for the same tile from every peer and sums them in rank order, so all
 * ranks return bit-identical grad_X.
 *   xmc_peer_create  allocates this rank's exchange buffer (cudaMalloc) and
 *                    writes its 64-byte cudaIpcMemHandle_t to `handle`;
 *   xmc_peer_connect maps every peer's buffer (`handles`: world x 64 bytes,
 *                    rank order, swapped by the caller, e.g. all_gather);
 *   xmc_head_attach_peers  makes xmc_head_step* return the node's grad_X
 *                    (NULL detaches).  Every rank must run the same steps. */
typedef struct xmc_peer* xmc_peer_t;
xmc_status xmc_peer_create(int32_t rank, int32_t world, int32_t dim, int32_t max_batch, xmc_peer_t* out,
                           void* handle);
xmc_status xmc_peer_connect(xmc_peer_t p, const void* handles);
xmc_status xmc_peer_destroy(xmc_peer_t p);
xmc_status xmc_head_attach_peers(xmc_head_t h, xmc_peer_t p);

/* ---- measurement (no reference counterpart; used by bench.py) ---- */
/* Bracket every logits+G (fwd) and grad_X+update (bwd) launch with CUDA
 * events on its stream; xmc_profile_read syncs them, returns summed device ms
 * and launch counts since the previous read, and clears the record. */
xmc_status xmc_profile_enable(int32_t on);
xmc_status xmc_profile_read(double* ms_fwd, int64_t* n_fwd, double* ms_bwd, int64_t* n_bwd);
/* Effective SM clock of the same kernels: block 0 of every fwd / bwd launch
 * adds its clock64 cycles and globaltimer ns; out4 = {fwd cycles, fwd ns,
 * bwd cycles, bwd ns} since the previous read (cleared; synchronises). */
xmc_status xmc_profile_clock(uint64_t* out4);

#ifdef __cplusplus
}
#endif

#endif /* XMC_HEAD_H_ */
