// C-ABI implementation: workspace layout, TMA descriptor encoding, the small
// per-step kernels (X cast, positive-list bucketing, grad_X reduction), the
// bit-exact elementwise numeric core, and launch orchestration of the two
// tcgen05 kernels per chunk (xmc_fwd.cuh, xmc_bwd.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/xmc_head.h"
#include "xmc_bwd.cuh"
#include "xmc_fwd.cuh"
#include "xmc_ptx.cuh"
#include "xmc_round.cuh"

using namespace xmc;

// ============================================================== errors
static thread_local std::string g_err;

static xmc_status fail(xmc_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(XMC_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                                     \
  } while (0)

#define XMC_TRY(expr)              \
  do {                             \
    xmc_status s_ = (expr);        \
    if (s_ != XMC_OK) return s_;   \
  } while (0)

extern "C" const char* xmc_last_error(void) { return g_err.c_str(); }
extern "C" const char* xmc_version(void) { return "xmc-b200 0.1 (sm_100a tcgen05)"; }

// ============================================================== TMA maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// 2-D row-major tensor [rows][cols] of `eb`-byte elements, box [box_rows][128 B], 128-B swizzle.
// Tensor maps are pure functions of (base, shape, box): a small per-thread
// cache saves the ~1-2 us host encode per map on every step (6 maps per chunk).
struct MapEntry {
  CUtensorMap map;
  const void* base;
  uint64_t cols, rows, ld;
  int eb;
  uint32_t box;
};
static xmc_status encode_map(CUtensorMap* m, const void* base, int eb, uint64_t cols, uint64_t rows,
                             uint64_t ld_elems, uint32_t box_rows);

static xmc_status make_map(CUtensorMap* m, const void* base, int eb, uint64_t cols, uint64_t rows,
                           uint64_t ld_elems, uint32_t box_rows) {
  constexpr int kCache = 64;
  static thread_local std::vector<MapEntry> cache;
  static thread_local int next = 0;
  for (const MapEntry& e : cache)
    if (e.base == base && e.cols == cols && e.rows == rows && e.ld == ld_elems && e.eb == eb && e.box == box_rows) {
      *m = e.map;
      return XMC_OK;
    }
  XMC_TRY(encode_map(m, base, eb, cols, rows, ld_elems, box_rows));
  MapEntry e{*m, base, cols, rows, ld_elems, eb, box_rows};
  if (static_cast<int>(cache.size()) < kCache) cache.push_back(e);
  else cache[next++ % kCache] = e;
  return XMC_OK;
}

static xmc_status encode_map(CUtensorMap* m, const void* base, int eb, uint64_t cols, uint64_t rows,
                             uint64_t ld_elems, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(XMC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const CUtensorMapDataType dt = eb == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * eb};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / eb), box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(XMC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) cols=%llu rows=%llu", (int)r,
                (unsigned long long)cols, (unsigned long long)rows);
  return XMC_OK;
}

// ============================================================== profiling
// Optional CUDA-event bracketing of every fwd / bwd launch on its own stream
// (bench.py reads per-kernel device time of the timed region from here).
struct ProfRec {
  int kind;  // 0 = fwd, 1 = bwd
  cudaEvent_t a, b;
};
static bool g_prof = false;
static std::vector<ProfRec> g_prof_recs;

static void prof_begin(int kind, cudaStream_t st, ProfRec* r) {
  r->kind = kind;
  r->a = r->b = nullptr;
  if (!g_prof) return;
  cudaEventCreate(&r->a);
  cudaEventCreate(&r->b);
  cudaEventRecord(r->a, st);
}
static void prof_end(cudaStream_t st, ProfRec* r) {
  if (!g_prof || !r->a) return;
  cudaEventRecord(r->b, st);
  g_prof_recs.push_back(*r);
}

extern "C" xmc_status xmc_profile_enable(int32_t on) {
  g_prof = on != 0;
  return XMC_OK;
}

// Sum of device milliseconds and launch counts per kernel kind since the last
// read (synchronises on the recorded events, then clears them).
extern "C" xmc_status xmc_profile_read(double* ms_fwd, int64_t* n_fwd, double* ms_bwd, int64_t* n_bwd) {
  double t[2] = {0, 0};
  int64_t n[2] = {0, 0};
  for (auto& r : g_prof_recs) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      t[r.kind] += ms;
      n[r.kind] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof_recs.clear();
  if (ms_fwd) *ms_fwd = t[0];
  if (n_fwd) *n_fwd = n[0];
  if (ms_bwd) *ms_bwd = t[1];
  if (n_bwd) *n_bwd = n[1];
  return XMC_OK;
}

// ============================================================== helpers
static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline size_t align_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

static int elem_bytes(int fmt) { return fmt == XMC_FMT_E4M3 || fmt == XMC_FMT_E5M2 ? 1 : (fmt == XMC_FMT_FP32 ? 4 : 2); }

// padded batch = N of the logits MMA = G leading dimension
static int padded_batch(int eb, int B) {
  const int opts1[] = {128, 256};
  const int opts2[] = {64, 128, 256, 512};
  if (eb == 1) {
    for (int o : opts1) if (B <= o) return o;
  } else {
    for (int o : opts2) if (B <= o) return o;
  }
  return -1;
}

static std::vector<std::pair<int64_t, int64_t>> partition(int64_t total, int64_t parts) {
  std::vector<std::pair<int64_t, int64_t>> out;  // head.py:51-57
  for (int64_t i = 0; i < parts; ++i) {
    const int64_t a = (i * total) / parts, b = ((i + 1) * total) / parts;
    if (b > a) out.emplace_back(a, b);
  }
  return out;
}

// ============================================================== handle
struct xmc_head {
  xmc_head_desc desc;
  int eb;              // W / X / G element bytes
  int max_bp;          // padded batch capacity
  int num_sms;
  int dtiles;
  std::vector<std::pair<int64_t, int64_t>> chunks;  // local row ranges
  std::vector<int32_t> tile_base;                   // per chunk, plus total at the end
  int64_t total_tiles;
  int64_t max_chunk_rows;
  // workspace carve-up (device pointers)
  uint8_t* xq;         // [max_bp][d]
  uint8_t* xqt;        // [d][max_bp]
  uint8_t* gbuf;       // [max_chunk_rows][max_bp]
  float* gx_ws;        // [R][d][256]
  int32_t* tile_cnt;   // [total_tiles + 1]
  int32_t* tile_ptr;   // [total_tiles + 1]
  int32_t* tile_cur;   // [total_tiles + 1] scatter cursors (tile_cnt is re-zeroed by the scan)
  uint32_t* entries;   // [max_positives]
  uint32_t* tmp_tile;  // [max_positives] tile id per positive (bucketing scratch)
  uint32_t* tmp_entry; // [max_positives] packed entry per positive
  int64_t* chunk_dev;  // [k+1] chunk starts (local rows) + [k+1] tile bases
  int32_t* status;     // [4]
  int32_t* ring_ready;      // [max chunk tiles + 1] fused step flags (zeroed per launch)
  int32_t* ring_consumed;   // [max chunk tiles + 1]
  int R_step;          // grad_X partial slots written by the current step's backward
  uint8_t* xq_topk;    // Xq rows of the current top-k launch (sample offset applied)
  uint8_t* wm;         // [max_chunk_rows + 128][d] masked W chunk (dropout only)
  uint32_t* keep;      // [max_chunk_rows + 128][d / 32] dropout keep bits (dropout only)
  int64_t comp_rows;   // local rows [0, comp_rows) carry a Kahan compensation
  float* cand_s;       // [max_bp][4 num_sms][kTopK] streaming top-k candidates (scores)
  int32_t* cand_l;     // [max_bp][4 num_sms][kTopK] (global labels)
  int R;               // bwd CTAs per d-tile
  int gcl;             // bwd G-sharing cluster size (TMA multicast across consecutive d-tiles)
  int fwd_max_clusters;   // co-resident CTA pairs of the forward (grid cap, PDL safety)
  bool pdl_ok;
  // Adam-style head step in flight (xmc_head_step_adamw sets it for the call):
  // moments at local row 0 and the kahan_adamw_step constants
  struct {
    float* m = nullptr;
    float* v = nullptr;
    float b1, b2, omb1, omb2, bc1, bc2, eps;
  } adam;
  size_t l2_persist;   // persisting-L2 bytes granted for the G window (0 = off)
  size_t l2_window_max;
  struct xmc_peer* peer = nullptr;   // node-local grad_X all-reduce group (xmc_head_attach_peers)
};

// ---- node-local grad_X all-reduce over peer memory (CUDA IPC / NVLink P2P) ----
// Every rank cudaMallocs one exchange buffer and maps every peer's (IPC
// handles swapped by the caller).  Layout, identical on all ranks:
//   xin   [2 parity][world src][nblocks][1024] fp32   32x32 grad_X tiles pushed by rank src
//   flags [2 parity][world src][nblocks] int32         epoch of the step that pushed the tile
constexpr int kMaxPeers = 8;
struct xmc_peer {
  int rank = 0, world = 1, dim = 0, max_bp = 0, nblocks = 0;
  uint8_t* local = nullptr;   // own exchange buffer
  size_t bytes = 0, flag_off = 0;
  void* base[kMaxPeers] = {};   // every rank's buffer as mapped here (own = local)
  int32_t epoch = 0;
  bool connected = false;
};

// ---- fused step: forward and backward of a chunk in ONE persistent launch ----
// Hypothesis: the forward is DRAM-bound (W streams in once) and the backward
// is bound by shared-memory bandwidth, so they would overlap on disjoint SMs:
// the first
// nfwd CTAs run the forward (split layout, cta_group::1 like the backward)
// and hand G to the other CTAs through an L2-resident ring of 128-row tiles
// (FwdParams / BwdParams ring_* fields); the backward then re-reads each W
// tile from L2 shortly after the forward streamed it in.  Every CTA of the
// grid is resident (one per SM, grid <= SMs), so the flag waits cannot
// deadlock: the smallest tile not yet written only waits for the backward of
// a smaller tile, which only waits for tiles written before it.
// Measured: slower than the two launches at every split
// (4.97 / 3.90 ms per step with 34 / 44 forward CTAs vs 1.96 ms), because the
// forward is not idle-SM work: its epilogue and W pipeline cost ~84 SM-ms per
// step in the pair layout and more in the split one, so moving it beside the
// backward cannot shorten the sum.  Kept as a tested option.
template <int KC>
__global__ void __launch_bounds__(kBwdThreads, 1)
    xmc_step_kernel(const __grid_constant__ CUtensorMap fw, const __grid_constant__ CUtensorMap fx,
                    const __grid_constant__ CUtensorMap bw, const __grid_constant__ CUtensorMap bg,
                    const __grid_constant__ CUtensorMap bxt, const __grid_constant__ CUtensorMap bws, FwdParams fp,
                    BwdParams bp, int nfwd) {
  static_assert(FwdCfg<1, 128, false, true>::kThreads == kBwdThreads, "one block shape for both roles");
  const int b = static_cast<int>(blockIdx.x);
  if (b < nfwd) fwd_body<1, 128, false, false, true, true>(fw, fx, fp, b >> 1, nfwd >> 1, b & 1);
  else bwd_body<1, true, KC, 0, true, false, true>(bw, bg, bxt, bws, bp, b - nfwd, static_cast<int>(gridDim.x) - nfwd);
}

constexpr int kStepSmem = FwdCfg<1, 128, false, true>::kSmemBytes > BwdCfg<1, true, 2>::kSmemBytes
                              ? FwdCfg<1, 128, false, true>::kSmemBytes
                              : BwdCfg<1, true, 2>::kSmemBytes;

struct Layout {
  size_t xq, xqt, gbuf, gx, cnt, ptr, cur, ent, tmp, chunk, status, flags, wm, keep, cand, total;
};

static xmc_status compute_layout(const xmc_head_desc* d, Layout* L, int* eb_out, int* bp_out, int* R_out,
                                 int64_t* tiles_out, int64_t* maxrows_out, int num_sms) {
  if (!d) return fail(XMC_ERR_ARG, "null desc");
  if (d->fmt != XMC_FMT_E4M3 && d->fmt != XMC_FMT_BF16)
    return fail(XMC_ERR_UNSUPPORTED, "head format must be e4m3 or bf16 (got %d)", d->fmt);
  const int eb = elem_bytes(d->fmt);
  if (d->dim <= 0 || d->dim % 128 != 0)
    return fail(XMC_ERR_SHAPE, "dim must be a positive multiple of 128 (got %d)", d->dim);
  if (d->num_chunks < 1) return fail(XMC_ERR_ARG, "num_chunks must be >= 1");
  if (d->comp_bytes != 0 && d->comp_bytes != 2 && d->comp_bytes != 4)
    return fail(XMC_ERR_ARG, "comp_bytes must be 0 (none), 2 (bf16) or 4 (fp32)");
  if (d->num_labels_local < 1 || d->label_offset < 0 ||
      d->label_offset + d->num_labels_local > d->num_labels_global)
    return fail(XMC_ERR_ARG, "bad label shard [%lld, +%lld) of %lld", (long long)d->label_offset,
                (long long)d->num_labels_local, (long long)d->num_labels_global);
  if (d->max_batch < 1 || d->max_batch > 65535) return fail(XMC_ERR_ARG, "max_batch out of range");
  const int bp = padded_batch(eb, d->max_batch);
  if (bp < 0) return fail(XMC_ERR_UNSUPPORTED, "batch %d too large for format", d->max_batch);
  auto ch = partition(d->num_labels_local, d->num_chunks);
  int64_t tiles = 0, maxrows = 0;
  for (auto& c : ch) {
    tiles += cdiv(c.second - c.first, 128);
    maxrows = std::max(maxrows, c.second - c.first);
  }
  const int dtiles = d->dim / 128;
  int R = std::max(1, num_sms / dtiles);
  const int64_t D = d->dim;
  L->xq = 0;
  L->xqt = align_up(L->xq + (size_t)bp * D * eb, 1024);
  L->gbuf = align_up(L->xqt + (size_t)bp * D * eb, 1024);
  L->gx = align_up(L->gbuf + (size_t)(maxrows + 128) * bp * eb, 1024);
  L->cnt = align_up(L->gx + (size_t)R * D * bp * 4, 256);
  L->ptr = align_up(L->cnt + (size_t)(tiles + 1) * 4, 256);
  L->cur = align_up(L->ptr + (size_t)(tiles + 1) * 4, 256);
  L->ent = align_up(L->cur + (size_t)(tiles + 1) * 4, 256);
  L->tmp = align_up(L->ent + (size_t)std::max<int64_t>(d->max_positives, 1) * 4, 256);
  L->chunk = align_up(L->tmp + (size_t)std::max<int64_t>(d->max_positives, 1) * 8, 256);
  L->status = align_up(L->chunk + (size_t)(2 * (ch.size() + 1)) * 8, 256);
  L->flags = align_up(L->status + 64, 256);   // fused step: ready + consumed per chunk tile
  L->wm = align_up(L->flags + (size_t)2 * (cdiv(maxrows, 128) + 1) * 4, 1024);
  L->keep = align_up(L->wm + (d->dropout ? (size_t)(maxrows + 128) * D * eb : 0), 1024);
  L->cand = align_up(L->keep + (d->dropout ? (size_t)(maxrows + 128) * (D / 32) * 4 : 0), 1024);
  L->total = align_up(L->cand + (size_t)bp * 4 * num_sms * kTopK * 8, 1024);
  *eb_out = eb;
  *bp_out = bp;
  *R_out = R;
  *tiles_out = tiles;
  *maxrows_out = maxrows;
  return XMC_OK;
}

static int device_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

extern "C" xmc_status xmc_head_workspace_size(const xmc_head_desc* desc, size_t* bytes) {
  Layout L;
  int eb, bp, R;
  int64_t t, m;
  const int sms = desc && desc->num_sms > 0 ? desc->num_sms : device_sms();
  XMC_TRY(compute_layout(desc, &L, &eb, &bp, &R, &t, &m, sms));
  *bytes = L.total;
  return XMC_OK;
}

template <int EB, int BN>
static void set_fwd_attr() {
  cudaFuncSetAttribute(xmc_fwd_kernel<EB, BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       FwdCfg<EB, BN, false>::kSmemBytes);
  if constexpr (BN <= 256)
    cudaFuncSetAttribute(xmc_fwd_kernel<EB, BN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FwdCfg<EB, BN, false>::kSmemBytes);
  if constexpr (BN <= 256 && BN >= 128)
    cudaFuncSetAttribute(xmc_fwd_kernel<EB, BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FwdCfg<EB, BN, true>::kSmemBytes);
  if constexpr (EB == 1 && BN <= 256 && BN >= 128)
    cudaFuncSetAttribute(xmc_fwd_kernel<EB, BN, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FwdCfg<EB, BN, true, true>::kSmemBytes);
  if constexpr (EB == 1 && BN == 128)
    cudaFuncSetAttribute(xmc_fwd_kernel<EB, BN, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FwdCfg<EB, BN, false, true>::kSmemBytes);
  if constexpr (EB == 1 && BN == 256)
    cudaFuncSetAttribute(xmc_fwd_kernel<EB, BN, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         FwdCfg<EB, BN, true, true>::kSmemBytes);
}
template <int EB, bool XR, int KC>
static void set_bwd_attr() {
  cudaFuncSetAttribute(xmc_bwd_kernel<EB, XR, KC, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       BwdCfg<EB, XR, KC>::kSmemBytes);
  cudaFuncSetAttribute(xmc_bwd_kernel<EB, XR, KC, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       BwdCfg<EB, XR, KC>::kSmemBytes);
  cudaFuncSetAttribute(xmc_bwd_kernel<EB, XR, KC, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       BwdCfg<EB, XR, KC>::kSmemBytes);
  cudaFuncSetAttribute(xmc_bwd_kernel<EB, XR, KC, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       BwdCfg<EB, XR, KC>::kSmemBytes);
}

// Measurement only: XMC_TRACE=1 records clock64 per tile and pipeline event
// of the first backward CTA (xmc_trace_read, tools/trace_bwd.py).
static uint64_t* trace_buf() {
  static uint64_t* buf = nullptr;
  static const bool on = getenv("XMC_TRACE") && atoi(getenv("XMC_TRACE")) != 0;
  if (on && !buf && cudaMalloc(&buf, kTraceTiles * 16 * 8) != cudaSuccess) {
    cudaGetLastError();
    buf = nullptr;
  }
  return on ? buf : nullptr;
}

extern "C" xmc_status xmc_trace_read(uint64_t* out, int64_t n) {
  uint64_t* b = trace_buf();
  if (!b) return fail(XMC_ERR_ARG, "tracing is off (set XMC_TRACE=1)");
  CUDA_TRY(cudaMemcpy(out, b, std::min<int64_t>(n, kTraceTiles * 16) * 8, cudaMemcpyDeviceToHost));
  return XMC_OK;
}

// Backward G sharing: the d-tiles of one label tile run as a cluster and each G
// tile is read from L2 once per cluster (TMA multicast) instead of once per
// d-tile.  The cluster size c divides d/128; R (CTAs per d-tile) shrinks if
// fewer than R*dtiles/c clusters can be co-resident (a second wave would cost
// more than the shared reads save).  XMC_BWD_GCL overrides (1 = off).
static void choose_bwd_cluster(xmc_head* h) {
  const char* env = getenv("XMC_BWD_GCL");
  const int want = env ? atoi(env) : 1;
  h->gcl = 1;
  for (int c : {want, 6, 3, 2}) {
    if (c <= 1 || c > 8 || c > want || h->dtiles % c != 0) continue;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(h->R * h->dtiles);
    cfg.blockDim = dim3(kBwdThreads);
    cfg.dynamicSmemBytes = BwdCfg<1, true, 2>::kSmemBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, xmc_bwd_kernel<1, true, 2, 0>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    const int r = std::min(h->R, n * c / h->dtiles);
    if (getenv("XMC_VERBOSE")) fprintf(stderr, "xmc: bwd cluster %d: %d co-resident clusters\n", c, n);
    if (r >= 1 && r * 10 >= h->R * 9) {   // keep >= 90 % of the CTAs
      h->R = r;
      h->gcl = c;
      return;
    }
  }
}

extern "C" xmc_status xmc_head_create(const xmc_head_desc* desc, void* workspace, size_t workspace_bytes,
                                      xmc_head_t* out) {
  if (!out) return fail(XMC_ERR_ARG, "null out");
  Layout L;
  int eb, bp, R;
  int64_t tiles, maxrows;
  const int sms = desc && desc->num_sms > 0 ? desc->num_sms : device_sms();
  XMC_TRY(compute_layout(desc, &L, &eb, &bp, &R, &tiles, &maxrows, sms));
  if (!workspace || workspace_bytes < L.total)
    return fail(XMC_ERR_CAPACITY, "workspace too small: need %zu bytes", L.total);
  if (reinterpret_cast<uintptr_t>(workspace) % 1024 != 0)
    return fail(XMC_ERR_ARG, "workspace must be 1024-byte aligned");
  xmc_head* h = new xmc_head();
  h->desc = *desc;
  h->eb = eb;
  h->max_bp = bp;
  h->num_sms = sms;
  h->dtiles = desc->dim / 128;
  h->R = R;
  h->R_step = R;
  h->chunks = partition(desc->num_labels_local, desc->num_chunks);
  h->total_tiles = tiles;
  h->max_chunk_rows = maxrows;
  uint8_t* w = static_cast<uint8_t*>(workspace);
  h->xq = w + L.xq;
  h->xqt = w + L.xqt;
  h->gbuf = w + L.gbuf;
  h->gx_ws = reinterpret_cast<float*>(w + L.gx);
  h->tile_cnt = reinterpret_cast<int32_t*>(w + L.cnt);
  h->tile_ptr = reinterpret_cast<int32_t*>(w + L.ptr);
  h->tile_cur = reinterpret_cast<int32_t*>(w + L.cur);
  h->entries = reinterpret_cast<uint32_t*>(w + L.ent);
  // Optional L2 persistence for the G chunk buffer (XMC_L2_PERSIST=1).  Off by
  // default: measured on B200 it thrashes once G exceeds the persisting carve-
  // out and gains nothing below it (profiles/r1_notes.md).
  h->l2_persist = 0;
  h->l2_window_max = 0;
  {
    const char* env = getenv("XMC_L2_PERSIST");
    int dev = 0, pmax = 0, wmax = 0;
    if ((env && atoi(env) != 0) && cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&pmax, cudaDevAttrMaxPersistingL2CacheSize, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&wmax, cudaDevAttrMaxAccessPolicyWindowSize, dev) == cudaSuccess && pmax > 0 &&
        wmax > 0) {
      const size_t want = std::min<size_t>(pmax, (size_t)(maxrows + 128) * bp * eb);
      if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
        h->l2_persist = want;
        h->l2_window_max = wmax;
      }
      cudaGetLastError();
    }
  }
  h->tmp_tile = reinterpret_cast<uint32_t*>(w + L.tmp);
  h->tmp_entry = h->tmp_tile + std::max<int64_t>(desc->max_positives, 1);
  h->chunk_dev = reinterpret_cast<int64_t*>(w + L.chunk);
  h->status = reinterpret_cast<int32_t*>(w + L.status);
  h->ring_ready = reinterpret_cast<int32_t*>(w + L.flags);
  h->ring_consumed = h->ring_ready + (cdiv(maxrows, 128) + 1);
  h->wm = desc->dropout ? w + L.wm : nullptr;
  h->keep = desc->dropout ? reinterpret_cast<uint32_t*>(w + L.keep) : nullptr;
  h->comp_rows = desc->comp_bytes == 0 ? 0
                 : desc->comp_labels <= 0
                     ? desc->num_labels_local
                     : std::min<int64_t>(desc->num_labels_local,
                                         std::max<int64_t>(0, desc->comp_labels - desc->label_offset));
  h->cand_s = reinterpret_cast<float*>(w + L.cand);
  h->cand_l = reinterpret_cast<int32_t*>(w + L.cand + (size_t)bp * 4 * sms * kTopK * 4);
  std::vector<int64_t> host(2 * (h->chunks.size() + 1));
  int64_t tb = 0;
  for (size_t c = 0; c < h->chunks.size(); ++c) {
    host[c] = h->chunks[c].first;
    host[h->chunks.size() + 1 + c] = tb;
    h->tile_base.push_back(static_cast<int32_t>(tb));
    tb += cdiv(h->chunks[c].second - h->chunks[c].first, 128);
  }
  host[h->chunks.size()] = desc->num_labels_local;
  host[2 * h->chunks.size() + 1] = tb;
  h->tile_base.push_back(static_cast<int32_t>(tb));
  cudaError_t e1 = cudaMemcpy(h->chunk_dev, host.data(), host.size() * 8, cudaMemcpyHostToDevice);
  cudaError_t e2 = cudaMemset(h->status, 0, 64);
  if (e2 == cudaSuccess) e2 = cudaMemset(h->tile_cnt, 0, (tiles + 1) * 4);   // re-zeroed by every scan
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    delete h;
    return fail(XMC_ERR_CUDA, "workspace init failed: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  set_fwd_attr<1, 128>();
  set_fwd_attr<1, 256>();
  set_fwd_attr<2, 64>();
  set_fwd_attr<2, 128>();
  set_fwd_attr<2, 256>();
  set_fwd_attr<2, 512>();
  set_bwd_attr<1, true, 1>();
  set_bwd_attr<1, true, 2>();
  set_bwd_attr<2, true, 1>();
  set_bwd_attr<2, true, 2>();
  set_bwd_attr<2, true, 4>();
  set_bwd_attr<2, false, 8>();
  cudaFuncSetAttribute(xmc_step_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem);
  choose_bwd_cluster(h);
  // forward pairs: how many CTA pairs are co-resident.  The persistent grid is
  // capped there, which keeps every primary of a PDL chain fully resident.
  {
    h->fwd_max_clusters = h->num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (h->num_sms / 2));
    cfg.blockDim = dim3(FwdCfg<1, 256, true, true>::kThreads);
    cfg.dynamicSmemBytes = FwdCfg<1, 256, true, true>::kSmemBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    h->pdl_ok = cudaOccupancyMaxActiveClusters(&n, xmc_fwd_kernel<1, 256, true, false, true>, &cfg) == cudaSuccess &&
                n > 0;
    cudaGetLastError();
    if (h->pdl_ok) h->fwd_max_clusters = std::min(h->fwd_max_clusters, n);
  }
  *out = h;
  return XMC_OK;
}

// ---- peer group (C ABI) ----
extern "C" xmc_status xmc_peer_create(int32_t rank, int32_t world, int32_t dim, int32_t max_batch, xmc_peer_t* out,
                                      void* handle) {
  if (!out || !handle) return fail(XMC_ERR_ARG, "null argument");
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return fail(XMC_ERR_ARG, "rank %d / world %d outside [0, %d)", rank, world, kMaxPeers);
  if (dim <= 0 || dim % 128 != 0) return fail(XMC_ERR_SHAPE, "dim must be a positive multiple of 128");
  if (max_batch < 1 || max_batch > 512) return fail(XMC_ERR_ARG, "max_batch outside [1, 512]");
  auto* p = new xmc_peer();
  p->rank = rank;
  p->world = world;
  p->dim = dim;
  p->max_bp = std::max(padded_batch(2, max_batch), 128);   // covers either format's padded batch
  p->nblocks = (dim / 32) * (p->max_bp / 32);
  const size_t xin = static_cast<size_t>(2) * world * p->nblocks * 1024 * 4;
  p->flag_off = align_up(xin, 256);
  p->bytes = p->flag_off + static_cast<size_t>(2) * world * p->nblocks * 4;
  cudaError_t e = cudaMalloc(&p->local, p->bytes);
  if (e == cudaSuccess) e = cudaMemset(p->local, 0, p->bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), p->local);
  if (e != cudaSuccess) {
    if (p->local) cudaFree(p->local);
    delete p;
    cudaGetLastError();
    return fail(XMC_ERR_CUDA, "peer exchange buffer: %s", cudaGetErrorString(e));
  }
  p->base[rank] = p->local;
  *out = p;
  return XMC_OK;
}

extern "C" xmc_status xmc_peer_connect(xmc_peer_t p, const void* handles) {
  if (!p || !handles) return fail(XMC_ERR_ARG, "null argument");
  if (p->connected) return XMC_OK;
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int r = 0; r < p->world; ++r) {
    if (r == p->rank) continue;
    void* q = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&q, hs[r], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (int k = 0; k < r; ++k)
        if (k != p->rank && p->base[k]) cudaIpcCloseMemHandle(p->base[k]);
      return fail(XMC_ERR_CUDA, "peer %d exchange buffer not mappable: %s", r, cudaGetErrorString(e));
    }
    p->base[r] = q;
  }
  p->connected = true;
  return XMC_OK;
}

extern "C" xmc_status xmc_peer_destroy(xmc_peer_t p) {
  if (!p) return XMC_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < p->world; ++r)
    if (r != p->rank && p->base[r]) cudaIpcCloseMemHandle(p->base[r]);
  if (p->local) cudaFree(p->local);
  delete p;
  cudaGetLastError();
  return XMC_OK;
}

extern "C" xmc_status xmc_head_attach_peers(xmc_head_t h, xmc_peer_t p) {
  if (!h) return fail(XMC_ERR_ARG, "null handle");
  if (p && (!p->connected || p->dim != h->desc.dim || p->max_bp < h->max_bp))
    return fail(XMC_ERR_ARG, "peer group not connected or built for another dim / batch");
  h->peer = p;
  return XMC_OK;
}

extern "C" xmc_status xmc_head_destroy(xmc_head_t h) {
  delete h;
  return XMC_OK;
}

// ============================================================== small kernels
// X fp32 [B][d] -> Xq [Bp][d] and Xq^T [d][Bp] on the head grid (RTN,
// head.py:265 / formats.py:197-206); padding rows/cols are zero.
template <int EB>
__device__ __forceinline__ void x_prep_body(const float* __restrict__ X, int B, int Bp, int d,
                                            uint8_t* __restrict__ xq, uint8_t* __restrict__ xqt, int32_t* status,
                                            int bx, int by, int tx, int ty, int ny) {
  __shared__ float tile[32][33];
  const int c0 = bx * 32, s0 = by * 32;
  bool bad = false;
  for (int i = ty; i < 32; i += ny) {
    const int s = s0 + i, c = c0 + tx;
    float v = 0.f;
    if (s < B) {
      v = X[(int64_t)s * d + c];
      bad |= !isfinite(v);
    }
    float q;
    if (EB == 1) q = dec_e4m3(enc_e4m3(v));
    else q = dec_bf16(enc_bf16(v));
    tile[i][tx] = q;
    if (EB == 1) xq[(int64_t)s * d + c] = enc_e4m3(v);
    else reinterpret_cast<uint16_t*>(xq)[(int64_t)s * d + c] = enc_bf16(v);
  }
  __syncthreads();
  for (int i = ty; i < 32; i += ny) {
    const int c = c0 + i, s = s0 + tx;
    const float q = tile[tx][i];
    if (EB == 1) xqt[(int64_t)c * Bp + s] = enc_e4m3(q);
    else reinterpret_cast<uint16_t*>(xqt)[(int64_t)c * Bp + s] = enc_bf16(q);
  }
  if (bad) atomicOr(status, ST_NONFINITE_X);
}

template <int EB>
__global__ void x_prep_kernel(const float* __restrict__ X, int B, int Bp, int d, uint8_t* __restrict__ xq,
                              uint8_t* __restrict__ xqt, int32_t* status) {
  x_prep_body<EB>(X, B, Bp, d, xq, xqt, status, blockIdx.x, blockIdx.y, threadIdx.x, threadIdx.y, blockDim.y);
}

struct PosGeom {
  const int64_t* chunk_start;  // [k+1]
  const int64_t* tile_base;    // [k+1]
  int32_t k;
  int64_t label_offset;
  int64_t num_local;
  int32_t B;
};

__device__ __forceinline__ int64_t pos_tile(const PosGeom& g, int64_t local, int32_t* row_in_tile) {
  // chunk c with chunk_start[c] <= local < chunk_start[c+1]; bounds are i*n/k,
  // so a float estimate is off by at most one and the loops fix it up
  int c = static_cast<int>(static_cast<float>(local) * (static_cast<float>(g.k) / static_cast<float>(g.num_local)));
  c = c < 0 ? 0 : c;
  if (c >= g.k) c = g.k - 1;
  while (c > 0 && g.chunk_start[c] > local) --c;
  while (c + 1 < g.k && g.chunk_start[c + 1] <= local) ++c;
  const int64_t off = local - g.chunk_start[c];
  *row_in_tile = static_cast<int32_t>(off & 127);
  return g.tile_base[c] + (off >> 7);
}

// grad_x[s][c] += sum_r ws[r][c][s - col0]   (fixed r order: deterministic)
// one thread per output element (block 32 x 32): R independent coalesced loads
// in flight per thread, fixed summation order r = 0..R-1 (deterministic)
__global__ void __launch_bounds__(1024) gx_reduce_kernel(const float* __restrict__ ws, int R, int d, int ld, int B,
                                                         float scale, int accumulate, float* __restrict__ gx) {
  __shared__ float tile[32][33];
  griddep_wait();   // launched as a PDL dependent of the last backward
  const int c = blockIdx.x * 32 + threadIdx.y, s = blockIdx.y * 32 + threadIdx.x;
  float acc = 0.f;
  if (s < B) {
    const float* p = ws + (int64_t)c * ld + s;
    const int64_t stride = (int64_t)d * ld;
    float v[8];
    int r = 0;
    for (; r + 8 <= R; r += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(p + (r + k) * stride);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
    for (; r < R; ++r) acc += __ldg(p + r * stride);
  }
  tile[threadIdx.y][threadIdx.x] = acc * scale;
  __syncthreads();
  const int s2 = blockIdx.y * 32 + threadIdx.y, c2 = blockIdx.x * 32 + threadIdx.x;
  if (s2 < B) {
    float* o = gx + (int64_t)s2 * d + c2;
    *o = accumulate ? *o + tile[threadIdx.x][threadIdx.y] : tile[threadIdx.x][threadIdx.y];
  }
}

struct PeerArgs {
  uint8_t* base[kMaxPeers];   // every rank's exchange buffer, mapped in this process
  int32_t rank, world, nblocks;
  int32_t epoch;
  int64_t flag_off;           // byte offset of the flags in a buffer
  int32_t* status;
};

// grad_X of the node in one kernel: each 32x32 tile of this rank's partial
// sum (its R slots, as gx_reduce_kernel) is pushed into every rank's exchange
// buffer over NVLink, released by a per-(rank, tile) epoch flag; then the
// block waits for the same tile from every peer and sums the world pushes in
// rank order, so every rank ends with bit-identical grad_X.  A block pushes
// before it waits and waits only for the same tile index, so the exchange
// needs no grid-wide co-residency.  Exchange buffers alternate by step parity;
// a rank rewrites parity p two steps later, after every peer has passed the
// next step's flags, i.e. finished reading parity p.
__global__ void __launch_bounds__(1024) gx_reduce_peer_kernel(const float* __restrict__ ws, int R, int d, int ld,
                                                              int B, float scale, float* __restrict__ gx,
                                                              const __grid_constant__ PeerArgs pa) {
  __shared__ float tile[32][33];
  griddep_wait();
  const int c = blockIdx.x * 32 + threadIdx.y, s = blockIdx.y * 32 + threadIdx.x;
  float acc = 0.f;
  if (s < B) {
    const float* p = ws + (int64_t)c * ld + s;
    const int64_t stride = (int64_t)d * ld;
    float v[8];
    int r = 0;
    for (; r + 8 <= R; r += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(p + (r + k) * stride);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
    for (; r < R; ++r) acc += __ldg(p + r * stride);
  }
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int bid = blockIdx.y * gridDim.x + blockIdx.x;
  const int par = pa.epoch & 1;
  const int64_t slot = (static_cast<int64_t>(par) * pa.world + pa.rank) * pa.nblocks + bid;
  for (int q = 0; q < pa.world; ++q) __stcg(reinterpret_cast<float*>(pa.base[q]) + slot * 1024 + tid, acc * scale);
  __threadfence_system();
  __syncthreads();
  if (tid < pa.world) {   // release this tile to rank tid, then wait for rank tid's tile
    st_release_sys(reinterpret_cast<int32_t*>(pa.base[tid] + pa.flag_off) + slot, pa.epoch);
    const int32_t* f = reinterpret_cast<const int32_t*>(pa.base[pa.rank] + pa.flag_off) +
                       (static_cast<int64_t>(par) * pa.world + tid) * pa.nblocks + bid;
    if (ld_acquire_sys(f) < pa.epoch) {
      const long long t0 = clock64();
      while (ld_acquire_sys(f) < pa.epoch) {
        if (clock64() - t0 > (1ll << 33)) {
          atomicOr(pa.status, ST_PEER_TIMEOUT);
          break;
        }
      }
    }
  }
  __syncthreads();
  const float* mine = reinterpret_cast<const float*>(pa.base[pa.rank]);
  float tot = 0.f;
  for (int q = 0; q < pa.world; ++q)
    tot += __ldcg(mine + ((static_cast<int64_t>(par) * pa.world + q) * pa.nblocks + bid) * 1024 + tid);
  tile[threadIdx.y][threadIdx.x] = tot;
  __syncthreads();
  const int s2 = blockIdx.y * 32 + threadIdx.y, c2 = blockIdx.x * 32 + threadIdx.x;
  if (s2 < B) gx[(int64_t)s2 * d + c2] = tile[threadIdx.x][threadIdx.y];
}

// Bitonic sort of 32 (key, value) pairs across a warp (15 shuffle exchanges).
__device__ __forceinline__ void warp_sort_pairs(uint32_t& key, uint32_t& val) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t ok = __shfl_xor_sync(0xffffffffu, key, j);
      const uint32_t ov = __shfl_xor_sync(0xffffffffu, val, j);
      const bool asc = (lane & k) == 0, lower = (lane & j) == 0;
      const bool take = (lower == asc) ? (ok < key) : (ok > key);
      if (take) {
        key = ok;
        val = ov;
      }
    }
  }
}

// After warp_sort_pairs: start lane of this lane's run of equal keys and the
// run length (valid on the run's first lane).
__device__ __forceinline__ void warp_runs(uint32_t key, int* start, int* len) {
  const int lane = threadIdx.x & 31;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = lane == 0 || prev != key;
  const uint32_t heads = __ballot_sync(0xffffffffu, head);
  *start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
  const uint32_t above = heads & ~(0xffffffffu >> (31 - lane));
  *len = (above ? __ffs(above) - 1 : 32) - lane;
}

// ---- multi-CTA positive bucketing: count -> scan -> scatter -------------
// K1: tile id per positive (kept for K3) + warp-aggregated global counts
__device__ __forceinline__ void pos_count_body(PosGeom g, const int32_t* __restrict__ ps,
                                               const int32_t* __restrict__ pl, int64_t nnz, int32_t* __restrict__ cnt,
                                               uint32_t* __restrict__ tmp_tile, uint32_t* __restrict__ tmp_entry,
                                               int32_t* status, int block) {
  const int64_t i = block * 256ll + threadIdx.x;
  uint32_t key = 0xffffffffu, val = 0;
  bool bad = false;
  if (i < nnz) {
    const int32_t s = ps[i];
    const int64_t local = static_cast<int64_t>(pl[i]) - g.label_offset;
    if (s < 0 || s >= g.B) bad = true;
    else if (local >= 0 && local < g.num_local) {
      int32_t r;
      key = static_cast<uint32_t>(pos_tile(g, local, &r));
      val = (static_cast<uint32_t>(r) << 16) | static_cast<uint32_t>(s);
    }
    tmp_tile[i] = key;
    tmp_entry[i] = val;
  }
  if (bad) atomicOr(status, ST_BAD_SAMPLE);
  warp_sort_pairs(key, val);
  int st, len;
  warp_runs(key, &st, &len);
  if (key != 0xffffffffu && (threadIdx.x & 31) == st) atomicAdd(&cnt[key], len);
}

__global__ void __launch_bounds__(256) pos_count_kernel(PosGeom g, const int32_t* __restrict__ ps,
                                                        const int32_t* __restrict__ pl, int64_t nnz,
                                                        int32_t* __restrict__ cnt, uint32_t* __restrict__ tmp_tile,
                                                        uint32_t* __restrict__ tmp_entry, int32_t* status) {
  pos_count_body(g, ps, pl, nnz, cnt, tmp_tile, tmp_entry, status, blockIdx.x);
}

// x_prep (blocks [0, nx)) and K1 (blocks [nx, ...)) in one launch: they are
// independent, and the counters they need zeroed were zeroed by the previous
// step's scan (or at handle creation)
template <int EB>
__global__ void __launch_bounds__(256) prep_count_kernel(const float* __restrict__ X, int B, int Bp, int d,
                                                         uint8_t* __restrict__ xq, uint8_t* __restrict__ xqt, int nx,
                                                         PosGeom g, const int32_t* __restrict__ ps,
                                                         const int32_t* __restrict__ pl, int64_t nnz,
                                                         int32_t* __restrict__ cnt, uint32_t* __restrict__ tmp_tile,
                                                         uint32_t* __restrict__ tmp_entry, int32_t* status) {
  if (static_cast<int>(blockIdx.x) < nx) {
    x_prep_body<EB>(X, B, Bp, d, xq, xqt, status, blockIdx.x % (d / 32), blockIdx.x / (d / 32), threadIdx.x & 31,
                    threadIdx.x >> 5, 8);
    return;
  }
  pos_count_body(g, ps, pl, nnz, cnt, tmp_tile, tmp_entry, status, blockIdx.x - nx);
}

// K2: exclusive scan of the T tile counters (one CTA; smem-staged segments)
__global__ void __launch_bounds__(1024) pos_scan_kernel(int32_t* __restrict__ cnt, int32_t* __restrict__ ptr,
                                                        int32_t* __restrict__ cur, int32_t T) {
  extern __shared__ int32_t sc[];   // [T]
  __shared__ int32_t wsum[32];
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < T; i += nth) sc[i] = cnt[i];
  __syncthreads();
  const int per = (T + nth - 1) / nth;
  const int a = min(T, tid * per), b = min(T, a + per);
  int32_t run = 0;
  for (int i = a; i < b; ++i) run += sc[i];
  int32_t x = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t v = lane < (nth >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  int32_t pre = (w > 0 ? wsum[w - 1] : 0) + x - run;
  for (int i = a; i < b; ++i) {
    const int32_t c = sc[i];
    sc[i] = pre;
    pre += c;
  }
  if (tid == nth - 1) ptr[T] = pre;
  __syncthreads();
  for (int i = tid; i < T; i += nth) {
    ptr[i] = sc[i];
    cur[i] = sc[i];   // the scatter cursor
    cnt[i] = 0;       // counters start the next step at zero (no memset launch)
  }
}

// K3: scatter packed entries to their tile buckets (warp-aggregated cursors)
__global__ void __launch_bounds__(256) pos_scatter_kernel(int64_t nnz, const uint32_t* __restrict__ tmp_tile,
                                                          const uint32_t* __restrict__ tmp_entry,
                                                          int32_t* __restrict__ cursor, uint32_t* __restrict__ entries) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  uint32_t key = 0xffffffffu, val = 0;
  if (i < nnz) {
    key = tmp_tile[i];
    val = tmp_entry[i];
  }
  warp_sort_pairs(key, val);
  int st, len;
  warp_runs(key, &st, &len);
  const int lane = threadIdx.x & 31;
  int32_t b = 0;
  if (key != 0xffffffffu && lane == st) b = atomicAdd(&cursor[key], len);
  b = __shfl_sync(0xffffffffu, b, st);
  if (key != 0xffffffffu) entries[b + (lane - st)] = val;
}

// Whole positive-list bucketing in one CTA with shared-memory counters:
// count per (chunk, 128-label tile) -> exclusive scan -> scatter.  Used when
// the tile count fits shared memory (every BASELINE config per rank).
constexpr int kPosMaxTiles = 48 * 1024;
__device__ __forceinline__ void pos_bucket_body(PosGeom g, const int32_t* __restrict__ ps,
                                                const int32_t* __restrict__ pl, int64_t nnz, int32_t T,
                                                int32_t* __restrict__ tile_ptr, uint32_t* __restrict__ entries,
                                                int32_t* status) {
  constexpr int kPer = 16;            // positives held in registers per thread per batch
  extern __shared__ int32_t cnt[];    // [T]
  __shared__ int64_t cs[65], tb[65];
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, w = tid >> 5, nw = nth >> 5;
  for (int i = tid; i <= g.k; i += nth) {
    cs[i] = g.chunk_start[i];
    tb[i] = g.tile_base[i];
  }
  const int T4 = (T + 3) / 4;
  for (int i = tid; i < T4; i += nth) reinterpret_cast<int4*>(cnt)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) carry = 0;
  __syncthreads();
  PosGeom sg = g;
  sg.chunk_start = cs;
  sg.tile_base = tb;
  // positives of this thread: i = tid + k * nth (all loads issued up front)
  const int64_t per_pass = static_cast<int64_t>(nth) * kPer;
  bool bad = false;
  for (int64_t base0 = 0; base0 < nnz; base0 += per_pass) {
    int32_t t[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int64_t i = base0 + tid + static_cast<int64_t>(k) * nth;
      t[k] = -1;
      if (i < nnz) {
        const int32_t s = ps[i];
        const int64_t local = static_cast<int64_t>(pl[i]) - g.label_offset;
        if (s < 0 || s >= g.B) bad = true;
        else if (local >= 0 && local < g.num_local) {
          int32_t r;
          t[k] = static_cast<int32_t>(pos_tile(sg, local, &r));
        }
      }
    }
    // Zipf labels pile onto a few low tiles: sort each warp's 32 tile ids and
    // issue one shared atomic per run of equal tiles (only the k rounds that
    // hold positives: nnz is often far below the 16 x 1024 slots)
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (base0 + static_cast<int64_t>(k) * nth >= nnz) break;   // block-uniform
      uint32_t key = t[k] >= 0 ? static_cast<uint32_t>(t[k]) : 0xffffffffu, val = 0;
      warp_sort_pairs(key, val);
      int st, len;
      warp_runs(key, &st, &len);
      if (key != 0xffffffffu && lane == st) atomicAdd(&cnt[key], len);
    }
  }
  if (bad) atomicOr(status, ST_BAD_SAMPLE);
  __syncthreads();
  // exclusive scan in coalesced rounds of nth counters
  for (int base = 0; base < T; base += nth) {
    const int i = base + tid;
    const int32_t v = i < T ? cnt[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int32_t s = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const int32_t excl = carry + (w > 0 ? wsum[w - 1] : 0) + x - v;
    if (i < T) {
      tile_ptr[i] = excl;
      cnt[i] = excl;   // becomes the scatter cursor
    }
    __syncthreads();
    if (tid == nth - 1) carry = excl + v;
    __syncthreads();
  }
  if (tid == 0) tile_ptr[T] = carry;
  for (int64_t base0 = 0; base0 < nnz; base0 += per_pass) {
    int32_t t[kPer];
    uint32_t e[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int64_t i = base0 + tid + static_cast<int64_t>(k) * nth;
      t[k] = -1;
      e[k] = 0;
      if (i < nnz) {
        const int32_t s = ps[i];
        const int64_t local = static_cast<int64_t>(pl[i]) - g.label_offset;
        if (s >= 0 && s < g.B && local >= 0 && local < g.num_local) {
          int32_t r;
          t[k] = static_cast<int32_t>(pos_tile(sg, local, &r));
          e[k] = (static_cast<uint32_t>(r) << 16) | static_cast<uint32_t>(s);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (base0 + static_cast<int64_t>(k) * nth >= nnz) break;   // block-uniform
      uint32_t key = t[k] >= 0 ? static_cast<uint32_t>(t[k]) : 0xffffffffu, val = e[k];
      warp_sort_pairs(key, val);
      int st, len;
      warp_runs(key, &st, &len);
      int32_t b = 0;
      if (key != 0xffffffffu && lane == st) b = atomicAdd(&cnt[key], len);
      b = __shfl_sync(0xffffffffu, b, st);
      if (key != 0xffffffffu) entries[b + (lane - st)] = val;
    }
  }
}

// Small batches: the whole step preparation in ONE launch.  Block 0 buckets
// the positives (pos_bucket_body, 1024 threads); blocks 1.. quantise X into Xq
// / Xq^T (x_prep_body, one 32x32 tile each).  The two jobs are independent.
template <int EB>
__global__ void __launch_bounds__(1024) prep_bucket_kernel(const float* __restrict__ X, int B, int Bp, int d,
                                                           uint8_t* __restrict__ xq, uint8_t* __restrict__ xqt,
                                                           PosGeom g, const int32_t* __restrict__ ps,
                                                           const int32_t* __restrict__ pl, int64_t nnz, int32_t T,
                                                           int32_t* __restrict__ tile_ptr,
                                                           uint32_t* __restrict__ entries, int32_t* status) {
  if (blockIdx.x == 0) {
    pos_bucket_body(g, ps, pl, nnz, T, tile_ptr, entries, status);
    return;
  }
  const int b = static_cast<int>(blockIdx.x) - 1, nxc = d / 32;
  x_prep_body<EB>(X, B, Bp, d, xq, xqt, status, b % nxc, b / nxc, threadIdx.x & 31, threadIdx.x >> 5, 32);
}

// fp32 G (rows x B, ld) -> backward operand format (e4m3 x scale or bf16), [rows][Bp]
template <int EB>
__global__ void g_quant_kernel(const float* __restrict__ G, int64_t ld, int64_t rows, int B, int Bp, float scale,
                               uint8_t* __restrict__ out, int32_t* status) {
  const int64_t n = rows * Bp;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / Bp;
    const int s = static_cast<int>(i - r * Bp);
    float v = 0.f;
    if (s < B) {
      v = G[r * ld + s];
      bad |= !isfinite(v);
    }
    if (EB == 1) out[i] = enc_e4m3(v * scale);
    else reinterpret_cast<uint16_t*>(out)[i] = enc_bf16(v);
  }
  if (bad) atomicOr(status, ST_NONFINITE_GRAD);
}

// ---- keyed weight dropout (head.py:138-161) ---------------------------------
// keep = u >= p with u = (mix(base + flat * gamma) >> 11) * 2^-53, i.e.
// (mix(...) >> 11) >= ceil(p * 2^53) exactly.  One thread per 32 consecutive
// elements of a row: one keep word, and (wm != null) the masked copy W * keep
// in storage format (dropped elements -> +0; the 1/(1-p) factor is applied to
// the fp32 accumulators by the consumers).
constexpr uint64_t kDropoutTag = 0xbfe79d70c7098ab2ull;   // tensor_tag("head.dropout"), head.py:43

template <int EB>
__global__ void __launch_bounds__(256) dropout_prep_kernel(const uint8_t* __restrict__ W, int64_t rows, int d,
                                                           int64_t row0_global, uint64_t base, uint64_t thr,
                                                           uint8_t* __restrict__ wm, uint32_t* __restrict__ keep) {
  const int wpr = d / 32;
  const int64_t n = rows * wpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / wpr;
    const int cw = static_cast<int>(i - r * wpr);
    const uint64_t flat0 = static_cast<uint64_t>(row0_global + r) * static_cast<uint64_t>(d) + cw * 32;
    uint32_t m = 0;
#pragma unroll 4
    for (int k = 0; k < 32; ++k)
      if ((sm64_mix(base + (flat0 + k) * kGamma) >> 11) >= thr) m |= 1u << k;
    keep[i] = m;
    if (wm) {
      const uint4* src = reinterpret_cast<const uint4*>(W + (r * d + cw * 32) * EB);
      uint4* dst = reinterpret_cast<uint4*>(wm + (r * d + cw * 32) * EB);
#pragma unroll
      for (int h = 0; h < 2 * EB; ++h) {
        uint4 v = src[h];
        uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t mask = 0;
          if constexpr (EB == 1) {
            const int e0 = h * 16 + q * 4;
#pragma unroll
            for (int b = 0; b < 4; ++b) mask |= ((m >> (e0 + b)) & 1u) ? (0xFFu << (8 * b)) : 0u;
          } else {
            const int e0 = h * 8 + q * 2;
#pragma unroll
            for (int b = 0; b < 2; ++b) mask |= ((m >> (e0 + b)) & 1u) ? (0xFFFFu << (16 * b)) : 0u;
          }
          wv[q] &= mask;
        }
        dst[h] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
  }
}

struct DropoutPlan {
  bool on = false;
  uint64_t base = 0, thr = 0;
  float scale = 1.0f;   // f32(1) / f32(1 - p): head.py:161 / :236, :243
};

static xmc_status dropout_plan(const xmc_head* h, const xmc_step_args* a, DropoutPlan* dp) {
  *dp = DropoutPlan{};
  if (!a || a->dropout_p == 0.0) return XMC_OK;
  if (!(a->dropout_p > 0.0 && a->dropout_p < 1.0))
    return fail(XMC_ERR_ARG, "dropout probability must lie in [0, 1)");
  if (!h->keep) return fail(XMC_ERR_ARG, "head created without dropout scratch (desc.dropout = 0)");
  dp->on = true;
  dp->base = sm64_base(a->seed, a->step, kDropoutTag);
  dp->thr = static_cast<uint64_t>(std::ceil(a->dropout_p * 9007199254740992.0));
  dp->scale = 1.0f / static_cast<float>(1.0 - a->dropout_p);
  return XMC_OK;
}

// keep bits (+ masked W copy when wm) for local rows [row0, row0 + rows)
static xmc_status launch_dropout_prep(const xmc_head* h, const void* W, int64_t row0, int64_t rows,
                                      const DropoutPlan& dp, uint8_t* wm, uint32_t* keep, cudaStream_t st) {
  const int D = h->desc.dim, eb = h->eb;
  const int64_t n = rows * (D / 32);
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16)));
  const uint8_t* src = W ? static_cast<const uint8_t*>(W) + row0 * D * eb : nullptr;
  const int64_t g0 = h->desc.label_offset + row0;
  if (eb == 1) dropout_prep_kernel<1><<<blocks, 256, 0, st>>>(src, rows, D, g0, dp.base, dp.thr, wm, keep);
  else dropout_prep_kernel<2><<<blocks, 256, 0, st>>>(src, rows, D, g0, dp.base, dp.thr, wm, keep);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

// ============================================================== launches
static xmc_status launch_x_prep(xmc_head* h, const float* X, int B, int Bp, cudaStream_t st) {
  dim3 grid(h->desc.dim / 32, Bp / 32), block(32, 8);
  if (h->eb == 1) x_prep_kernel<1><<<grid, block, 0, st>>>(X, B, Bp, h->desc.dim, h->xq, h->xqt, h->status);
  else x_prep_kernel<2><<<grid, block, 0, st>>>(X, B, Bp, h->desc.dim, h->xq, h->xqt, h->status);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

// Programmatic dependent launch for the fwd / bwd / reduce kernels: a kernel's
// CTAs start (barriers, TMEM, tensor maps) on SMs the previous kernel's CTAs
// vacate and then wait in griddepcontrol.wait.  Safe because every primary is
// persistent and fully co-resident (forward clusters capped at the measured
// co-resident count).  XMC_PDL=0 disables.
static bool pdl_enabled(const xmc_head* h) {
  static const bool env_on = !getenv("XMC_PDL") || atoi(getenv("XMC_PDL")) != 0;
  return env_on && h->pdl_ok;
}

// Launch with an optional L2 access-policy window: the chunk's G buffer is
// marked persisting so it survives in L2 between the forward that writes it
// and the backward that re-reads it once per d-tile, while W streams past.
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kernel)(KArgs...), int grid, int block, int smem, cudaStream_t st,
                             const xmc_head* h, size_t win_bytes, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  cfg.attrs = at;
  cfg.numAttrs = 0;
  if (h->l2_persist > 0 && win_bytes > 0) {
    const size_t nb = std::min(win_bytes, h->l2_window_max);
    at[cfg.numAttrs].id = cudaLaunchAttributeAccessPolicyWindow;
    at[cfg.numAttrs].val.accessPolicyWindow.base_ptr = h->gbuf;
    at[cfg.numAttrs].val.accessPolicyWindow.num_bytes = nb;
    at[cfg.numAttrs].val.accessPolicyWindow.hitRatio =
        std::min(1.0f, static_cast<float>(h->l2_persist) / static_cast<float>(nb));
    at[cfg.numAttrs].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[cfg.numAttrs].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++cfg.numAttrs;
  }
  if (cluster > 1) {
    at[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    at[cfg.numAttrs].val.clusterDim.x = cluster;
    at[cfg.numAttrs].val.clusterDim.y = 1;
    at[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  if (pdl_enabled(h)) {
    at[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// forward on CTA pairs (tcgen05 cta_group::2) unless XMC_FWD_PAIR=0
static bool fwd_pairs_enabled() {
  static const int v = getenv("XMC_FWD_PAIR") ? atoi(getenv("XMC_FWD_PAIR")) : 1;
  return v != 0;
}

// e4m3 batch 256 forward in the split layout instead of CTA pairs (XMC_FWD_SPLIT=1;
// the fused step always uses it)
static bool fwd_split_enabled() {
  static const int v = getenv("XMC_FWD_SPLIT") ? atoi(getenv("XMC_FWD_SPLIT")) : 0;
  return v != 0;
}

template <int EB, int BN, bool PAIR>
static xmc_status launch_fwd_t(xmc_head* h, const CUtensorMap& tw, const CUtensorMap& tx, const FwdParams& p,
                               cudaStream_t st) {
  using C = FwdCfg<EB, BN, PAIR>;
  int grid = static_cast<int>(std::min<int64_t>(h->num_sms, PAIR ? 2 * ((p.num_tiles + 1) / 2) : p.num_tiles));
  if (PAIR) grid = std::min(grid & ~1, 2 * h->fwd_max_clusters);
  if (grid <= 0) return XMC_OK;
  ProfRec pr;
  prof_begin(0, st, &pr);
  const size_t win = p.mode == 0 ? static_cast<size_t>(p.rows) * p.ld * EB : 0;
  // resident Xq (e4m3 pairs, d <= 768) unless XMC_FWD_XRES=0
  static const bool xres_on = !getenv("XMC_FWD_XRES") || atoi(getenv("XMC_FWD_XRES")) != 0;
  if constexpr (PAIR && EB == 1) {
    using CX = FwdCfg<EB, BN, true, true>;
    if (xres_on && p.d / CX::kBoxK <= CX::kXResChunks) {
      CUDA_TRY(launch_ex(xmc_fwd_kernel<EB, BN, true, false, true>, grid, CX::kThreads, CX::kSmemBytes, st, h, win, 2,
                         tw, tx, p));
      prof_end(st, &pr);
      return XMC_OK;
    }
  }
  CUDA_TRY(launch_ex(xmc_fwd_kernel<EB, BN, PAIR>, grid, C::kThreads, C::kSmemBytes, st, h, win, PAIR ? 2 : 1, tw,
                     tx, p));
  prof_end(st, &pr);
  return XMC_OK;
}

static FwdParams fwd_params(xmc_head* h, int64_t rows, int B, int mode, const int32_t* tile_ptr, void* out,
                            int64_t ld, float* stats, float logit_scale) {
  const int eb = h->eb, D = h->desc.dim;
  FwdParams p{};
  p.rows = static_cast<int32_t>(rows);
  p.B = B;
  p.d = D;
  p.num_tiles = static_cast<int32_t>(cdiv(rows, 128));
  p.mode = mode;
  p.g_fmt = eb == 1 ? FMT_E4M3 : FMT_BF16;
  p.tile_ptr = tile_ptr;
  p.entries = h->entries;
  p.out = out;
  p.ld = ld;
  p.stats = stats;
  p.logit_scale = logit_scale;
  p.status = h->status;
  static const int fdbg = getenv("XMC_DEBUG_FWD") ? atoi(getenv("XMC_DEBUG_FWD")) : 0;
  p.debug = fdbg;
  return p;
}

// rows [row0, row0+rows) of W (local), mode 0 -> G into gbuf, mode 1 -> fp32 logits
static xmc_status launch_fwd(xmc_head* h, const void* W, int64_t row0, int64_t rows, int B, int Bp, int mode,
                             const int32_t* tile_ptr, void* out, int64_t ld, float* stats, cudaStream_t st,
                             float logit_scale = 1.0f) {
  const int eb = h->eb, D = h->desc.dim;
  const bool pair = fwd_pairs_enabled() && (Bp == 128 || Bp == 256);
  CUtensorMap tw, tx;
  XMC_TRY(make_map(&tw, static_cast<const uint8_t*>(W) + row0 * D * eb, eb, D, rows, D, 128));
  XMC_TRY(make_map(&tx, h->xq, eb, D, Bp, D, std::min(pair ? Bp / 2 : Bp, 256)));
  FwdParams p = fwd_params(h, rows, B, mode, tile_ptr, out, ld, stats, logit_scale);
  if (eb == 2 && Bp == 512 && fwd_pairs_enabled()) {
    // batch 512 (bf16): two 256-sample passes of the CTA-pair kernel over the
    // same rows (double-buffered accumulators) instead of one 512-column
    // single-buffered pass; pass h writes G / logits columns [256h, 256h+256)
    for (int pass = 0; pass < 2 && pass * 256 < B; ++pass) {
      FwdParams q = p;
      q.sample0 = pass * 256;
      q.B = std::min(256, B - pass * 256);
      q.out = static_cast<uint8_t*>(out) + static_cast<size_t>(pass) * 256 * (mode == 1 ? 4 : eb);
      CUtensorMap txh;
      XMC_TRY(make_map(&txh, h->xq + static_cast<size_t>(pass) * 256 * D * eb, eb, D, 256, D, 128));
      XMC_TRY((launch_fwd_t<2, 256, true>(h, tw, txh, q, st)));
    }
    return XMC_OK;
  }
  if (eb == 1 && Bp == 256 && fwd_split_enabled() && D / 128 <= FwdCfg<1, 128, false, true>::kXResChunks) {
    // split layout (XMC_FWD_SPLIT=1): single-CTA tcgen05, CTA pair = sample halves
    using CS = FwdCfg<1, 128, false, true>;
    CUtensorMap txs;
    XMC_TRY(make_map(&txs, h->xq, eb, D, Bp, D, 128));
    const int grid = static_cast<int>(std::min<int64_t>(h->num_sms & ~1, 2 * p.num_tiles));
    const size_t win = mode == 0 ? static_cast<size_t>(rows) * ld * eb : 0;
    ProfRec pr;
    prof_begin(0, st, &pr);
    CUDA_TRY(launch_ex(xmc_fwd_kernel<1, 128, false, false, true>, grid, CS::kThreads, CS::kSmemBytes, st, h, win, 1,
                       tw, txs, p));
    prof_end(st, &pr);
    return XMC_OK;
  }
  if (eb == 1) {
    if (Bp == 128) return pair ? launch_fwd_t<1, 128, true>(h, tw, tx, p, st) : launch_fwd_t<1, 128, false>(h, tw, tx, p, st);
    if (Bp == 256) return pair ? launch_fwd_t<1, 256, true>(h, tw, tx, p, st) : launch_fwd_t<1, 256, false>(h, tw, tx, p, st);
  } else {
    if (Bp == 64) return launch_fwd_t<2, 64, false>(h, tw, tx, p, st);
    if (Bp == 128) return pair ? launch_fwd_t<2, 128, true>(h, tw, tx, p, st) : launch_fwd_t<2, 128, false>(h, tw, tx, p, st);
    if (Bp == 256) return pair ? launch_fwd_t<2, 256, true>(h, tw, tx, p, st) : launch_fwd_t<2, 256, false>(h, tw, tx, p, st);
    if (Bp == 512) return launch_fwd_t<2, 512, false>(h, tw, tx, p, st);
  }
  return fail(XMC_ERR_UNSUPPORTED, "no forward kernel for padded batch %d", Bp);
}

template <int EB, bool XR, int KC>
static xmc_status launch_bwd_t(xmc_head* h, int R, const CUtensorMap& tw, const CUtensorMap& tg,
                               const CUtensorMap& tx, const CUtensorMap& tws, const BwdParams& p, size_t g_bytes,
                               cudaStream_t st) {
  constexpr int sm = BwdCfg<EB, XR, KC>::kSmemBytes;
  const int cluster = p.gcl;
  const int grid = R * h->dtiles;
  ProfRec pr;
  prof_begin(1, st, &pr);
  const int ce = p.comp ? h->desc.comp_bytes : 0;
  if (p.adam_m != nullptr) {
    if constexpr (XR || EB == 2) {
      cudaFuncSetAttribute(xmc_bwd_kernel<EB, XR, KC, 4, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           sm);
      CUDA_TRY(launch_ex(xmc_bwd_kernel<EB, XR, KC, 4, false, true>, grid, kBwdThreads, sm, st, h, g_bytes, cluster,
                         tw, tg, tx, tws, p));
      prof_end(st, &pr);
      return XMC_OK;
    }
  }
  if (ce == 2)
    CUDA_TRY(launch_ex(xmc_bwd_kernel<EB, XR, KC, 2>, grid, kBwdThreads, sm, st, h, g_bytes, cluster, tw, tg, tx, tws,
                       p));
  else if (ce == 4)
    CUDA_TRY(launch_ex(xmc_bwd_kernel<EB, XR, KC, 4>, grid, kBwdThreads, sm, st, h, g_bytes, cluster, tw, tg, tx, tws,
                       p));
#ifdef XMC_TRACE_FAST
  else if (p.rounding == ROUND_SR_FAST && p.keep == nullptr && p.debug == 0)
#else
  else if (p.rounding == ROUND_SR_FAST && p.keep == nullptr && p.trace == nullptr && p.debug == 0)
#endif
    CUDA_TRY(launch_ex(xmc_bwd_kernel<EB, XR, KC, 0, true>, grid, kBwdThreads, sm, st, h, g_bytes, cluster, tw, tg, tx,
                       tws, p));
  else
    CUDA_TRY(launch_ex(xmc_bwd_kernel<EB, XR, KC, 0>, grid, kBwdThreads, sm, st, h, g_bytes, cluster, tw, tg, tx, tws,
                       p));
  prof_end(st, &pr);
  return XMC_OK;
}

// one bwd pass over local rows [row0, row0+rows), G from gbuf; grad_X partials
// accumulate into the [R][d][Bp] workspace (zeroed by the caller per step)
struct BwdLaunch {
  CUtensorMap tw, tg, tx, tws;
  BwdParams p;
  int R;
  size_t gb;
};

static xmc_status setup_bwd(xmc_head* h, void* W, void* comp, int64_t row0, int64_t rows, int Bp, bool update,
                            int gx_kc0, int gx_kc_count, bool gx_overwrite, const xmc_step_args* a,
                            const uint32_t* keep, float drop_scale, BwdLaunch* L) {
  const int eb = h->eb, D = h->desc.dim;
  const int box_k = 128 / eb;
  CUtensorMap &tw = L->tw, &tg = L->tg, &tx = L->tx, &tws = L->tws;
  XMC_TRY(make_map(&tw, static_cast<uint8_t*>(W) + row0 * D * eb, eb, D, rows, D, 128));
  XMC_TRY(make_map(&tws, static_cast<uint8_t*>(W) + row0 * D * eb, eb, D, rows, D, 32));
  const int64_t tiles = cdiv(rows, 128);
  const int R = static_cast<int>(std::min<int64_t>(h->R, tiles));
  // clusters span d-tiles of one row group, so every R keeps them on the same
  // label tiles; G sharing needs the resident-Xq^T layout (not bf16 batch 512)
  const int gcl = (eb == 2 && Bp == 512) ? 1 : h->gcl;
  XMC_TRY(make_map(&tg, h->gbuf, eb, Bp, rows, Bp, gcl > 1 ? 32 : 128));
  XMC_TRY(make_map(&tx, h->xqt, eb, Bp, D, Bp, 128));
  BwdParams& p = L->p;
  p = BwdParams{};
  p.rows = static_cast<int32_t>(rows);
  p.d = D;
  p.num_tiles = static_cast<int32_t>(tiles);
  p.dtiles = h->dtiles;
  p.kc_count = Bp / box_k;
  p.do_update = update ? 1 : 0;
  p.gx_kc0 = gx_kc0;
  p.gx_kc_count = gx_kc_count;
  p.W = static_cast<uint8_t*>(W) + row0 * D * eb;
  const int64_t crows = comp ? std::min<int64_t>(rows, std::max<int64_t>(0, h->comp_rows - row0)) : 0;
  p.comp = crows > 0 ? static_cast<uint8_t*>(comp) + row0 * D * h->desc.comp_bytes : nullptr;
  p.comp_rows = static_cast<int32_t>(crows);
  p.row0_global = h->desc.label_offset + row0;
  p.lr = a ? a->lr : 0.f;
  p.wd = a ? a->weight_decay : 0.f;
  p.dw_scale = eb == 1 ? (1.0f / 256.0f) : 1.0f;
  p.rounding = a ? a->rounding : 0;
  p.rng_base = a ? sm64_base(a->seed, a->step, a->tensor_id) : 0;
  p.sr_bits = a ? a->sr_bits : 0;
  p.gx_ws = h->gx_ws;
  p.gx_ld = Bp;
  p.gx_accumulate = gx_overwrite ? 0 : 1;
  static const int dbg = getenv("XMC_DEBUG_BWD") ? atoi(getenv("XMC_DEBUG_BWD")) : 0;
  p.debug = dbg;
  p.gcl = gcl;
  if (h->adam.m && update) {
    p.adam_m = h->adam.m + row0 * D;
    p.adam_v = h->adam.v + row0 * D;
    p.b1 = h->adam.b1;
    p.b2 = h->adam.b2;
    p.omb1 = h->adam.omb1;
    p.omb2 = h->adam.omb2;
    p.bc1 = h->adam.bc1;
    p.bc2 = h->adam.bc2;
    p.eps = h->adam.eps;
  }
  static const int poln = getenv("XMC_POL_NORMAL") ? atoi(getenv("XMC_POL_NORMAL")) : 0;
  p.pol_normal = poln;
  p.trace = trace_buf();
  p.keep = keep;
  p.drop_scale = drop_scale;
  p.status = h->status;
  L->R = R;
  L->gb = static_cast<size_t>(rows) * Bp * eb;
  return XMC_OK;
}

static xmc_status launch_bwd(xmc_head* h, void* W, void* comp, int64_t row0, int64_t rows, int Bp, bool update,
                             int gx_kc0, int gx_kc_count, bool gx_overwrite, const xmc_step_args* a,
                             cudaStream_t st, const uint32_t* keep = nullptr, float drop_scale = 1.0f) {
  BwdLaunch L;
  XMC_TRY(setup_bwd(h, W, comp, row0, rows, Bp, update, gx_kc0, gx_kc_count, gx_overwrite, a, keep, drop_scale, &L));
  const int eb = h->eb, R = L.R;
  const size_t gb = L.gb;
  const CUtensorMap &tw = L.tw, &tg = L.tg, &tx = L.tx, &tws = L.tws;
  const BwdParams& p = L.p;
  if (eb == 1) {
    if (Bp == 128) return launch_bwd_t<1, true, 1>(h, R, tw, tg, tx, tws, p, gb, st);
    if (Bp == 256) return launch_bwd_t<1, true, 2>(h, R, tw, tg, tx, tws, p, gb, st);
  } else {
    if (Bp == 64) return launch_bwd_t<2, true, 1>(h, R, tw, tg, tx, tws, p, gb, st);
    if (Bp == 128) return launch_bwd_t<2, true, 2>(h, R, tw, tg, tx, tws, p, gb, st);
    if (Bp == 256) return launch_bwd_t<2, true, 4>(h, R, tw, tg, tx, tws, p, gb, st);
    if (Bp == 512) return launch_bwd_t<2, false, 8>(h, R, tw, tg, tx, tws, p, gb, st);
  }
  return fail(XMC_ERR_UNSUPPORTED, "no backward kernel for padded batch %d", Bp);
}

// grad_X partials + update for one chunk whose G is in gbuf (Bp = 512 takes two passes)
static xmc_status run_backward(xmc_head* h, void* W, void* comp, int64_t row0, int64_t rows, int Bp, bool gx,
                               bool update, bool gx_overwrite, const xmc_step_args* a, cudaStream_t st) {
  const int kcs = Bp * h->eb / 128;
  const int per = 256 * h->eb / 128;   // k-chunks whose grad_X columns fit 256 TMEM columns
  if (!gx) return launch_bwd(h, W, comp, row0, rows, Bp, update, 0, 0, false, a, st);
  // passes over grad_X column groups; the update rides on the LAST pass so
  // every grad_X pass reads the pre-update weights (head.py:290-291)
  const int groups = (kcs + per - 1) / per;
  for (int gi = groups - 1; gi >= 0; --gi) {
    const int kc0 = gi * per;
    const int cnt = std::min(per, kcs - kc0);
    XMC_TRY(launch_bwd(h, W, comp, row0, rows, Bp, update && gi == 0, kc0, cnt, gx_overwrite, a, st));
  }
  return XMC_OK;
}

// ---- fused step (XMC_FUSED=1; kernel and measurements: xmc_step_kernel) ----
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// the fused step runs the SR_FAST e4m3 batch-256 step without compensation,
// dropout, Adam-style moments or measurement knobs (XMC_FUSED=0 turns it off)
static bool fused_step_ok(const xmc_head* h, void* comp, int Bp, const xmc_step_args* a) {
  static const int on = env_int("XMC_FUSED", 0);
  return on && h->eb == 1 && Bp == 256 && comp == nullptr && h->adam.m == nullptr && a &&
         a->rounding == ROUND_SR_FAST && h->gcl == 1 && h->desc.dim / 128 <= FwdCfg<1, 128, false, true>::kXResChunks &&
         !getenv("XMC_DEBUG_BWD") && !getenv("XMC_DEBUG_FWD") && trace_buf() == nullptr &&
         h->num_sms >= 2 * h->dtiles + 2;
}

// CTAs the fused step gives the forward / backward (R backward CTAs per d-tile)
static void fused_split(const xmc_head* h, int64_t tiles, int* nfwd, int* R) {
  int f = env_int("XMC_FUSED_FWD", 34) & ~1;
  f = std::max(2, std::min(f, h->num_sms - h->dtiles));
  *R = static_cast<int>(std::min<int64_t>((h->num_sms - f) / h->dtiles, tiles));
  *nfwd = static_cast<int>(std::min<int64_t>(f, 2 * tiles));
}

static xmc_status launch_fused(xmc_head* h, void* W, int64_t row0, int64_t rows, int B, int Bp,
                               const int32_t* tile_ptr, float* stats, bool gx_overwrite, const xmc_step_args* a,
                               cudaStream_t st) {
  const int eb = h->eb, D = h->desc.dim;
  const int64_t tiles = cdiv(rows, 128);
  int nfwd, R;
  fused_split(h, tiles, &nfwd, &R);
  const int ring = static_cast<int>(std::min<int64_t>(std::max(1, env_int("XMC_RING", 256)), tiles));
  BwdLaunch L;
  XMC_TRY(setup_bwd(h, W, nullptr, row0, rows, Bp, true, 0, Bp / 128, gx_overwrite, a, nullptr, 1.0f, &L));
  XMC_TRY(make_map(&L.tg, h->gbuf, eb, Bp, std::min<int64_t>(static_cast<int64_t>(ring) * 128, rows), Bp, 128));
  L.p.ring_tiles = ring;
  L.p.ready_target = 2 * FwdCfg<1, 128, false, true>::kEpiWarps;
  L.p.ready = h->ring_ready;
  L.p.consumed = h->ring_consumed;
  CUtensorMap tw, tx;
  XMC_TRY(make_map(&tw, static_cast<const uint8_t*>(W) + row0 * D * eb, eb, D, rows, D, 128));
  XMC_TRY(make_map(&tx, h->xq, eb, D, Bp, D, 128));
  FwdParams fp = fwd_params(h, rows, B, 0, tile_ptr, h->gbuf, Bp, stats, 1.0f);
  fp.ring_tiles = ring;
  fp.consumed_target = h->dtiles;
  fp.ready = h->ring_ready;
  fp.consumed = h->ring_consumed;
  CUDA_TRY(cudaMemsetAsync(h->ring_ready, 0, static_cast<size_t>(2) * (cdiv(h->max_chunk_rows, 128) + 1) * 4, st));
  ProfRec pr;
  prof_begin(1, st, &pr);
  CUDA_TRY(launch_ex(xmc_step_kernel<2>, nfwd + R * h->dtiles, kBwdThreads, kStepSmem, st, h, 0, 1, tw, tx, L.tw,
                     L.tg, L.tx, L.tws, fp, L.p, nfwd));
  prof_end(st, &pr);
  return XMC_OK;
}

// acc[s][c] (+)= scale * sum_r ws[r][c][s]  -- one deterministic reduction per step
static xmc_status reduce_gx(xmc_head* h, int B, int Bp, float* acc, bool accumulate, cudaStream_t st,
                            float scale = 1.0f) {
  const int D = h->desc.dim;
  dim3 g(D / 32, (Bp + 31) / 32), b(32, 32);
  if (h->peer && h->peer->connected && !accumulate) {
    // fused local reduction + node all-reduce (replaces reduce + ncclAllReduce)
    xmc_peer* pg = h->peer;
    if (D != pg->dim || Bp > pg->max_bp) return fail(XMC_ERR_SHAPE, "peer group built for another dim / batch");
    PeerArgs pa{};
    for (int r = 0; r < pg->world; ++r) pa.base[r] = static_cast<uint8_t*>(pg->base[r]);
    pa.rank = pg->rank;
    pa.world = pg->world;
    pa.nblocks = pg->nblocks;
    pa.flag_off = static_cast<int64_t>(pg->flag_off);
    pa.epoch = ++pg->epoch;
    pa.status = h->status;
    cudaLaunchConfig_t pc{};
    pc.gridDim = g;
    pc.blockDim = b;
    pc.stream = st;
    cudaLaunchAttribute pat[1];
    pat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pat[0].val.programmaticStreamSerializationAllowed = 1;
    pc.attrs = pat;
    pc.numAttrs = pdl_enabled(h) ? 1 : 0;
    CUDA_TRY(cudaLaunchKernelEx(&pc, gx_reduce_peer_kernel, static_cast<const float*>(h->gx_ws), h->R_step, D, Bp,
                                B, (h->eb == 1 ? (1.0f / 256.0f) : 1.0f) * scale, acc, pa));
    CUDA_TRY(cudaGetLastError());
    return XMC_OK;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(h) ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, gx_reduce_kernel, static_cast<const float*>(h->gx_ws), h->R_step, D, Bp, B,
                              (h->eb == 1 ? (1.0f / 256.0f) : 1.0f) * scale, accumulate ? 1 : 0, acc));
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

static xmc_status zero_gx_ws(xmc_head* h, int Bp, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(h->gx_ws, 0, (size_t)h->R * h->desc.dim * Bp * 4, st));
  return XMC_OK;
}

static xmc_status check_args(const xmc_step_args* a) {
  if (!a) return fail(XMC_ERR_ARG, "null step args");
  if (!(a->lr > 0.0f)) return fail(XMC_ERR_ARG, "lr must be positive");
  if (!(a->weight_decay >= 0.0f)) return fail(XMC_ERR_ARG, "weight_decay must be non-negative");
  if (a->rounding < 0 || a->rounding > 2) return fail(XMC_ERR_ARG, "unknown rounding mode %d", a->rounding);
  if (a->sr_bits < 0 || a->sr_bits > 1) return fail(XMC_ERR_ARG, "unknown SR bit generator %d", a->sr_bits);
  return XMC_OK;
}

// Xq / Xq^T and the positive buckets of one step.  Small batches: x_prep +
// one single-CTA bucketing kernel; otherwise x_prep fused with the counting
// pass, then scan and scatter (the scan re-zeroes the counters).
static xmc_status prepare_step(xmc_head* h, const float* X, int Bp, const int32_t* ps, const int32_t* pl,
                               int64_t nnz, int B, cudaStream_t st) {
  if (nnz > h->desc.max_positives)
    return fail(XMC_ERR_CAPACITY, "%lld positives exceed workspace capacity %lld", (long long)nnz,
                (long long)h->desc.max_positives);
  PosGeom g{h->chunk_dev, h->chunk_dev + h->chunks.size() + 1, static_cast<int32_t>(h->chunks.size()),
            h->desc.label_offset, h->desc.num_labels_local, B};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prep_bucket_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPosMaxTiles * 4);
    cudaFuncSetAttribute(prep_bucket_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPosMaxTiles * 4);
    cudaFuncSetAttribute(pos_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPosMaxTiles * 4);
    attr = true;
  }
  const int32_t T = static_cast<int32_t>(h->total_tiles);
  if (T > kPosMaxTiles || h->chunks.size() > 64)
    return fail(XMC_ERR_UNSUPPORTED, "%d label tiles per rank exceed the bucketing capacity %d; use more ranks", T,
                kPosMaxTiles);
  if (nnz <= 2048) {
    // tiny batches: one launch (block 0 buckets in shared memory, the rest prepare Xq)
    const int nblk = 1 + (h->desc.dim / 32) * (Bp / 32);
    if (h->eb == 1)
      prep_bucket_kernel<1><<<nblk, 1024, T * 4, st>>>(X, B, Bp, h->desc.dim, h->xq, h->xqt, g, ps, pl, nnz, T,
                                                       h->tile_ptr, h->entries, h->status);
    else
      prep_bucket_kernel<2><<<nblk, 1024, T * 4, st>>>(X, B, Bp, h->desc.dim, h->xq, h->xqt, g, ps, pl, nnz, T,
                                                       h->tile_ptr, h->entries, h->status);
    CUDA_TRY(cudaGetLastError());
    return XMC_OK;
  }
  const int blocks = static_cast<int>(cdiv(nnz, 256));
  const int nx = (h->desc.dim / 32) * (Bp / 32);
  if (h->eb == 1)
    prep_count_kernel<1><<<nx + blocks, 256, 0, st>>>(X, B, Bp, h->desc.dim, h->xq, h->xqt, nx, g, ps, pl, nnz,
                                                      h->tile_cnt, h->tmp_tile, h->tmp_entry, h->status);
  else
    prep_count_kernel<2><<<nx + blocks, 256, 0, st>>>(X, B, Bp, h->desc.dim, h->xq, h->xqt, nx, g, ps, pl, nnz,
                                                      h->tile_cnt, h->tmp_tile, h->tmp_entry, h->status);
  CUDA_TRY(cudaGetLastError());
  pos_scan_kernel<<<1, 1024, T * 4, st>>>(h->tile_cnt, h->tile_ptr, h->tile_cur, T);
  CUDA_TRY(cudaGetLastError());
  pos_scatter_kernel<<<blocks, 256, 0, st>>>(nnz, h->tmp_tile, h->tmp_entry, h->tile_cur, h->entries);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

static xmc_status read_status(xmc_head* h, cudaStream_t st, bool clear) {
  int32_t s = 0;
  CUDA_TRY(cudaMemcpyAsync(&s, h->status, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (s != 0 && clear) CUDA_TRY(cudaMemsetAsync(h->status, 0, 4, st));
  if (s & ST_NONFINITE_X) return fail(XMC_ERR_NONFINITE, "non-finite input to rounding operation");
  if (s & ST_BAD_SAMPLE) return fail(XMC_ERR_INDEX, "positive sample index out of range");
  if (s & ST_LABEL_OUTSIDE) return fail(XMC_ERR_LABEL, "label outside chunk range");
  if (s & ST_NONFINITE_GRAD) return fail(XMC_ERR_NONFINITE, "non-finite values in fused scratch block");
  if (s & ST_RING_TIMEOUT) return fail(XMC_ERR_CUDA, "fused step: a G ring flag timed out (CTAs not co-resident)");
  if (s & ST_PEER_TIMEOUT) return fail(XMC_ERR_CUDA, "peer grad_X all-reduce: a peer's tile never arrived");
  return XMC_OK;
}

extern "C" xmc_status xmc_head_check(xmc_head_t h, void* stream) {
  if (!h) return fail(XMC_ERR_ARG, "null handle");
  return read_status(h, static_cast<cudaStream_t>(stream), true);
}

extern "C" xmc_status xmc_head_step(xmc_head_t h, void* W, const float* X, int32_t B, const int32_t* pos_sample,
                                    const int32_t* pos_label, int64_t nnz, const xmc_step_args* args,
                                    float* grad_x, float* stats, void* stream) {
  return xmc_head_step_kahan(h, W, nullptr, X, B, pos_sample, pos_label, nnz, args, grad_x, stats, stream);
}

extern "C" xmc_status xmc_head_step_kahan(xmc_head_t h, void* W, void* comp, const float* X, int32_t B,
                                          const int32_t* pos_sample, const int32_t* pos_label, int64_t nnz,
                                          const xmc_step_args* args, float* grad_x, float* stats, void* stream) {
  if (!h || !W || !X || !grad_x) return fail(XMC_ERR_ARG, "null argument");
  if (comp && h->desc.comp_bytes != 2 && h->desc.comp_bytes != 4)
    return fail(XMC_ERR_ARG, "head created without a Kahan compensation format (comp_bytes 2 or 4)");
  XMC_TRY(check_args(args));
  if (B < 1 || B > h->desc.max_batch) return fail(XMC_ERR_SHAPE, "batch %d outside [1, %d]", B, h->desc.max_batch);
  if (nnz < 0 || (nnz > 0 && (!pos_sample || !pos_label))) return fail(XMC_ERR_ARG, "bad positives");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int Bp = padded_batch(h->eb, B);
  XMC_TRY(prepare_step(h, X, Bp, pos_sample, pos_label, nnz, B, st));
  DropoutPlan dp;
  XMC_TRY(dropout_plan(h, args, &dp));
  const bool fused = !dp.on && fused_step_ok(h, comp, Bp, args);
  // grad_X partial slots of this step (the fused step gives the backward fewer CTAs)
  h->R_step = h->R;
  if (fused) {
    int nf, Rf;
    fused_split(h, INT64_MAX / 4, &nf, &Rf);
    h->R_step = Rf;
  }
  // the first chunk overwrites every partial slot unless it has fewer tiles
  // than slots; later chunks accumulate
  const bool first_covers = !h->chunks.empty() && cdiv(h->chunks[0].second - h->chunks[0].first, 128) >= h->R_step;
  if (!first_covers) XMC_TRY(zero_gx_ws(h, Bp, st));
  if (stats) CUDA_TRY(cudaMemsetAsync(stats, 0, 8, st));
  for (size_t c = 0; c < h->chunks.size(); ++c) {
    const int64_t r0 = h->chunks[c].first, rows = h->chunks[c].second - h->chunks[c].first;
    const int32_t* tp = h->tile_ptr + h->tile_base[c];
    if (fused) {
      XMC_TRY(launch_fused(h, W, r0, rows, B, Bp, tp, stats, first_covers && c == 0, args, st));
      continue;
    }
    if (!dp.on) {
      XMC_TRY(launch_fwd(h, W, r0, rows, B, Bp, 0, tp, h->gbuf, Bp, stats, st));
      XMC_TRY(run_backward(h, W, comp, r0, rows, Bp, true, true, first_covers && c == 0, args, st));
      continue;
    }
    // keyed dropout (head.py:155-161, 239-242): logits and grad_X read the
    // masked chunk copy W*keep (1/(1-p) applied to the fp32 accumulators);
    // the update pass reads W and scales kept dW by 1/(1-p)
    XMC_TRY(launch_dropout_prep(h, W, r0, rows, dp, h->wm, h->keep, st));
    XMC_TRY(launch_fwd(h, h->wm, 0, rows, B, Bp, 0, tp, h->gbuf, Bp, stats, st, dp.scale));
    XMC_TRY(run_backward(h, h->wm, nullptr, 0, rows, Bp, true, false, first_covers && c == 0, args, st));
    XMC_TRY(launch_bwd(h, W, comp, r0, rows, Bp, true, 0, 0, false, args, st, h->keep, dp.scale));
  }
  return reduce_gx(h, B, Bp, grad_x, false, st, dp.scale);
}

// Adam-style head step: head_update with the chunk gradient fed to
// kahan_adamw_step (optimizers.py:112-137) in the fused backward epilogue.
extern "C" xmc_status xmc_head_step_adamw(xmc_head_t h, void* W, float* comp, float* m, float* v, const float* X,
                                          int32_t B, const int32_t* pos_sample, const int32_t* pos_label,
                                          int64_t nnz, const xmc_adamw_args* adam, const xmc_step_args* args,
                                          float* grad_x, float* stats, void* stream) {
  if (!h || !comp || !m || !v || !adam || !args) return fail(XMC_ERR_ARG, "null argument");
  if (h->desc.comp_bytes != 4 || h->comp_rows != h->desc.num_labels_local)
    return fail(XMC_ERR_ARG, "the Adam-style head needs an fp32 compensation for every label (comp_bytes 4)");
  if (!(adam->beta1 >= 0.0 && adam->beta1 < 1.0 && adam->beta2 >= 0.0 && adam->beta2 < 1.0))
    return fail(XMC_ERR_ARG, "betas must lie in [0, 1)");
  if (!(adam->eps > 0.0f)) return fail(XMC_ERR_ARG, "eps must be positive");
  if (adam->t < 1) return fail(XMC_ERR_ARG, "step index t must be >= 1");
  xmc_step_args a = *args;
  a.lr = adam->lr;
  a.weight_decay = adam->weight_decay;
  a.rounding = 0;   // kahan_add rounds to nearest
  h->adam.m = m;
  h->adam.v = v;
  h->adam.b1 = static_cast<float>(adam->beta1);
  h->adam.b2 = static_cast<float>(adam->beta2);
  h->adam.omb1 = 1.0f - h->adam.b1;
  h->adam.omb2 = 1.0f - h->adam.b2;
  h->adam.bc1 = static_cast<float>(1.0 - std::pow(adam->beta1, static_cast<double>(adam->t)));
  h->adam.bc2 = static_cast<float>(1.0 - std::pow(adam->beta2, static_cast<double>(adam->t)));
  h->adam.eps = adam->eps;
  const xmc_status st = xmc_head_step_kahan(h, W, comp, X, B, pos_sample, pos_label, nnz, &a, grad_x, stats, stream);
  h->adam.m = nullptr;
  h->adam.v = nullptr;
  return st;
}

// ---- streaming top-k scoring ------------------------------------
// Merge the per-(CTA, sub-partition) candidate lists of one sample into its
// top-k, ordered by (score desc, label asc) (metrics.py:38-47).  One CTA per sample.
__global__ void __launch_bounds__(256) topk_merge_kernel(const float* __restrict__ cs, const int32_t* __restrict__ cl,
                                                         int nslots, int k, float* __restrict__ out_s,
                                                         int64_t* __restrict__ out_l) {
  __shared__ float ss[256 * kTopK];
  __shared__ int32_t sl[256 * kTopK];
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  float ls[kTopK];
  int32_t ll[kTopK];
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    ls[i] = -INFINITY;
    ll[i] = 0x7fffffff;
  }
  const int n = nslots * kTopK;
  const float* a = cs + static_cast<size_t>(s) * n;
  const int32_t* b = cl + static_cast<size_t>(s) * n;
  for (int i = tid; i < n; i += blockDim.x) topk_insert(ls, ll, a[i], b[i]);
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    ss[tid * kTopK + i] = ls[i];
    sl[tid * kTopK + i] = ll[i];
  }
  __syncthreads();
  if (tid >= 32) return;
  // warp 0: lane l folds the lists of threads l, l+32, ... into its own
  for (int t = tid + 32; t < blockDim.x; t += 32)
    for (int i = 0; i < kTopK; ++i) topk_insert(ls, ll, ss[t * kTopK + i], sl[t * kTopK + i]);
  // k rounds of a warp-wide best-of-heads selection
  int head = 0;
  for (int r = 0; r < k; ++r) {
    float v = -INFINITY;
    int32_t lv = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kTopK; ++i)
      if (i == head) {
        v = ls[i];
        lv = ll[i];
      }
    float bv = v;
    int32_t bl = lv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (topk_better(ov, ol, bv, bl)) {
        bv = ov;
        bl = ol;
      }
    }
    if (v == bv && lv == bl) ++head;   // labels are unique: exactly one lane owns the winner
    if (lane == 0) {
      out_s[static_cast<size_t>(s) * k + r] = bv;
      out_l[static_cast<size_t>(s) * k + r] = bl;
    }
  }
}

// e4m3 batch-256 scoring on CTA pairs with resident Xq (the training forward's
// mainloop), unless XMC_TOPK_PAIR=0
static bool topk_pairs() {
  static const int v = getenv("XMC_TOPK_PAIR") ? atoi(getenv("XMC_TOPK_PAIR")) : 1;
  return v != 0;
}
static int topk_grid(const xmc_head* h, int64_t tiles, int eb, int bn, int D) {
  if (topk_pairs() && eb == 1 && bn == 256 && D / 128 <= FwdCfg<1, 256, true, true>::kXResChunks)
    return static_cast<int>(std::min<int64_t>(2 * h->fwd_max_clusters, 2 * ((tiles + 1) / 2)));
  return static_cast<int>(std::min<int64_t>(h->num_sms, tiles));
}

template <int EB, int BN>
static xmc_status launch_topk_t(xmc_head* h, const CUtensorMap& tw, const CUtensorMap& tx, const FwdParams& p,
                                cudaStream_t st) {
  using C = FwdCfg<EB, BN, false>;
  const int grid = topk_grid(h, p.num_tiles, EB, BN, p.d);
  if constexpr (EB == 1 && BN == 256) {
    if (topk_pairs() && p.d / 128 <= FwdCfg<1, 256, true, true>::kXResChunks) {
      using CP = FwdCfg<1, 256, true, true>;
      CUtensorMap txp;   // each CTA of a pair stages its 128 samples
      XMC_TRY(make_map(&txp, h->xq_topk, 1, p.d, 256, p.d, 128));
      CUDA_TRY(launch_ex(xmc_fwd_kernel<1, 256, true, true, true>, grid, CP::kThreads, CP::kSmemBytes, st, h, 0, 2,
                         tw, txp, p));
      return XMC_OK;
    }
  }
  CUDA_TRY(launch_ex(xmc_fwd_kernel<EB, BN, false, true>, grid, C::kThreads, C::kSmemBytes, st, h, 0, 1, tw, tx, p));
  return XMC_OK;
}

extern "C" xmc_status xmc_head_topk(xmc_head_t h, const void* W, const float* X, int32_t B, int32_t k,
                                    float* top_scores, int64_t* top_labels, void* stream) {
  if (!h || !W || !X || !top_scores || !top_labels) return fail(XMC_ERR_ARG, "null argument");
  if (B < 1 || B > h->desc.max_batch) return fail(XMC_ERR_SHAPE, "batch %d outside [1, %d]", B, h->desc.max_batch);
  if (k < 1 || k > h->desc.num_labels_local) return fail(XMC_ERR_ARG, "k must lie in [1, %lld]",
                                                         (long long)h->desc.num_labels_local);
  if (k > kTopK) return fail(XMC_ERR_UNSUPPORTED, "fused top-k supports k <= %d (got %d)", kTopK, k);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int eb = h->eb, D = h->desc.dim, Bp = padded_batch(eb, B);
  const int64_t rows = h->desc.num_labels_local;
  XMC_TRY(launch_x_prep(h, X, B, Bp, st));
  CUtensorMap tw;
  XMC_TRY(make_map(&tw, static_cast<const uint8_t*>(W), eb, D, rows, D, 128));
  const int bn0 = std::min(Bp, 256);
  const int nslots = 4 * topk_grid(h, cdiv(rows, 128), eb, bn0, D);
  // Bp = 512 runs as two N = 256 launches over the sample halves (the 512-wide
  // epilogue would need twice the candidate registers)
  const int bn = std::min(Bp, 256);
  for (int s0 = 0; s0 < B; s0 += bn) {
    CUtensorMap tx;
    XMC_TRY(make_map(&tx, h->xq + static_cast<size_t>(s0) * D * eb, eb, D, bn, D, bn));
    h->xq_topk = h->xq + static_cast<size_t>(s0) * D * eb;
    FwdParams p{};
    p.rows = static_cast<int32_t>(rows);
    p.B = std::min(bn, B - s0);
    p.d = D;
    p.num_tiles = static_cast<int32_t>(cdiv(rows, 128));
    p.mode = 2;
    p.logit_scale = 1.0f;
    p.cand_s = h->cand_s + static_cast<size_t>(s0) * nslots * kTopK;
    p.cand_l = h->cand_l + static_cast<size_t>(s0) * nslots * kTopK;
    p.label0 = h->desc.label_offset;
    p.status = h->status;
    xmc_status r = XMC_ERR_UNSUPPORTED;
    if (eb == 1) {
      if (bn == 128) r = launch_topk_t<1, 128>(h, tw, tx, p, st);
      else if (bn == 256) r = launch_topk_t<1, 256>(h, tw, tx, p, st);
    } else {
      if (bn == 64) r = launch_topk_t<2, 64>(h, tw, tx, p, st);
      else if (bn == 128) r = launch_topk_t<2, 128>(h, tw, tx, p, st);
      else if (bn == 256) r = launch_topk_t<2, 256>(h, tw, tx, p, st);
    }
    if (r != XMC_OK) return r == XMC_ERR_UNSUPPORTED ? fail(r, "no top-k kernel for padded batch %d", Bp) : r;
  }
  topk_merge_kernel<<<B, 256, 0, st>>>(h->cand_s, h->cand_l, nslots, k, top_scores, top_labels);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

extern "C" xmc_status xmc_head_logits(xmc_head_t h, const void* W, const float* X, int32_t B, int64_t row0,
                                      int64_t row1, float* logits, int64_t ld, const xmc_step_args* args,
                                      void* stream) {
  if (!h || !W || !X || !logits) return fail(XMC_ERR_ARG, "null argument");
  if (B < 1 || B > h->desc.max_batch) return fail(XMC_ERR_SHAPE, "batch %d outside [1, %d]", B, h->desc.max_batch);
  if (row0 < 0 || row1 > h->desc.num_labels_local || row1 <= row0) return fail(XMC_ERR_ARG, "bad row range");
  if (ld < B) return fail(XMC_ERR_ARG, "ld < B");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int Bp = padded_batch(h->eb, B);
  DropoutPlan dp;
  XMC_TRY(dropout_plan(h, args, &dp));
  XMC_TRY(launch_x_prep(h, X, B, Bp, st));
  if (!dp.on) return launch_fwd(h, W, row0, row1 - row0, B, Bp, 1, nullptr, logits, ld, nullptr, st);
  if (row1 - row0 > h->max_chunk_rows + 128) return fail(XMC_ERR_CAPACITY, "row range exceeds the dropout scratch");
  XMC_TRY(launch_dropout_prep(h, W, row0, row1 - row0, dp, h->wm, h->keep, st));
  return launch_fwd(h, h->wm, 0, row1 - row0, B, Bp, 1, nullptr, logits, ld, nullptr, st, dp.scale);
}

// standalone dropout_mask (head.py:138-152) for any column count
__global__ void dropout_mask_kernel(int64_t row0, int64_t rows, int32_t cols, uint64_t base, uint64_t thr,
                                    uint32_t* __restrict__ keep) {
  const int wpr = (cols + 31) / 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * wpr; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / wpr;
    const int c0 = static_cast<int>(i - r * wpr) * 32;
    const uint64_t flat0 = static_cast<uint64_t>(row0 + r) * static_cast<uint64_t>(cols) + c0;
    uint32_t m = 0;
    for (int k = 0; k < 32 && c0 + k < cols; ++k)
      if ((sm64_mix(base + (flat0 + k) * kGamma) >> 11) >= thr) m |= 1u << k;
    keep[i] = m;
  }
}

extern "C" xmc_status xmc_dropout_mask(int64_t row0, int64_t row1, int32_t num_cols, uint64_t seed, uint64_t step,
                                       double p, uint32_t* keep, void* stream) {
  if (!keep) return fail(XMC_ERR_ARG, "null argument");
  if (row0 < 0 || row1 < row0 || num_cols < 0) return fail(XMC_ERR_ARG, "bad row range");
  if (!(p >= 0.0 && p < 1.0)) return fail(XMC_ERR_ARG, "dropout probability must lie in [0, 1)");
  const int64_t n = (row1 - row0) * ((num_cols + 31) / 32);
  if (n == 0) return XMC_OK;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16)));
  dropout_mask_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      row0, row1 - row0, num_cols, sm64_base(seed, step, kDropoutTag),
      static_cast<uint64_t>(std::ceil(p * 9007199254740992.0)), keep);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

extern "C" xmc_status xmc_head_backward(xmc_head_t h, void* W, const float* G, int64_t ld, const float* X,
                                        int32_t B, int64_t row0, int64_t row1, float* acc, int32_t accumulate_gx,
                                        int32_t update, const xmc_step_args* args, void* stream) {
  if (!h || !W || !G || (update && !X)) return fail(XMC_ERR_ARG, "null argument");
  if (update) XMC_TRY(check_args(args));
  if (B < 1 || B > h->desc.max_batch) return fail(XMC_ERR_SHAPE, "batch %d outside [1, %d]", B, h->desc.max_batch);
  if (row0 < 0 || row1 > h->desc.num_labels_local || row1 <= row0) return fail(XMC_ERR_ARG, "bad row range");
  if (row1 - row0 > h->max_chunk_rows + 128) return fail(XMC_ERR_CAPACITY, "row range exceeds the G buffer");
  if (accumulate_gx && !acc) return fail(XMC_ERR_ARG, "null acc");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int Bp = padded_batch(h->eb, B);
  if (X) XMC_TRY(launch_x_prep(h, X, B, Bp, st));
  const int64_t rows = row1 - row0;
  const int blocks = static_cast<int>(std::min<int64_t>(cdiv(rows * Bp, 256), 4096));
  if (h->eb == 1) g_quant_kernel<1><<<blocks, 256, 0, st>>>(G, ld, rows, B, Bp, 256.0f, h->gbuf, h->status);
  else g_quant_kernel<2><<<blocks, 256, 0, st>>>(G, ld, rows, B, Bp, 1.0f, h->gbuf, h->status);
  CUDA_TRY(cudaGetLastError());
  DropoutPlan dp;
  XMC_TRY(dropout_plan(h, args, &dp));
  h->R_step = h->R;
  if (accumulate_gx) XMC_TRY(zero_gx_ws(h, Bp, st));
  if (!dp.on) {
    XMC_TRY(run_backward(h, W, nullptr, row0, rows, Bp, accumulate_gx != 0, update != 0, false, args, st));
  } else {
    XMC_TRY(launch_dropout_prep(h, W, row0, rows, dp, accumulate_gx ? h->wm : nullptr, h->keep, st));
    if (accumulate_gx) XMC_TRY(run_backward(h, h->wm, nullptr, 0, rows, Bp, true, false, false, args, st));
    if (update) XMC_TRY(launch_bwd(h, W, nullptr, row0, rows, Bp, true, 0, 0, false, args, st, h->keep, dp.scale));
  }
  if (accumulate_gx) XMC_TRY(reduce_gx(h, B, Bp, acc, true, st, dp.scale));
  return XMC_OK;
}

// ============================================================== elementwise core
static GridFmt grid_from(xmc_grid g, xmc_status* s) {
  GridFmt f{};
  if (g.exp_bits < 2 || g.exp_bits > 8 || g.man_bits < 0 || g.man_bits > 23) {
    *s = fail(XMC_ERR_ARG, "bad format e%dm%d", g.exp_bits, g.man_bits);
    return f;
  }
  const bool ext = g.extended_range < 0 ? (g.exp_bits == 4 && g.man_bits == 3) : g.extended_range != 0;
  if (ext && g.man_bits == 0) {
    *s = fail(XMC_ERR_ARG, "extended range needs at least one mantissa bit");
    return f;
  }
  const int bias = (1 << (g.exp_bits - 1)) - 1;
  f.man_bits = g.man_bits;
  f.min_normal_exp = 1 - bias;
  f.max_exp = ext ? bias + 1 : bias;
  const double top = ext ? 2.0 - std::ldexp(1.0, 1 - g.man_bits) : 2.0 - std::ldexp(1.0, -g.man_bits);
  f.max_finite = std::ldexp(top, f.max_exp);
  *s = XMC_OK;
  return f;
}

__global__ void finite_check_kernel(const float* __restrict__ x, int64_t n, int32_t* status, int32_t bit) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, bit);
}

__global__ void round_kernel(GridFmt f, const float* __restrict__ x, float* __restrict__ out, int64_t n, int mode,
                             uint64_t base, const uint64_t* __restrict__ index, const int32_t* status) {
  if (*status != 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    if (mode == 0) out[i] = grid_round_nearest(f, v);
    else out[i] = grid_round_stochastic(f, v, sm64_uniform(base, index ? index[i] : static_cast<uint64_t>(i)));
  }
}

// sgd_sr_step (optimizers.py:51-74); kahan=1 -> head-Kahan composition (A8k)
__global__ void sgd_kernel(GridFmt f, bool working_precision, float* __restrict__ w, float* __restrict__ comp,
                           const float* __restrict__ grad, int64_t n, float lr, float wd, int rounding,
                           uint64_t base, const uint64_t* __restrict__ index, const int32_t* status) {
  if (*status != 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float s = w[i];
    const float g = wd != 0.0f ? __fadd_rn(grad[i], __fmul_rn(wd, s)) : grad[i];
    const uint64_t key = index ? index[i] : static_cast<uint64_t>(i);
    if (comp == nullptr) {
      const float upd = __fsub_rn(s, __fmul_rn(lr, g));
      w[i] = rounding == 0 ? grid_round_nearest(f, upd) : grid_round_stochastic(f, upd, sm64_uniform(base, key));
    } else {
      const float v = -__fmul_rn(lr, g);
      if (working_precision) {
        w[i] = __fadd_rn(s, v);
        continue;
      }
      const float c = comp[i];
      const float y = __fsub_rn(v, c);
      const float x = __fadd_rn(s, y);
      const float t = rounding == 0 ? grid_round_nearest(f, x) : grid_round_stochastic(f, x, sm64_uniform(base, key));
      comp[i] = __fsub_rn(__fsub_rn(t, s), y);
      w[i] = t;
    }
  }
}

static int ew_blocks(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8192))); }

static int32_t* scratch_status() {
  static int32_t* p = nullptr;
  if (!p) cudaMalloc(&p, 64);
  return p;
}

static xmc_status status_to_error(int32_t s) {
  if (s & ST_NONFINITE_X) return fail(XMC_ERR_NONFINITE, "non-finite input to rounding operation");
  if (s & ST_NONFINITE_GRAD) return fail(XMC_ERR_NONFINITE, "non-finite gradient entry");
  if (s & ST_NONFINITE_MOMENTS) return fail(XMC_ERR_NONFINITE, "non-finite optimizer moments");
  return XMC_OK;
}

// run a finite check then the op; sync and report (the reference raises before writing)
static xmc_status checked_elementwise(const float* chk, int64_t n, int32_t bit, int32_t* status, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(status, 0, 4, st));
  finite_check_kernel<<<ew_blocks(n), 256, 0, st>>>(chk, n, status, bit);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

static xmc_status finish_elementwise(int32_t* status, cudaStream_t st) {
  int32_t s = 0;
  CUDA_TRY(cudaMemcpyAsync(&s, status, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return status_to_error(s);
}

extern "C" xmc_status xmc_round_nearest(xmc_grid g, const float* x, float* out, int64_t n, void* stream) {
  xmc_status s;
  const GridFmt f = grid_from(g, &s);
  XMC_TRY(s);
  if (n <= 0) return XMC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* status = scratch_status();
  XMC_TRY(checked_elementwise(x, n, ST_NONFINITE_X, status, st));
  round_kernel<<<ew_blocks(n), 256, 0, st>>>(f, x, out, n, 0, 0, nullptr, status);
  CUDA_TRY(cudaGetLastError());
  return finish_elementwise(status, st);
}

extern "C" xmc_status xmc_round_stochastic(xmc_grid g, const float* x, float* out, int64_t n, uint64_t seed,
                                           uint64_t step, uint64_t tensor_id, const uint64_t* index, void* stream) {
  xmc_status s;
  const GridFmt f = grid_from(g, &s);
  XMC_TRY(s);
  if (n <= 0) return XMC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* status = scratch_status();
  XMC_TRY(checked_elementwise(x, n, ST_NONFINITE_X, status, st));
  round_kernel<<<ew_blocks(n), 256, 0, st>>>(f, x, out, n, 1, sm64_base(seed, step, tensor_id), index, status);
  CUDA_TRY(cudaGetLastError());
  return finish_elementwise(status, st);
}

static xmc_status sgd_common(xmc_grid g, float* w, float* comp, const float* grad, int64_t n, float lr, float wd,
                             int32_t rounding, uint64_t seed, uint64_t step, uint64_t tensor_id,
                             const uint64_t* index, int32_t* status, void* stream) {
  xmc_status s;
  const GridFmt f = grid_from(g, &s);
  XMC_TRY(s);
  if (!(lr > 0.0f)) return fail(XMC_ERR_ARG, "lr must be positive");
  if (!(wd >= 0.0f)) return fail(XMC_ERR_ARG, "weight_decay must be non-negative");
  if (rounding != 0 && rounding != 1) return fail(XMC_ERR_ARG, "elementwise SGD supports nearest / exact SR");
  if (n <= 0) return XMC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* stw = status ? status : scratch_status();
  XMC_TRY(checked_elementwise(grad, n, ST_NONFINITE_GRAD, stw, st));
  const bool wp = g.exp_bits == 8 && g.man_bits == 23;
  sgd_kernel<<<ew_blocks(n), 256, 0, st>>>(f, wp, w, comp, grad, n, lr, wd, rounding, sm64_base(seed, step, tensor_id),
                                           index, stw);
  CUDA_TRY(cudaGetLastError());
  return finish_elementwise(stw, st);
}

extern "C" xmc_status xmc_sgd_sr_step(xmc_grid g, float* w, const float* grad, int64_t n, float lr, float wd,
                                      int32_t rounding, uint64_t seed, uint64_t step, uint64_t tensor_id,
                                      const uint64_t* index, int32_t* status, void* stream) {
  return sgd_common(g, w, nullptr, grad, n, lr, wd, rounding, seed, step, tensor_id, index, status, stream);
}

extern "C" xmc_status xmc_kahan_sgd_step(xmc_grid g, float* w, float* comp, const float* grad, int64_t n, float lr,
                                         float wd, int32_t rounding, uint64_t seed, uint64_t step, uint64_t tensor_id,
                                         const uint64_t* index, int32_t* status, void* stream) {
  if (!comp) return fail(XMC_ERR_ARG, "null compensation buffer");
  return sgd_common(g, w, comp, grad, n, lr, wd, rounding, seed, step, tensor_id, index, status, stream);
}

// kahan_adamw_step (optimizers.py:112-137) elementwise, every operation an
// explicitly rounded fp32 op in the reference's (numpy's) order; kahan_add
// formats.py:246-263 with RTN onto the grid.  write = 0: only flag non-finite
// moments / updates (the reference raises before the parameter changes).
struct AdamWArgs {
  float lr, b1, b2, omb1, omb2, eps, wd, bc1, bc2;
};
__device__ __forceinline__ void adamw_elem(const AdamWArgs& a, float g, float m, float v, float s, float& m1, float& v1,
                                           float& upd) {
  m1 = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));
  v1 = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(__fmul_rn(a.omb2, g), g));
  const float mhat = __fdiv_rn(m1, a.bc1);
  const float vhat = __fdiv_rn(v1, a.bc2);
  const float den = __fadd_rn(__fsqrt_rn(vhat), a.eps);
  upd = __fmul_rn(-a.lr, __fadd_rn(__fdiv_rn(mhat, den), __fmul_rn(a.wd, s)));
}
__global__ void adamw_kernel(GridFmt f, bool working_precision, AdamWArgs a, float* __restrict__ w,
                             float* __restrict__ comp, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ grad, int64_t n, int write, int32_t* status) {
  if (write && *status != 0) return;
  bool bad_mom = false, bad_upd = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float s = w[i];
    float m1, v1, upd;
    adamw_elem(a, grad[i], m[i], v[i], s, m1, v1, upd);
    if (!write) {
      bad_mom |= !isfinite(m1) || !isfinite(v1);
      bad_upd |= !isfinite(upd);
      continue;
    }
    m[i] = m1;
    v[i] = v1;
    if (working_precision) {
      w[i] = __fadd_rn(s, upd);
      continue;
    }
    const float c = comp[i];
    const float y = __fsub_rn(upd, c);
    const float t = grid_round_nearest(f, __fadd_rn(s, y));
    comp[i] = __fsub_rn(__fsub_rn(t, s), y);
    w[i] = t;
  }
  if (bad_mom) atomicOr(status, ST_NONFINITE_MOMENTS);
  if (bad_upd) atomicOr(status, ST_NONFINITE_X);
}

extern "C" xmc_status xmc_kahan_adamw_step(xmc_grid g, float* w, float* comp, float* m, float* v, const float* grad,
                                           int64_t n, float lr, double beta1, double beta2, float eps, float wd,
                                           int64_t t, void* stream) {
  xmc_status s;
  const GridFmt f = grid_from(g, &s);
  XMC_TRY(s);
  if (!w || !comp || !m || !v || !grad) return fail(XMC_ERR_ARG, "null argument");
  if (!(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0))
    return fail(XMC_ERR_ARG, "betas must lie in [0, 1)");
  if (!(eps > 0.0f)) return fail(XMC_ERR_ARG, "eps must be positive");
  if (t < 1) return fail(XMC_ERR_ARG, "step index t must be >= 1");
  if (n <= 0) return XMC_OK;
  AdamWArgs a;
  a.lr = lr;
  a.b1 = static_cast<float>(beta1);   // np.float32(cfg.beta1)
  a.b2 = static_cast<float>(beta2);
  a.omb1 = 1.0f - a.b1;   // np.float32(1) - b1: fp32 subtraction
  a.omb2 = 1.0f - a.b2;
  a.eps = eps;
  a.wd = wd;
  // np.float32(1.0 - beta ** t): double, then one rounding to fp32
  a.bc1 = static_cast<float>(1.0 - std::pow(beta1, static_cast<double>(t)));
  a.bc2 = static_cast<float>(1.0 - std::pow(beta2, static_cast<double>(t)));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* status = scratch_status();
  CUDA_TRY(cudaMemsetAsync(status, 0, 4, st));
  const bool wp = g.exp_bits == 8 && g.man_bits == 23;
  adamw_kernel<<<ew_blocks(n), 256, 0, st>>>(f, wp, a, w, comp, m, v, grad, n, 0, status);
  adamw_kernel<<<ew_blocks(n), 256, 0, st>>>(f, wp, a, w, comp, m, v, grad, n, 1, status);
  CUDA_TRY(cudaGetLastError());
  return finish_elementwise(status, st);
}

__global__ void cast_kernel(const float* __restrict__ x, void* __restrict__ out, int64_t n, int fmt, int32_t* status) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    bad |= !isfinite(v);
    if (fmt == FMT_E4M3) static_cast<uint8_t*>(out)[i] = enc_e4m3(v);
    else if (fmt == FMT_E5M2) static_cast<uint8_t*>(out)[i] = enc_e5m2(v);
    else static_cast<uint16_t*>(out)[i] = enc_bf16(v);
  }
  if (bad && status) atomicOr(status, ST_NONFINITE_X);
}

extern "C" xmc_status xmc_cast_rn(const float* x, void* out, int64_t n, int32_t fmt, int32_t* status, void* stream) {
  if (fmt != XMC_FMT_E4M3 && fmt != XMC_FMT_E5M2 && fmt != XMC_FMT_BF16)
    return fail(XMC_ERR_UNSUPPORTED, "cast target must be e4m3, e5m2 or bf16");
  if (n <= 0) return XMC_OK;
  cast_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, out, n, fmt, status);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

// logit_gradient (head.py:181-196): accurate expf + IEEE division like numpy fp32
__global__ void sigmoid_clip_kernel(const float* __restrict__ z, int64_t rows, int B, int64_t ld, float* __restrict__ G) {
  const int64_t n = rows * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / B;
    const int s = static_cast<int>(i - r * B);
    float g = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z[r * ld + s])));
    g = g < 5.9604644775390625e-08f ? 5.9604644775390625e-08f : g;
    g = g > 0.99999994039535522461f ? 0.99999994039535522461f : g;
    G[r * ld + s] = g;
  }
}

__global__ void positives_apply_kernel(const float* __restrict__ z, int64_t rows, int B, int64_t ld,
                                       const int32_t* __restrict__ ps, const int32_t* __restrict__ pl, int64_t nnz,
                                       int64_t start, float* __restrict__ G, int32_t* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = static_cast<int64_t>(pl[i]) - start;
    const int s = ps[i];
    if (r < 0 || r >= rows) {
      atomicOr(status, ST_LABEL_OUTSIDE);
      continue;
    }
    if (s < 0 || s >= B) {
      atomicOr(status, ST_BAD_SAMPLE);
      continue;
    }
    float g = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z[r * ld + s])));
    g = g < 5.9604644775390625e-08f ? 5.9604644775390625e-08f : g;
    g = g > 0.99999994039535522461f ? 0.99999994039535522461f : g;
    G[r * ld + s] = __fsub_rn(g, 1.0f);
  }
}

extern "C" xmc_status xmc_logit_gradient(const float* logits, int64_t rows, int32_t B, int64_t ld,
                                         const int32_t* pos_sample, const int32_t* pos_label, int64_t nnz,
                                         int64_t chunk_start, float* G, void* stream) {
  if (!logits || !G || rows < 0 || B < 1 || ld < B) return fail(XMC_ERR_ARG, "bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t* status = scratch_status();
  CUDA_TRY(cudaMemsetAsync(status, 0, 4, st));
  if (rows > 0) {
    sigmoid_clip_kernel<<<ew_blocks(rows * B), 256, 0, st>>>(logits, rows, B, ld, G);
    CUDA_TRY(cudaGetLastError());
  }
  if (nnz > 0) {
    positives_apply_kernel<<<ew_blocks(nnz), 256, 0, st>>>(logits, rows, B, ld, pos_sample, pos_label, nnz,
                                                          chunk_start, G, status);
    CUDA_TRY(cudaGetLastError());
  }
  int32_t s = 0;
  CUDA_TRY(cudaMemcpyAsync(&s, status, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (s & ST_LABEL_OUTSIDE) return fail(XMC_ERR_LABEL, "label outside chunk range");
  if (s & ST_BAD_SAMPLE) return fail(XMC_ERR_INDEX, "positive sample index out of range");
  return XMC_OK;
}
