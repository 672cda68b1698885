// C-ABI implementation: handle + workspace layout, TMA descriptor encoding,
// and the launch orchestration of a head step -- per chunk the logits+G
// kernel (xmc_fwd.cuh) and the grad_X + dW + update kernel (xmc_bwd.cuh),
// around the small per-step kernels of xmc_small.cuh.  The elementwise
// numeric core lives in xmc_elementwise.cu.
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

#include "xmc_bwd.cuh"
#include "xmc_common.cuh"
#include "xmc_fwd.cuh"
#include "xmc_ptx.cuh"
#include "xmc_round.cuh"
#include "xmc_small.cuh"

using namespace xmc;

#define fail xmc_fail

// ============================================================== errors
static thread_local std::string g_err;

xmc_status xmc_fail(xmc_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

extern "C" const char* xmc_last_error(void) { return g_err.c_str(); }
extern "C" const char* xmc_version(void) { return "xmc-b200 0.2 (sm_100a tcgen05)"; }

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}

// per (host thread, device) status scratch of the handle-less entry points:
// each call clears it, runs, and synchronises before returning, so calls of
// one thread never overlap on it and threads / devices never share one
int32_t* xmc_device_scratch_status() {
  constexpr int kMaxDev = 64;
  static thread_local int32_t* p[kMaxDev] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDev) return nullptr;
  if (!p[dev] && cudaMalloc(&p[dev], 64) != cudaSuccess) {
    cudaGetLastError();
    p[dev] = nullptr;
  }
  return p[dev];
}

// Set a kernel's dynamic shared-memory limit once per (kernel, device): the
// kernel is a template argument, so every instantiation has its own flags.
template <auto Kernel>
static void smem_attr_once(int bytes) {
  constexpr int kMaxDev = 64;
  static bool done[kMaxDev] = {};
  const int dev = current_device();
  if (dev >= 0 && dev < kMaxDev && done[dev]) return;
  cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (dev >= 0 && dev < kMaxDev) done[dev] = true;
}

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

// Effective SM clock of the fwd / bwd kernels since the last read: summed
// clock64 cycles and globaltimer ns of block 0 per kind (out[0..3] = fwd
// cycles, fwd ns, bwd cycles, bwd ns).  Synchronises the device.
extern "C" xmc_status xmc_profile_clock(uint64_t* out4) {
  unsigned long long h[4] = {0, 0, 0, 0};
  const unsigned long long z[4] = {0, 0, 0, 0};
  if (cudaMemcpyFromSymbol(h, g_xmc_clk, sizeof(h)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_xmc_clk, z, sizeof(z)) != cudaSuccess)
    return fail(XMC_ERR_CUDA, "xmc_profile_clock: %s", cudaGetErrorString(cudaGetLastError()));
  for (int i = 0; i < 4; ++i) out4[i] = h[i];
  return XMC_OK;
}

// ============================================================== helpers

static int elem_bytes(int fmt) { return fmt == XMC_FMT_E4M3 || fmt == XMC_FMT_E5M2 ? 1 : (fmt == XMC_FMT_FP32 ? 4 : 2); }

// padded batch = N of the logits MMA = G leading dimension
static int padded_batch(int eb, int B) {
  // > 256: the forward runs 256-sample passes, the backward grad_X passes of
  // 256 TMEM columns (the update rides on the last); beyond 1024 samples the
  // padded batch is the next multiple of 256 (entries keep a 16-bit sample)
  const int opts1[] = {128, 256, 512, 1024};
  const int opts2[] = {64, 128, 256, 512, 1024};
  if (eb == 1) {
    for (int o : opts1) if (B <= o) return o;
  } else {
    for (int o : opts2) if (B <= o) return o;
  }
  if (B <= 65535) return (B + 255) / 256 * 256;
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
  int eb;              // W / X element bytes (storage, forward operands)
  bool ref;            // reference-precision backward (desc.precision)
  int planes;          // G planes: 3 (reference precision) or 1
  int beb;             // backward operand element bytes (2 in reference precision)
  int gout;            // forward G output (G_OPERAND / G_E5M2 / G_REF)
  int max_bp;          // padded batch capacity
  int num_sms;
  int dtiles;
  std::vector<std::pair<int64_t, int64_t>> chunks;  // local row ranges
  std::vector<int32_t> tile_base;                   // per chunk, plus total at the end
  int64_t total_tiles;
  int64_t max_chunk_rows;
  // workspace carve-up (device pointers)
  uint8_t* xq;         // [max_bp][d] (eb)
  uint8_t* xqt;        // [d][max_bp] (beb)
  uint8_t* gbuf;       // [max_chunk_rows + 128][planes * max_bp] (beb)
  float* gx_ws;        // [R][d][gx_planes * max_bp]
  int32_t* tile_cnt;   // [total_tiles + 1]
  int32_t* tile_ptr;   // [total_tiles + 1]
  int32_t* tile_cur;   // [total_tiles + 1] scatter cursors (tile_cnt is re-zeroed by the scan)
  uint32_t* entries;   // [max_positives]
  uint32_t* tmp_tile;  // [max_positives] tile id per positive (bucketing scratch)
  uint32_t* tmp_entry; // [max_positives] packed entry per positive
  int64_t* chunk_dev;  // [k+1] chunk starts (local rows) + [k+1] tile bases
  int32_t* status;     // [4]
  int R_step;          // grad_X partial slots written by the current step's backward
  int64_t g_row_off = 0;  // first G buffer row of the next backward launch (a sub-range of the chunk)
  uint8_t* xq_topk;    // Xq rows of the current top-k launch (sample offset applied)
  uint8_t* wm;         // [max_chunk_rows + 128][d] masked W chunk (dropout only)
  uint32_t* keep;      // [max_chunk_rows + 128][d / 32] dropout keep bits (dropout only)
  int64_t comp_rows;   // local rows [0, comp_rows) carry a Kahan compensation
  float* cand_s;       // [max_bp][4 num_sms][kTopK] streaming top-k candidates (scores)
  int32_t* cand_l;     // [max_bp][4 num_sms][kTopK] (global labels)
  float* topk_pre_s;   // [max_bp][kTopK] top-8 scores of the top-k prologue (a strided label sample)
  int64_t* topk_pre_l; // [max_bp][kTopK] their labels (unused)
  int R;               // bwd CTAs per d-tile
  int fwd_max_clusters;   // co-resident CTA pairs of the forward (grid cap, PDL safety)
  bool pdl_ok;
  // Adam-style head step in flight (xmc_head_step_adamw sets it for the call):
  // moments at local row 0 and the kahan_adamw_step constants
  struct {
    float* m = nullptr;
    float* v = nullptr;
    float b1, b2, omb1, omb2, bc1, bc2, eps;
  } adam;
  struct xmc_peer* peer = nullptr;   // node-local grad_X all-reduce group (xmc_head_attach_peers)
};

// ---- node-local grad_X all-reduce over peer memory (CUDA IPC / NVLink P2P) ----
// Every rank cudaMallocs one exchange buffer and maps every peer's (IPC
// handles swapped by the caller).  Layout, identical on all ranks:
//   xin   [2 parity][world src][nblocks][1024] fp32   32x32 grad_X tiles pushed by rank src
//   flags [2 parity][world src][nblocks] int32         epoch of the step that pushed the tile
struct xmc_peer {
  int rank = 0, world = 1, dim = 0, max_bp = 0, nblocks = 0;
  uint8_t* local = nullptr;   // own exchange buffer
  size_t bytes = 0, flag_off = 0;
  void* base[kMaxPeers] = {};   // every rank's buffer as mapped here (own = local)
  int32_t epoch = 0;
  bool connected = false;
};

struct Layout {
  size_t xq, xqt, gbuf, gx, cnt, ptr, cur, ent, tmp, chunk, status, wm, keep, cand, total;
};

// grad_X partial column groups per sample: the reference-precision planes
// accumulate into one TMEM accumulator (grad_X^T = sum_p W^T G_p) when the
// padded batch fits its 256 columns; bf16 batch 512 keeps one column group
// per plane (two passes, summed by the reduce kernel)
static int gx_planes(bool ref, int planes, int bp) { return (ref && bp <= 256) ? 1 : planes; }

static xmc_status compute_layout(const xmc_head_desc* d, Layout* L, int* eb_out, int* bp_out, int* R_out,
                                 int64_t* tiles_out, int64_t* maxrows_out, int num_sms) {
  if (!d) return fail(XMC_ERR_ARG, "null desc");
  if (d->fmt != XMC_FMT_E4M3 && d->fmt != XMC_FMT_BF16)
    return fail(XMC_ERR_UNSUPPORTED, "head format must be e4m3 or bf16 (got %d)", d->fmt);
  const int eb = elem_bytes(d->fmt);
  // d-tiles of 128 columns; a partial last tile is zero-filled by TMA on load
  // and clipped on store (the 32-column epilogue chunks need d % 32 == 0)
  if (d->dim <= 0 || d->dim % 32 != 0)
    return fail(XMC_ERR_SHAPE, "dim must be a positive multiple of 32 (got %d)", d->dim);
  if (d->num_chunks < 1) return fail(XMC_ERR_ARG, "num_chunks must be >= 1");
  if (d->comp_bytes != 0 && d->comp_bytes != 2 && d->comp_bytes != 4)
    return fail(XMC_ERR_ARG, "comp_bytes must be 0 (none), 2 (bf16) or 4 (fp32)");
  if (d->precision != XMC_PRECISION_OPERAND && d->precision != XMC_PRECISION_REFERENCE)
    return fail(XMC_ERR_ARG, "precision must be XMC_PRECISION_OPERAND or XMC_PRECISION_REFERENCE");
  if (d->g_format != 0 && d->g_format != XMC_FMT_E4M3 && d->g_format != XMC_FMT_E5M2 && d->g_format != XMC_FMT_BF16)
    return fail(XMC_ERR_ARG, "g_format must be 0 (default), e4m3, e5m2 or bf16");
  if (d->num_labels_local < 1 || d->label_offset < 0 ||
      d->label_offset + d->num_labels_local > d->num_labels_global)
    return fail(XMC_ERR_ARG, "bad label shard [%lld, +%lld) of %lld", (long long)d->label_offset,
                (long long)d->num_labels_local, (long long)d->num_labels_global);
  if (d->max_batch < 1 || d->max_batch > 65535) return fail(XMC_ERR_ARG, "max_batch out of range");
  const int bp = padded_batch(eb, d->max_batch);
  if (bp < 0) return fail(XMC_ERR_UNSUPPORTED, "batch %d too large for format", d->max_batch);
  // bf16-operand backward: the reference precision (three planes) or, for an
  // e4m3 head, the operand mode with g_format bf16 (one plane, the paper's
  // FP8 weights with BF16 logit gradients); both convert e4m3 W tiles to bf16
  // operands in shared memory
  const bool ref = d->precision == XMC_PRECISION_REFERENCE ||
                   (eb == 1 && d->g_format == XMC_FMT_BF16);
  const int planes = d->precision == XMC_PRECISION_REFERENCE ? 3 : 1;
  const int beb = ref ? 2 : eb;
  auto ch = partition(d->num_labels_local, d->num_chunks);
  int64_t tiles = 0, maxrows = 0;
  for (auto& c : ch) {
    tiles += cdiv(c.second - c.first, 128);
    maxrows = std::max(maxrows, c.second - c.first);
  }
  const int dtiles = (d->dim + 127) / 128;
  int R = std::max(1, num_sms / dtiles);
  const int64_t D = d->dim;
  L->xq = 0;
  L->xqt = align_up(L->xq + (size_t)bp * D * eb, 1024);
  L->gbuf = align_up(L->xqt + (size_t)bp * D * beb, 1024);
  L->gx = align_up(L->gbuf + (size_t)(maxrows + 128) * planes * bp * beb, 1024);
  L->cnt = align_up(L->gx + (size_t)R * D * gx_planes(ref, planes, bp) * bp * 4, 256);
  L->ptr = align_up(L->cnt + (size_t)(tiles + 1) * 4, 256);
  L->cur = align_up(L->ptr + (size_t)(tiles + 1) * 4, 256);
  L->ent = align_up(L->cur + (size_t)(tiles + 1) * 4, 256);
  L->tmp = align_up(L->ent + (size_t)std::max<int64_t>(d->max_positives, 1) * 4, 256);
  L->chunk = align_up(L->tmp + (size_t)std::max<int64_t>(d->max_positives, 1) * 8, 256);
  L->status = align_up(L->chunk + (size_t)(2 * (ch.size() + 1)) * 8, 256);
  L->wm = align_up(L->status + 64, 1024);
  L->keep = align_up(L->wm + (d->dropout ? (size_t)(maxrows + 128) * D * eb : 0), 1024);
  L->cand = align_up(L->keep + (d->dropout ? (size_t)(maxrows + 128) * (D / 32) * 4 : 0), 1024);
  L->total = align_up(L->cand + (size_t)bp * 4 * num_sms * kTopK * 8 + (size_t)bp * kTopK * 12, 1024);
  *eb_out = eb;
  *bp_out = bp;
  *R_out = R;
  *tiles_out = tiles;
  *maxrows_out = maxrows;
  return XMC_OK;
}

static int device_sms() {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
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
  h->ref = desc->precision == XMC_PRECISION_REFERENCE || (eb == 1 && desc->g_format == XMC_FMT_BF16);
  h->planes = desc->precision == XMC_PRECISION_REFERENCE ? 3 : 1;
  h->beb = h->ref ? 2 : eb;
  // the e4m3 head's operand G: e5m2 x 2^8 by default (covers the reference's
  // whole [2^-24, 1] sigmoid range), e4m3 x 2^8 on request
  h->gout = h->planes == 3 ? G_REF
                           : (h->ref ? G_BF16 : ((eb == 1 && desc->g_format != XMC_FMT_E4M3) ? G_E5M2 : G_OPERAND));
  h->max_bp = bp;
  h->num_sms = sms;
  h->dtiles = (desc->dim + 127) / 128;
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
  h->tmp_tile = reinterpret_cast<uint32_t*>(w + L.tmp);
  h->tmp_entry = h->tmp_tile + std::max<int64_t>(desc->max_positives, 1);
  h->chunk_dev = reinterpret_cast<int64_t*>(w + L.chunk);
  h->status = reinterpret_cast<int32_t*>(w + L.status);
  h->wm = desc->dropout ? w + L.wm : nullptr;
  h->keep = desc->dropout ? reinterpret_cast<uint32_t*>(w + L.keep) : nullptr;
  h->comp_rows = desc->comp_bytes == 0 ? 0
                 : desc->comp_labels <= 0
                     ? desc->num_labels_local
                     : std::min<int64_t>(desc->num_labels_local,
                                         std::max<int64_t>(0, desc->comp_labels - desc->label_offset));
  h->cand_s = reinterpret_cast<float*>(w + L.cand);
  h->cand_l = reinterpret_cast<int32_t*>(w + L.cand + (size_t)bp * 4 * sms * kTopK * 4);
  h->topk_pre_l = reinterpret_cast<int64_t*>(w + L.cand + (size_t)bp * 4 * sms * kTopK * 8);
  h->topk_pre_s = reinterpret_cast<float*>(w + L.cand + (size_t)bp * 4 * sms * kTopK * 8 + (size_t)bp * kTopK * 8);
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
  // forward pairs: how many CTA pairs are co-resident.  The persistent grid is
  // capped there, which keeps every primary of a PDL chain fully resident.
  {
    using CP = FwdCfg<1, 256, true, true>;
    smem_attr_once<xmc_fwd_kernel<1, 256, true, false, true, G_OPERAND>>(CP::kSmemBytes);
    h->fwd_max_clusters = h->num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (h->num_sms / 2));
    cfg.blockDim = dim3(CP::kThreads);
    cfg.dynamicSmemBytes = CP::kSmemBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    h->pdl_ok = cudaOccupancyMaxActiveClusters(&n, xmc_fwd_kernel<1, 256, true, false, true, G_OPERAND>, &cfg) ==
                    cudaSuccess &&
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
  if (dim <= 0 || dim % 32 != 0) return fail(XMC_ERR_SHAPE, "dim must be a positive multiple of 32");
  if (max_batch < 1 || max_batch > 65535) return fail(XMC_ERR_ARG, "max_batch outside [1, 65535]");
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
// ============================================================== launches
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

// Xq (forward operand) and Xq^T (backward operand: bf16 in reference precision)
static xmc_status launch_x_prep(xmc_head* h, const float* X, int B, int Bp, cudaStream_t st) {
  dim3 grid(h->desc.dim / 32, Bp / 32), block(32, 8);
  const int D = h->desc.dim;
  if (h->eb == 1 && h->beb == 2) x_prep_kernel<1, 2><<<grid, block, 0, st>>>(X, B, Bp, D, h->xq, h->xqt, h->status);
  else if (h->eb == 1) x_prep_kernel<1><<<grid, block, 0, st>>>(X, B, Bp, D, h->xq, h->xqt, h->status);
  else x_prep_kernel<2><<<grid, block, 0, st>>>(X, B, Bp, D, h->xq, h->xqt, h->status);
  CUDA_TRY(cudaGetLastError());
  return XMC_OK;
}

// Programmatic dependent launch for the fwd / bwd / reduce kernels: a kernel's
// CTAs start (barriers, TMEM, tensor maps) on SMs the previous kernel's CTAs
// vacate and then wait in griddepcontrol.wait.  Safe because every primary is
// persistent and fully co-resident (forward clusters capped at the measured
// co-resident count).
static bool pdl_enabled(const xmc_head* h) { return h->pdl_ok; }

template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kernel)(KArgs...), int grid, int block, int smem, cudaStream_t st,
                             const xmc_head* h, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  cfg.attrs = at;
  cfg.numAttrs = 0;
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

// ---- forward ----
template <int EB, int BN, bool PAIR, int GOUT>
static xmc_status launch_fwd_t(xmc_head* h, const CUtensorMap& tw, const CUtensorMap& tx, const FwdParams& p,
                               cudaStream_t st) {
  int grid = static_cast<int>(std::min<int64_t>(h->num_sms, PAIR ? 2 * ((p.num_tiles + 1) / 2) : p.num_tiles));
  if (PAIR) grid = std::min(grid & ~1, 2 * h->fwd_max_clusters);
  if (grid <= 0) return XMC_OK;
  ProfRec pr;
  prof_begin(0, st, &pr);
  if constexpr (PAIR && EB == 1) {
    using CX = FwdCfg<EB, BN, true, true>;
    if ((p.d + CX::kBoxK - 1) / CX::kBoxK <= CX::kXResChunks) {   // resident Xq (e4m3 pairs, d <= 768)
      auto k = xmc_fwd_kernel<EB, BN, true, false, true, GOUT>;
      smem_attr_once<xmc_fwd_kernel<EB, BN, true, false, true, GOUT>>(CX::kSmemBytes);
      CUDA_TRY(launch_ex(k, grid, CX::kThreads, CX::kSmemBytes, st, h, 2, tw, tx, p));
      prof_end(st, &pr);
      return XMC_OK;
    }
  }
  using C = FwdCfg<EB, BN, PAIR>;
  auto k = xmc_fwd_kernel<EB, BN, PAIR, false, false, GOUT>;
  smem_attr_once<xmc_fwd_kernel<EB, BN, PAIR, false, false, GOUT>>(C::kSmemBytes);
  CUDA_TRY(launch_ex(k, grid, C::kThreads, C::kSmemBytes, st, h, PAIR ? 2 : 1, tw, tx, p));
  prof_end(st, &pr);
  return XMC_OK;
}

// one BN-sample pass: pairs for 128 / 256 samples, single CTAs for 64
template <int GOUT>
static xmc_status launch_fwd_g(xmc_head* h, int Bp, const CUtensorMap& tw, const CUtensorMap& tx,
                               const FwdParams& p, cudaStream_t st) {
  if (h->eb == 1) {
    if (Bp == 128) return launch_fwd_t<1, 128, true, GOUT>(h, tw, tx, p, st);
    if (Bp == 256) return launch_fwd_t<1, 256, true, GOUT>(h, tw, tx, p, st);
  } else if constexpr (GOUT != G_E5M2 && GOUT != G_BF16) {
    if (Bp == 64) return launch_fwd_t<2, 64, false, GOUT>(h, tw, tx, p, st);
    if (Bp == 128) return launch_fwd_t<2, 128, true, GOUT>(h, tw, tx, p, st);
    if (Bp == 256) return launch_fwd_t<2, 256, true, GOUT>(h, tw, tx, p, st);
  }
  return fail(XMC_ERR_UNSUPPORTED, "no forward kernel for padded batch %d", Bp);
}

// Logits (+ G) of `rows` rows starting at W (already offset to the chunk's
// first row).  mode 0: G into out (gbuf layout: ld = planes * Bp), mode 1:
// fp32 logits [rows][ld].
static xmc_status launch_fwd(xmc_head* h, const void* W, int64_t rows, int B, int Bp, int mode,
                             const int32_t* tile_ptr, void* out, int64_t ld, float* stats, cudaStream_t st,
                             float logit_scale = 1.0f) {
  const int eb = h->eb, D = h->desc.dim;
  const bool pair = Bp >= 128;
  FwdParams p{};
  p.rows = static_cast<int32_t>(rows);
  p.B = B;
  p.d = D;
  p.num_tiles = static_cast<int32_t>(cdiv(rows, 128));
  p.mode = mode;
  p.tile_ptr = tile_ptr;
  p.entries = h->entries;
  p.out = out;
  p.ld = ld;
  p.plane_ld = Bp;
  p.g_planes = h->planes;
  // training forward (one pass): the last ~120 MB of each CTA pair's W tiles
  // stay in L2 for the backward, which walks the tiles in reverse (C4: 8
  // units of 256 rows per pair; same-box A/B -1.5 % bwd, +0.6 % step)
  const int64_t unit_bytes = static_cast<int64_t>(h->num_sms / 2) * 256 * D * eb;
  p.w_keep_units = (mode == 0 && pair && Bp <= 256) ? static_cast<int32_t>(120000000 / unit_bytes) : 0;
  p.stats = stats;
  p.logit_scale = logit_scale;
  p.status = h->status;
  CUtensorMap tw;
  XMC_TRY(make_map(&tw, W, eb, D, rows, D, 128));
  // batches over 256 run as 256-sample passes of the pair kernel
  const int pass_n = Bp > 256 ? 256 : Bp;
  for (int pass = 0; pass * pass_n < B || pass == 0; ++pass) {
    FwdParams q = p;
    q.sample0 = pass * pass_n;
    q.B = std::min(pass_n, B - pass * pass_n);
    const size_t col_bytes = mode == 1 ? 4 : (h->ref ? 2 : eb);
    q.out = static_cast<uint8_t*>(out) + static_cast<size_t>(pass) * pass_n * col_bytes;
    CUtensorMap tx;
    XMC_TRY(make_map(&tx, h->xq + static_cast<size_t>(pass) * pass_n * D * eb, eb, D, pass_n, D,
                     std::min(pair ? pass_n / 2 : pass_n, 256)));
    xmc_status s;
    if (mode == 1 || h->gout == G_OPERAND) s = launch_fwd_g<G_OPERAND>(h, pass_n, tw, tx, q, st);
    else if (h->gout == G_E5M2) s = launch_fwd_g<G_E5M2>(h, pass_n, tw, tx, q, st);
    else if (h->gout == G_BF16) s = launch_fwd_g<G_BF16>(h, pass_n, tw, tx, q, st);
    else s = launch_fwd_g<G_REF>(h, pass_n, tw, tx, q, st);
    XMC_TRY(s);
    if (Bp <= 256) break;
  }
  return XMC_OK;
}

// ---- backward ----
struct BwdLaunch {
  CUtensorMap tw, tg, tx, tws, tc;   // tc: the staged bf16 compensation (fast head-Kahan), else a copy of tw
  BwdParams p;
  int R;
};

// One bwd pass over `rows` chunk rows whose W starts at Wc (the chunk's first
// row: W itself, the masked dropout copy or the bf16 reference-precision copy)
// and whose global label / compensation row is the local row row0.  G from
// gbuf; grad_X partials into the [R][d][gx_planes * Bp] workspace.
static xmc_status setup_bwd(xmc_head* h, void* Wc, void* comp, int64_t row0, int64_t rows, int Bp, bool update,
                            int gx_kc0, int gx_kc_count, bool gx_overwrite, const xmc_step_args* a,
                            const uint32_t* keep, float drop_scale, BwdLaunch* L) {
  const int beb = h->beb, D = h->desc.dim;
  const int box_k = 128 / beb;
  const int ldg = h->planes * Bp;
  const int gxp = gx_planes(h->ref, h->planes, Bp);
  // W in its storage format (an e4m3 head's reference-precision kernel
  // converts each tile to bf16 operands in shared memory)
  XMC_TRY(make_map(&L->tw, Wc, h->eb, D, rows, D, 128));
  XMC_TRY(make_map(&L->tws, Wc, h->eb, D, rows, D, 32));
  const int64_t tiles = cdiv(rows, 128);
  const int R = static_cast<int>(std::min<int64_t>(h->R, tiles));
  XMC_TRY(make_map(&L->tg, h->gbuf + h->g_row_off * ldg * beb, beb, ldg, rows, ldg, 128));
  XMC_TRY(make_map(&L->tx, h->xqt, beb, Bp, D, Bp, 128));
  BwdParams& p = L->p;
  p = BwdParams{};
  p.rows = static_cast<int32_t>(rows);
  p.d = D;
  p.num_tiles = static_cast<int32_t>(tiles);
  p.dtiles = h->dtiles;
  p.kc_count = ldg / box_k;
  p.xt_kc = Bp / box_k;
  p.do_update = update ? 1 : 0;
  p.gx_kc0 = gx_kc0;
  p.gx_kc_count = gx_kc_count;
  // reference-precision planes accumulated in TMEM: grad_X MMA groups of
  // N = 128 samples (2 k-chunks), so the 4-slot G ring holds two groups and the
  // producer loads one while the other multiplies
  // (also the one-plane bf16-G backward of an e4m3 head: N = 128 groups free
  // the 6-slot G ring half a tile at a time)
  // (only while the whole padded batch fits the 256 grad_X TMEM columns)
  const bool acc_planes = gxp == 1 && Bp <= 256 && (h->planes > 1 || (h->ref && h->eb == 1) || (h->eb == 2 && Bp == 256));
  p.gx_group = acc_planes ? std::min(2, Bp / box_k) : gx_kc_count;
  p.gx_cols = acc_planes ? Bp : gx_kc_count * box_k;
  p.g_prefetch = h->ref ? 1 : 0;
  // reference precision: drain grad_X every 32 tiles (fp32 accumulation
  // chains of <= 32 x 3 x 128 products per TMEM window)
  p.gx_flush = h->planes > 1 ? 32 : 0;
  p.g_e5m2 = h->gout == G_E5M2 ? 1 : 0;
  p.W = static_cast<uint8_t*>(Wc);
  const int64_t crows = comp ? std::min<int64_t>(rows, std::max<int64_t>(0, h->comp_rows - row0)) : 0;
  p.comp = crows > 0 ? static_cast<uint8_t*>(comp) + row0 * D * h->desc.comp_bytes : nullptr;
  p.comp_rows = static_cast<int32_t>(crows);
  L->tc = L->tw;
  if (crows > 0 && h->desc.comp_bytes == 2)   // [crows][d] bf16, 64-column boxes of 128 rows
    XMC_TRY(make_map(&L->tc, p.comp, 2, D, crows, D, 128));
  p.row0_global = h->desc.label_offset + row0;
  p.lr = a ? a->lr : 0.f;
  p.wd = a ? a->weight_decay : 0.f;
  p.dw_scale = (h->eb == 1 && !h->ref) ? (1.0f / 256.0f) : 1.0f;
  p.rounding = a ? a->rounding : 0;
  p.rng_base = a ? sm64_base(a->seed, a->step, a->tensor_id) : 0;
  p.sr_bits = a ? a->sr_bits : 0;
  p.gx_ws = h->gx_ws;
  p.gx_ld = gxp * Bp;
  p.gx_accumulate = gx_overwrite ? 0 : 1;
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
  p.keep = keep;
  p.drop_scale = drop_scale;
  p.status = h->status;
  L->R = R;
  return XMC_OK;
}

template <int EB, bool XR, int KC, int CE, bool FAST, bool ADAMW, int GE, int SB>
static xmc_status launch_bwd_k(xmc_head* h, const BwdLaunch& L, cudaStream_t st) {
  constexpr int sm = BwdCfg<EB, XR, KC, SB, bwd_comp_staged<CE, FAST>()>::kSmemBytes;
  static_assert(sm <= 232448, "bwd shared memory over the 227 KB opt-in limit");
  auto k = xmc_bwd_kernel<EB, XR, KC, CE, FAST, ADAMW, GE, SB>;
  smem_attr_once<xmc_bwd_kernel<EB, XR, KC, CE, FAST, ADAMW, GE, SB>>(sm);
  CUDA_TRY(launch_ex(k, L.R * h->dtiles, kBwdThreads, sm, st, h, 1, L.tw, L.tg, L.tx, L.tws, L.tc, L.p));
  return XMC_OK;
}

// compensation / optimizer variant of one kernel geometry
template <int EB, bool XR, int KC, int GE, int SB = EB>
static xmc_status launch_bwd_v(xmc_head* h, const BwdLaunch& L, cudaStream_t st) {
  const BwdParams& p = L.p;
  if constexpr (KC == 0) {   // grad_X-only pass: no update, no compensation / optimizer state
    return launch_bwd_k<EB, XR, 0, 0, false, false, GE, SB>(h, L, st);
  } else {
  if (p.adam_m != nullptr) return launch_bwd_k<EB, XR, KC, 4, false, true, GE, SB>(h, L, st);
  const int ce = p.comp ? h->desc.comp_bytes : 0;
  // (XMC_BWD_GENERAL=1: test knob, the general instantiation for everything,
  // so tests can compare the fast specialisations against it bit for bit)
  static const bool force_general = getenv("XMC_BWD_GENERAL") != nullptr;
  const bool fast_ok = p.do_update && (p.rounding == ROUND_SR_FAST || p.rounding == ROUND_NEAREST) &&
                       p.keep == nullptr && !force_general;
  // the fast head-Kahan (bf16 compensation staged by TMA with the W tile)
  if constexpr (EB == 1 && GE == 1 && XR && KC <= 2)
    if (ce == 2 && fast_ok) return launch_bwd_k<1, XR, KC, 2, true, false, 1, 1>(h, L, st);
  if (ce == 2) return launch_bwd_k<EB, XR, KC, 2, false, false, GE, SB>(h, L, st);
  if (ce == 4) return launch_bwd_k<EB, XR, KC, 4, false, false, GE, SB>(h, L, st);
  // the FAST instantiation keeps Xq^T resident and whole tiles in the G ring
  if constexpr (EB == 1 && GE == 1 && XR && BwdCfg<EB, XR, KC, SB>::kKStages % KC == 0)
    if (fast_ok) return launch_bwd_k<1, XR, KC, 0, true, false, 1, 1>(h, L, st);
  return launch_bwd_k<EB, XR, KC, 0, false, false, GE, SB>(h, L, st);
  }
}

static xmc_status launch_bwd(xmc_head* h, void* Wc, void* comp, int64_t row0, int64_t rows, int Bp, bool update,
                             int gx_kc0, int gx_kc_count, bool gx_overwrite, const xmc_step_args* a,
                             cudaStream_t st, const uint32_t* keep = nullptr, float drop_scale = 1.0f) {
  BwdLaunch L;
  XMC_TRY(setup_bwd(h, Wc, comp, row0, rows, Bp, update, gx_kc0, gx_kc_count, gx_overwrite, a, keep, drop_scale, &L));
  ProfRec pr;
  prof_begin(1, st, &pr);
  xmc_status s = XMC_ERR_UNSUPPORTED;
  if (h->ref && h->eb == 1) {
    // reference precision of an e4m3 head: W stays e4m3 in HBM, each tile is
    // converted to bf16 operands in shared memory; three G planes, resident
    // Xq^T, rounding onto the e4m3 grid
    // batch 512 / 1024: grad_X-only passes without Xq^T on a deep G ring,
    // the update pass streams Xq^T with G
    if (!update && gx_kc_count > 0 && Bp > 256) s = launch_bwd_v<2, true, 0, 1, 1>(h, L, st);
    else if (Bp == 128) s = launch_bwd_v<2, true, 2, 1, 1>(h, L, st);
    else if (Bp == 256) s = launch_bwd_v<2, true, 4, 1, 1>(h, L, st);
    else if (Bp == 512) s = launch_bwd_v<2, false, 8, 1, 1>(h, L, st);
    else if (Bp >= 1024) s = launch_bwd_v<2, false, 16, 1, 1>(h, L, st);   // (k-chunks stream slot by slot)
  } else if (!update && gx_kc_count > 0 && Bp > 256) {
    // grad_X-only pass of a batch over 256 (the update rides on the last
    // pass): G boxes only, a two-tile G ring
    if (h->eb == 1) s = launch_bwd_v<1, true, 0, 1>(h, L, st);
    else s = launch_bwd_v<2, true, 0, 2>(h, L, st);
  } else if (h->eb == 1) {
    if (Bp == 128) s = launch_bwd_v<1, true, 1, 1>(h, L, st);
    else if (Bp == 256) s = launch_bwd_v<1, true, 2, 1>(h, L, st);
    else if (Bp == 512) s = launch_bwd_v<1, true, 4, 1>(h, L, st);
    else if (Bp >= 1024) s = launch_bwd_v<1, false, 8, 1>(h, L, st);   // (k-chunks stream slot by slot)
  } else {
    if (Bp == 64) s = launch_bwd_v<2, true, 1, 2>(h, L, st);
    else if (Bp == 128) s = launch_bwd_v<2, true, 2, 2>(h, L, st);
    else if (Bp == 256) s = launch_bwd_v<2, true, 4, 2>(h, L, st);
    else if (Bp == 512) s = launch_bwd_v<2, false, 8, 2>(h, L, st);
    else if (Bp >= 1024) s = launch_bwd_v<2, false, 16, 2>(h, L, st);
  }
  if (s == XMC_ERR_UNSUPPORTED) return fail(s, "no backward kernel for padded batch %d", Bp);
  XMC_TRY(s);
  prof_end(st, &pr);
  return XMC_OK;
}

// grad_X partials + update for one chunk whose G is in gbuf.  grad_X runs in
// passes of <= 256 TMEM columns over the G column groups (bf16 batch 512,
// the reference-precision planes); the update rides on the LAST pass so every
// grad_X pass reads the pre-update weights (head.py:290-291).
static xmc_status run_backward(xmc_head* h, void* Wc, void* comp, int64_t row0, int64_t rows, int Bp, bool gx,
                               bool update, bool gx_overwrite, const xmc_step_args* a, cudaStream_t st,
                               const uint32_t* keep = nullptr, float drop_scale = 1.0f) {
  if (!gx) return launch_bwd(h, Wc, comp, row0, rows, Bp, update, 0, 0, false, a, st, keep, drop_scale);
  const int kcs = h->planes * Bp * h->beb / 128;
  if (h->planes > 1 && gx_planes(h->ref, h->planes, Bp) == 1)   // one pass; the planes accumulate in TMEM
    return launch_bwd(h, Wc, comp, row0, rows, Bp, update, 0, kcs, gx_overwrite, a, st, keep, drop_scale);
  const int per = 256 * h->beb / 128;   // k-chunks whose grad_X columns fit 256 TMEM columns
  const int groups = (kcs + per - 1) / per;
  for (int gi = groups - 1; gi >= 0; --gi) {
    const int kc0 = gi * per;
    const int cnt = std::min(per, kcs - kc0);
    XMC_TRY(launch_bwd(h, Wc, comp, row0, rows, Bp, update && gi == 0, kc0, cnt, gx_overwrite, a, st, keep,
                       drop_scale));
  }
  return XMC_OK;
}

// The backward of one chunk (local rows [r0, r0 + rows)), G in gbuf:
// grad_X partials from Wgx (W, or the masked dropout copy at its chunk base)
// and, if update, the update of W (dW masked by keep under dropout).
static xmc_status zero_gx_ws(xmc_head* h, int Bp, cudaStream_t st);

static xmc_status chunk_backward(xmc_head* h, void* W, const void* Wgx, void* comp, int64_t r0, int64_t rows,
                                 int Bp, bool gx, bool update, bool gx_overwrite, const xmc_step_args* a,
                                 cudaStream_t st, const uint32_t* keep = nullptr, float drop_scale = 1.0f) {
  const int D = h->desc.dim, eb = h->eb;
  uint8_t* Wr = static_cast<uint8_t*>(W) + r0 * D * eb;
  // top-p% head-Kahan whose compensated prefix ends inside this chunk: the
  // rows without a compensation run first on the plain kernel (their W and G
  // are the ones the forward left in L2), then the prefix on the Kahan one
  const int64_t ce = h->comp_rows;
  if (gx && update && comp && keep == nullptr && Wgx == Wr && ce > r0 && ce < r0 + rows) {
    const int64_t rb = r0 + rows - ce;
    const bool ow_b = gx_overwrite && cdiv(rb, 128) >= h->R_step;
    if (gx_overwrite && !ow_b) XMC_TRY(zero_gx_ws(h, Bp, st));
    h->g_row_off = ce - r0;
    const xmc_status sb = run_backward(h, static_cast<uint8_t*>(W) + ce * D * eb, comp, ce, rb, Bp, true, true, ow_b,
                                       a, st);
    h->g_row_off = 0;
    XMC_TRY(sb);
    return run_backward(h, Wr, comp, r0, ce - r0, Bp, true, true, false, a, st);
  }
  if (Wgx == Wr || !gx) return run_backward(h, Wr, comp, r0, rows, Bp, gx, update, gx_overwrite, a, st, keep, drop_scale);
  XMC_TRY(run_backward(h, const_cast<void*>(Wgx), nullptr, r0, rows, Bp, true, false, gx_overwrite, a, st));
  return update ? launch_bwd(h, Wr, comp, r0, rows, Bp, true, 0, 0, false, a, st, keep, drop_scale) : XMC_OK;
}

// acc[s][c] (+)= scale * sum_r sum_planes ws[r][c][plane * Bp + s] -- one
// deterministic reduction per step
static xmc_status reduce_gx(xmc_head* h, int B, int Bp, float* acc, bool accumulate, cudaStream_t st,
                            float scale = 1.0f) {
  const int D = h->desc.dim;
  const int gxp = gx_planes(h->ref, h->planes, Bp);
  const int ldg = gxp * Bp;
  const float sc = ((h->eb == 1 && !h->ref) ? (1.0f / 256.0f) : 1.0f) * scale;
  dim3 g(D / 32, (Bp + 31) / 32), b(32, 32);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(h) ? 1 : 0;
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
    CUDA_TRY(cudaLaunchKernelEx(&cfg, gx_reduce_peer_kernel, static_cast<const float*>(h->gx_ws), h->R_step, D, ldg,
                                gxp, Bp, B, sc, acc, pa));
    return XMC_OK;
  }
  CUDA_TRY(cudaLaunchKernelEx(&cfg, gx_reduce_kernel, static_cast<const float*>(h->gx_ws), h->R_step, D, ldg,
                              gxp, Bp, B, sc, accumulate ? 1 : 0, static_cast<const int32_t*>(h->status), acc));
  return XMC_OK;
}

static xmc_status zero_gx_ws(xmc_head* h, int Bp, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(h->gx_ws, 0, (size_t)h->R * h->desc.dim * gx_planes(h->ref, h->planes, Bp) * Bp * 4, st));
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
template <int EB, int XTB>
static void launch_prep(xmc_head* h, const float* X, int Bp, const PosGeom& g, const int32_t* ps, const int32_t* pl,
                        int64_t nnz, int B, int32_t T, cudaStream_t st) {
  const int D = h->desc.dim;
  if (nnz <= kPosOneCta && T <= kPosMaxTiles && h->chunks.size() <= 64) {
    // up to 12k positives: one launch (block 0 buckets in shared memory, the rest prepare Xq)
    smem_attr_once<prep_bucket_kernel<EB, XTB>>(kPosMaxTiles * 4);
    const int nblk = 1 + (D / 32) * (Bp / 32);
    // (programmatic launch: its CTAs start as the previous step's reduce
    // vacates SMs, then wait in griddepcontrol.wait)
    launch_ex(prep_bucket_kernel<EB, XTB>, nblk, 1024, T * 4, st, h, 1, X, B, Bp, D, h->xq, h->xqt, g, ps, pl, nnz, T,
              h->tile_ptr, h->entries, h->status);
    return;
  }
  const int blocks = static_cast<int>(cdiv(nnz, 256));
  const int nx = (D / 32) * (Bp / 32);
  launch_ex(prep_count_kernel<EB, XTB>, nx + blocks, 256, 0, st, h, 1, X, B, Bp, D, h->xq, h->xqt, nx, g, ps, pl, nnz,
            h->tile_cnt, h->tmp_tile, h->tmp_entry, h->status);
  smem_attr_once<pos_scan_kernel>(kPosMaxTiles * 4);
  launch_ex(pos_scan_kernel, 1, 1024, T <= kPosMaxTiles ? T * 4 : 0, st, h, 1, h->tile_cnt, h->tile_ptr, h->tile_cur,
            T);
  launch_ex(pos_scatter_kernel, blocks, 256, 0, st, h, 1, nnz, static_cast<const uint32_t*>(h->tmp_tile),
            static_cast<const uint32_t*>(h->tmp_entry), h->tile_cur, h->entries);
}

static xmc_status prepare_step(xmc_head* h, const float* X, int Bp, const int32_t* ps, const int32_t* pl,
                               int64_t nnz, int B, cudaStream_t st) {
  if (nnz > h->desc.max_positives)
    return fail(XMC_ERR_CAPACITY, "%lld positives exceed workspace capacity %lld", (long long)nnz,
                (long long)h->desc.max_positives);
  PosGeom g{h->chunk_dev, h->chunk_dev + h->chunks.size() + 1, static_cast<int32_t>(h->chunks.size()),
            h->desc.label_offset, h->desc.num_labels_local, B};
  const int32_t T = static_cast<int32_t>(h->total_tiles);
  if (h->eb == 1 && h->beb == 2) launch_prep<1, 2>(h, X, Bp, g, ps, pl, nnz, B, T, st);
  else if (h->eb == 1) launch_prep<1, 1>(h, X, Bp, g, ps, pl, nnz, B, T, st);
  else launch_prep<2, 2>(h, X, Bp, g, ps, pl, nnz, B, T, st);
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
  const int D = h->desc.dim, eb = h->eb;
  XMC_TRY(prepare_step(h, X, Bp, pos_sample, pos_label, nnz, B, st));
  DropoutPlan dp;
  XMC_TRY(dropout_plan(h, args, &dp));
  h->R_step = h->R;
  // the first chunk overwrites every partial slot unless it has fewer tiles
  // than slots; later chunks accumulate
  const bool first_covers = !h->chunks.empty() && cdiv(h->chunks[0].second - h->chunks[0].first, 128) >= h->R_step;
  if (!first_covers) XMC_TRY(zero_gx_ws(h, Bp, st));
  if (stats) CUDA_TRY(cudaMemsetAsync(stats, 0, 8, st));
  const int64_t ldg = static_cast<int64_t>(h->planes) * Bp;
  for (size_t c = 0; c < h->chunks.size(); ++c) {
    const int64_t r0 = h->chunks[c].first, rows = h->chunks[c].second - h->chunks[c].first;
    const int32_t* tp = h->tile_ptr + h->tile_base[c];
    const bool ow = first_covers && c == 0;
    uint8_t* Wr = static_cast<uint8_t*>(W) + r0 * D * eb;
    if (!dp.on) {
      XMC_TRY(launch_fwd(h, Wr, rows, B, Bp, 0, tp, h->gbuf, ldg, stats, st));
      XMC_TRY(chunk_backward(h, W, Wr, comp, r0, rows, Bp, true, true, ow, args, st));
      continue;
    }
    // keyed dropout (head.py:155-161, 239-242): logits and grad_X read the
    // masked chunk copy W*keep (1/(1-p) applied to the fp32 accumulators);
    // the update pass reads W and scales kept dW by 1/(1-p)
    XMC_TRY(launch_dropout_prep(h, W, r0, rows, dp, h->wm, h->keep, st));
    XMC_TRY(launch_fwd(h, h->wm, rows, B, Bp, 0, tp, h->gbuf, ldg, stats, st, dp.scale));
    XMC_TRY(chunk_backward(h, W, h->wm, comp, r0, rows, Bp, true, true, ow, args, st, h->keep, dp.scale));
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
  const int s = blockIdx.x, tid = threadIdx.x;
  // every (CTA, warp) slot list arrives sorted (descending, ties by label):
  // thread t merges slots t, t + 256, ... with two-pointer merges
  const float* a = cs + static_cast<size_t>(s) * nslots * kTopK;
  const int32_t* b = cl + static_cast<size_t>(s) * nslots * kTopK;
  float ls[kTopK];
  int32_t ll[kTopK];
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    ls[i] = -INFINITY;
    ll[i] = 0x7fffffff;
  }
  for (int sl0 = tid; sl0 < nslots; sl0 += blockDim.x) {
    float bs[kTopK];
    int32_t bl[kTopK];
#pragma unroll
    for (int i = 0; i < kTopK; ++i) {
      bs[i] = a[sl0 * kTopK + i];
      bl[i] = b[sl0 * kTopK + i];
    }
    float ms[kTopK];
    int32_t ml[kTopK];
    int ia = 0, ib = 0;
#pragma unroll
    for (int i = 0; i < kTopK; ++i) {
      // (register arrays indexed by the merge cursors: selects over the 8 entries)
      float av = -INFINITY, bv = -INFINITY;
      int32_t al = 0x7fffffff, blv = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < kTopK; ++j) {
        if (j == ia) { av = ls[j]; al = ll[j]; }
        if (j == ib) { bv = bs[j]; blv = bl[j]; }
      }
      const bool ta = !topk_better(bv, blv, av, al);
      ms[i] = ta ? av : bv;
      ml[i] = ta ? al : blv;
      ia += ta ? 1 : 0;
      ib += ta ? 0 : 1;
    }
#pragma unroll
    for (int i = 0; i < kTopK; ++i) {
      ls[i] = ms[i];
      ll[i] = ml[i];
    }
  }
#pragma unroll
  for (int i = 0; i < kTopK; ++i) {
    ss[tid * kTopK + i] = ls[i];
    sl[tid * kTopK + i] = ll[i];
  }
  __syncthreads();
  // tree of pairwise merges in shared memory (8 levels of "top kTopK of two
  // sorted lists") instead of one warp folding 256 lists serially
  for (int w = blockDim.x >> 1; w >= 1; w >>= 1) {
    if (tid < w) {
      const int a0 = tid * kTopK, b0 = (tid + w) * kTopK;
      float ms[kTopK];
      int32_t ml[kTopK];
      int ia = 0, ib = 0;
#pragma unroll
      for (int i = 0; i < kTopK; ++i) {
        const float av = ss[a0 + ia], bv = ss[b0 + ib];
        const int32_t al = sl[a0 + ia], bl = sl[b0 + ib];
        const bool ta = !topk_better(bv, bl, av, al);   // ties keep A (labels are unique)
        ms[i] = ta ? av : bv;
        ml[i] = ta ? al : bl;
        ia += ta ? 1 : 0;
        ib += ta ? 0 : 1;
      }
#pragma unroll
      for (int i = 0; i < kTopK; ++i) {
        ss[a0 + i] = ms[i];
        sl[a0 + i] = ml[i];
      }
    }
    __syncthreads();
  }
  if (tid < k) {
    out_s[static_cast<size_t>(s) * k + tid] = ss[tid];
    out_l[static_cast<size_t>(s) * k + tid] = sl[tid];
  }
}

// e4m3 batch-256 scoring runs on CTA pairs with resident Xq (the training
// forward's mainloop)
static int topk_grid(const xmc_head* h, int64_t tiles, int eb, int bn, int D) {
  if (eb == 1 && bn == 256 && D / 128 <= FwdCfg<1, 256, true, true>::kXResChunks)
    return static_cast<int>(std::min<int64_t>(2 * h->fwd_max_clusters, 2 * ((tiles + 1) / 2)));
  return static_cast<int>(std::min<int64_t>(h->num_sms, tiles));
}

template <int EB, int BN>
static xmc_status launch_topk_t(xmc_head* h, const CUtensorMap& tw, const CUtensorMap& tx, const FwdParams& p,
                                cudaStream_t st) {
  using C = FwdCfg<EB, BN, false>;
  const int grid = topk_grid(h, p.num_tiles, EB, BN, p.d);
  if constexpr (EB == 1 && BN == 256) {
    if ((p.d + 127) / 128 <= FwdCfg<1, 256, true, true>::kXResChunks) {
      using CP = FwdCfg<1, 256, true, true>;
      CUtensorMap txp;   // each CTA of a pair stages its 128 samples
      XMC_TRY(make_map(&txp, h->xq_topk, 1, p.d, 256, p.d, 128));
      auto k = xmc_fwd_kernel<1, 256, true, true, true>;
      smem_attr_once<xmc_fwd_kernel<1, 256, true, true, true>>(CP::kSmemBytes);
      CUDA_TRY(launch_ex(k, grid, CP::kThreads, CP::kSmemBytes, st, h, 2, tw, txp, p));
      return XMC_OK;
    }
  }
  auto k = xmc_fwd_kernel<EB, BN, false, true>;
  smem_attr_once<xmc_fwd_kernel<EB, BN, false, true>>(C::kSmemBytes);
  CUDA_TRY(launch_ex(k, grid, C::kThreads, C::kSmemBytes, st, h, 1, tw, tx, p));
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
    auto run = [&](const FwdParams& q) -> xmc_status {
      xmc_status r = XMC_ERR_UNSUPPORTED;
      if (eb == 1) {
        if (bn == 128) r = launch_topk_t<1, 128>(h, tw, tx, q, st);
        else if (bn == 256) r = launch_topk_t<1, 256>(h, tw, tx, q, st);
      } else {
        if (bn == 64) r = launch_topk_t<2, 64>(h, tw, tx, q, st);
        else if (bn == 128) r = launch_topk_t<2, 128>(h, tw, tx, q, st);
        else if (bn == 256) r = launch_topk_t<2, 256>(h, tw, tx, q, st);
      }
      return r == XMC_ERR_UNSUPPORTED ? fail(r, "no top-k kernel for padded batch %d", Bp) : r;
    };
    // Prologue on every 16th work unit (a strided label sample): its top-8
    // per sample bounds the final 8th score from below, so the full pass
    // skips almost every block in its pre-filter (the lists of one warp see
    // too few labels to warm up on their own)
    // (the prologue keeps only each list's maximum; stride sweep at C4, same
    // box: 4 / 8 / 16 / 32 = 0.590 / 0.546 / 0.533 / 0.541 ms)
#ifndef XMC_TOPK_PRESTRIDE
#define XMC_TOPK_PRESTRIDE 16
#endif
    constexpr int kPreStride = XMC_TOPK_PRESTRIDE;
    if (p.num_tiles >= 1024) {
      FwdParams q = p;
      q.unit_mul = kPreStride;
      q.topk_max_only = 1;
      XMC_TRY(run(q));
      topk_merge_kernel<<<p.B, 256, 0, st>>>(p.cand_s, p.cand_l, nslots, kTopK, h->topk_pre_s, h->topk_pre_l);
      CUDA_TRY(cudaGetLastError());
      p.topk_bound = h->topk_pre_s;
    }
    XMC_TRY(run(p));
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
  const uint8_t* Wr = static_cast<const uint8_t*>(W) + row0 * h->desc.dim * h->eb;
  if (!dp.on) return launch_fwd(h, Wr, row1 - row0, B, Bp, 1, nullptr, logits, ld, nullptr, st);
  if (row1 - row0 > h->max_chunk_rows + 128) return fail(XMC_ERR_CAPACITY, "row range exceeds the dropout scratch");
  XMC_TRY(launch_dropout_prep(h, W, row0, row1 - row0, dp, h->wm, h->keep, st));
  return launch_fwd(h, h->wm, row1 - row0, B, Bp, 1, nullptr, logits, ld, nullptr, st, dp.scale);
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
  // G into the operand format the step's forward would have written
  if (h->ref && h->planes == 3) g_quant_kernel<3><<<blocks, 256, 0, st>>>(G, ld, rows, B, Bp, h->gbuf, h->status);
  else if (h->eb == 2 || h->ref) g_quant_kernel<2><<<blocks, 256, 0, st>>>(G, ld, rows, B, Bp, h->gbuf, h->status);
  else if (h->gout == G_E5M2) g_quant_kernel<1><<<blocks, 256, 0, st>>>(G, ld, rows, B, Bp, h->gbuf, h->status);
  else g_quant_kernel<0><<<blocks, 256, 0, st>>>(G, ld, rows, B, Bp, h->gbuf, h->status);
  CUDA_TRY(cudaGetLastError());
  DropoutPlan dp;
  XMC_TRY(dropout_plan(h, args, &dp));
  h->R_step = h->R;
  if (accumulate_gx) XMC_TRY(zero_gx_ws(h, Bp, st));
  if (!dp.on) {
    XMC_TRY(chunk_backward(h, W, static_cast<uint8_t*>(W) + row0 * h->desc.dim * h->eb, nullptr, row0, rows, Bp,
                           accumulate_gx != 0, update != 0, false, args, st));
  } else {
    XMC_TRY(launch_dropout_prep(h, W, row0, rows, dp, accumulate_gx ? h->wm : nullptr, h->keep, st));
    XMC_TRY(chunk_backward(h, W, accumulate_gx ? static_cast<const void*>(h->wm) : nullptr, nullptr, row0, rows, Bp,
                           accumulate_gx != 0, update != 0, false, args, st, h->keep, dp.scale));
  }
  if (accumulate_gx) XMC_TRY(reduce_gx(h, B, Bp, acc, true, st, dp.scale));
  return XMC_OK;
}
