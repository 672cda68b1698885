// The small per-step kernels around the two tcgen05 kernels of a chunk:
// X quantisation (head.py:265), positive-list bucketing per 128-label tile
// (the sort of head.py:272-274 plus the chunk filter of :281), the
// deterministic grad_X partial reduction (with the node all-reduce over peer
// memory), keyed-dropout preparation (head.py:138-161, 239-242), the fp32-G
// operand conversions of the unfused backward entry point and the bf16 W
// chunk copies of the reference-precision e4m3 backward.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "xmc_ptx.cuh"
#include "xmc_round.cuh"

namespace xmc {

constexpr int kMaxPeers = 8;

// X fp32 [B][d] -> Xq [Bp][d] and Xq^T [d][Bp] on the head grid (RTN,
// head.py:265 / formats.py:197-206); padding rows/cols are zero.
// XTB: element bytes of the Xq^T copy (EB, or 2: the e4m3 grid values as bf16
// for the reference-precision backward's kind::f16 operand)
template <int EB, int XTB = EB>
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
    if (XTB == 1) xqt[(int64_t)c * Bp + s] = enc_e4m3(q);
    else reinterpret_cast<uint16_t*>(xqt)[(int64_t)c * Bp + s] = enc_bf16(q);
  }
  if (bad) atomicOr(status, ST_NONFINITE_X);
}

template <int EB, int XTB = EB>
__global__ void x_prep_kernel(const float* __restrict__ X, int B, int Bp, int d, uint8_t* __restrict__ xq,
                              uint8_t* __restrict__ xqt, int32_t* status) {
  x_prep_body<EB, XTB>(X, B, Bp, d, xq, xqt, status, blockIdx.x, blockIdx.y, threadIdx.x, threadIdx.y, blockDim.y);
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

// Sum of one grad_X element over the R partial slots and the G planes, fixed
// order (deterministic): planes p = P-1 .. 0 (lo, mid, hi of the
// reference-precision split, or just the one operand plane), r = 0 .. R-1.
__device__ __forceinline__ float gx_partial_sum(const float* __restrict__ ws, int R, int d, int ld, int planes,
                                                int plane_ld, int c, int s) {
  float tot = 0.f;
  const int64_t stride = (int64_t)d * ld;
  for (int pl = planes - 1; pl >= 0; --pl) {
    const float* p = ws + (int64_t)c * ld + pl * plane_ld + s;
    float acc = 0.f;
    float v[8];
    int r = 0;
    for (; r + 8 <= R; r += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(p + (r + k) * stride);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
    for (; r < R; ++r) acc += __ldg(p + r * stride);
    tot += acc;
  }
  return tot;
}

// grad_x[s][c] (+)= scale * sum ws  (one thread per output element, block
// 32 x 32 transposed through shared memory).  A latched error of the step
// (the backward kernels were no-ops) yields NaN instead of stale partials.
__global__ void __launch_bounds__(1024) gx_reduce_kernel(const float* __restrict__ ws, int R, int d, int ld,
                                                         int planes, int plane_ld, int B, float scale, int accumulate,
                                                         const int32_t* __restrict__ status, float* __restrict__ gx) {
  __shared__ float tile[32][33];
  griddep_wait();   // launched as a PDL dependent of the last backward
  const bool bad = *status != 0;
  const int c = blockIdx.x * 32 + threadIdx.y, s = blockIdx.y * 32 + threadIdx.x;
  float acc = 0.f;
  if (s < B && !bad) acc = gx_partial_sum(ws, R, d, ld, planes, plane_ld, c, s);
  tile[threadIdx.y][threadIdx.x] = bad ? __int_as_float(0x7fc00000) : acc * scale;
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
                                                              int planes, int plane_ld, int B, float scale,
                                                              float* __restrict__ gx,
                                                              const __grid_constant__ PeerArgs pa) {
  __shared__ float tile[32][33];
  griddep_wait();
  // a rank whose step failed still takes part in the exchange (its peers wait
  // for its tiles) and pushes NaN, so every rank sees the failure
  const bool bad = *pa.status != 0;
  const int c = blockIdx.x * 32 + threadIdx.y, s = blockIdx.y * 32 + threadIdx.x;
  float acc = 0.f;
  if (s < B && !bad) acc = gx_partial_sum(ws, R, d, ld, planes, plane_ld, c, s);
  if (bad) acc = __int_as_float(0x7fc00000);
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int bid = blockIdx.y * gridDim.x + blockIdx.x;
  const int par = pa.epoch & 1;
  const int64_t slot = (static_cast<int64_t>(par) * pa.world + pa.rank) * pa.nblocks + bid;
  for (int q = 0; q < pa.world; ++q)
    __stcg(reinterpret_cast<float*>(pa.base[q]) + slot * 1024 + tid, bad ? acc : acc * scale);
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
template <int EB, int XTB = EB>
__global__ void __launch_bounds__(256) prep_count_kernel(const float* __restrict__ X, int B, int Bp, int d,
                                                         uint8_t* __restrict__ xq, uint8_t* __restrict__ xqt, int nx,
                                                         PosGeom g, const int32_t* __restrict__ ps,
                                                         const int32_t* __restrict__ pl, int64_t nnz,
                                                         int32_t* __restrict__ cnt, uint32_t* __restrict__ tmp_tile,
                                                         uint32_t* __restrict__ tmp_entry, int32_t* status) {
  griddep_wait();   // a PDL dependent of the previous step's last kernel
  if (static_cast<int>(blockIdx.x) < nx) {
    x_prep_body<EB, XTB>(X, B, Bp, d, xq, xqt, status, blockIdx.x % (d / 32), blockIdx.x / (d / 32), threadIdx.x & 31,
                    threadIdx.x >> 5, 8);
    return;
  }
  pos_count_body(g, ps, pl, nnz, cnt, tmp_tile, tmp_entry, status, blockIdx.x - nx);
}

// K2: exclusive scan of the T tile counters (one CTA; a contiguous segment
// per thread, staged in shared memory when T fits, else straight from global)
constexpr int kPosMaxTiles = 48 * 1024;
__global__ void __launch_bounds__(1024) pos_scan_kernel(int32_t* __restrict__ cnt, int32_t* __restrict__ ptr,
                                                        int32_t* __restrict__ cur, int32_t T) {
  extern __shared__ int32_t sc_smem[];   // [T] when T <= kPosMaxTiles
  __shared__ int32_t wsum[32];
  griddep_wait();   // PDL dependent of the counting pass
  const bool staged = T <= kPosMaxTiles;
  int32_t* sc = staged ? sc_smem : cnt;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, w = tid >> 5;
  if (staged)
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
    if (staged) sc[i] = pre;
    else ptr[i] = pre;
    pre += c;
  }
  if (tid == nth - 1) ptr[T] = pre;
  __syncthreads();
  for (int i = tid; i < T; i += nth) {
    const int32_t v = staged ? sc[i] : ptr[i];
    if (staged) ptr[i] = v;
    cur[i] = v;       // the scatter cursor
    cnt[i] = 0;       // counters start the next step at zero (no memset launch)
  }
}

// K3: scatter packed entries to their tile buckets (warp-aggregated cursors)
__global__ void __launch_bounds__(256) pos_scatter_kernel(int64_t nnz, const uint32_t* __restrict__ tmp_tile,
                                                          const uint32_t* __restrict__ tmp_entry,
                                                          int32_t* __restrict__ cursor, uint32_t* __restrict__ entries) {
  griddep_wait();   // PDL dependent of the scan
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

// Whole positive-list bucketing in one CTA with shared-memory counters, for
// batches of up to kPosOneCta positives: each thread loads its positives ONCE
// (kPosPer register slots), takes its slot in the tile with a shared atomic
// (the returned rank), then one block scan of the T counters gives the tile
// offsets and every entry is written straight from registers.  The order of
// entries within a tile is not fixed; the forward only ORs them into a bitmap.
// (The earlier version warp-sorted every round of tile ids for run-aggregated
// atomics and re-read the positives for the scatter: 23 us per call at
// L = 351,536 under ncu, latency- and instruction-cache-bound.)
constexpr int kPosPer = 12;
constexpr int kPosOneCta = kPosPer * 1024;
__device__ __forceinline__ void pos_bucket_body(PosGeom g, const int32_t* __restrict__ ps,
                                                const int32_t* __restrict__ pl, int64_t nnz, int32_t T,
                                                int32_t* __restrict__ tile_ptr, uint32_t* __restrict__ entries,
                                                int32_t* status) {
  extern __shared__ int32_t cnt[];    // [T]
  __shared__ int64_t cs[65], tb[65];
  __shared__ int32_t wsum[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, w = tid >> 5, nw = nth >> 5;
  for (int i = tid; i <= g.k; i += nth) {
    cs[i] = g.chunk_start[i];
    tb[i] = g.tile_base[i];
  }
  const int T4 = (T + 3) / 4;
  for (int i = tid; i < T4; i += nth) reinterpret_cast<int4*>(cnt)[i] = make_int4(0, 0, 0, 0);
  // this thread's positives i = tid + k * nth: all loads issued up front
  int32_t sv[kPosPer], lv[kPosPer];
#pragma unroll
  for (int k = 0; k < kPosPer; ++k) {
    const int64_t i = tid + static_cast<int64_t>(k) * nth;
    sv[k] = i < nnz ? ps[i] : -1;
    lv[k] = i < nnz ? pl[i] : 0;
  }
  __syncthreads();
  PosGeom sg = g;
  sg.chunk_start = cs;
  sg.tile_base = tb;
  // per positive: tr = tile << 14 | rank in the tile (T <= 48k, rank < 16k), -1 = none
  static_assert(kPosMaxTiles <= (1 << 17) && kPosOneCta <= (1 << 14), "tile / rank packing");
  int32_t tr[kPosPer];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kPosPer; ++k) {
    tr[k] = -1;
    if (tid + static_cast<int64_t>(k) * nth < nnz) {
      const int32_t smp = sv[k];
      const int64_t local = static_cast<int64_t>(lv[k]) - g.label_offset;
      if (smp < 0 || smp >= g.B) {
        bad = true;
      } else if (local >= 0 && local < g.num_local) {
        int32_t r;
        const int32_t t = static_cast<int32_t>(pos_tile(sg, local, &r));
        tr[k] = (t << 14) | atomicAdd(&cnt[t], 1);
        sv[k] = static_cast<int32_t>((static_cast<uint32_t>(r) << 16) | static_cast<uint32_t>(smp));
      }
    }
  }
  if (bad) atomicOr(status, ST_BAD_SAMPLE);
  __syncthreads();
  // exclusive scan of the T counters: a contiguous segment per thread, one
  // warp scan of the segment sums, one scan of the warp sums
  const int per = (T + nth - 1) / nth;
  const int a = min(T, tid * per), b = min(T, a + per);
  int32_t run = 0;
  for (int i = a; i < b; ++i) run += cnt[i];
  int32_t x = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t v = lane < nw ? wsum[lane] : 0;
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
    const int32_t c = cnt[i];
    cnt[i] = pre;
    tile_ptr[i] = pre;
    pre += c;
  }
  if (tid == nth - 1) tile_ptr[T] = pre;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPosPer; ++k)
    if (tr[k] >= 0) entries[cnt[tr[k] >> 14] + (tr[k] & 0x3FFF)] = static_cast<uint32_t>(sv[k]);
}

// Small batches: the whole step preparation in ONE launch.  Block 0 buckets
// the positives (pos_bucket_body, 1024 threads); blocks 1.. quantise X into Xq
// / Xq^T (x_prep_body, one 32x32 tile each).  The two jobs are independent.
template <int EB, int XTB = EB>
__global__ void __launch_bounds__(1024) prep_bucket_kernel(const float* __restrict__ X, int B, int Bp, int d,
                                                           uint8_t* __restrict__ xq, uint8_t* __restrict__ xqt,
                                                           PosGeom g, const int32_t* __restrict__ ps,
                                                           const int32_t* __restrict__ pl, int64_t nnz, int32_t T,
                                                           int32_t* __restrict__ tile_ptr,
                                                           uint32_t* __restrict__ entries, int32_t* status) {
  griddep_wait();   // a PDL dependent of the previous step's last kernel
  if (blockIdx.x == 0) {
    pos_bucket_body(g, ps, pl, nnz, T, tile_ptr, entries, status);
    return;
  }
  const int b = static_cast<int>(blockIdx.x) - 1, nxc = d / 32;
  x_prep_body<EB, XTB>(X, B, Bp, d, xq, xqt, status, b % nxc, b / nxc, threadIdx.x & 31, threadIdx.x >> 5, 32);
}

// fp32 G (rows x B, ld) -> backward operand format, [rows][Bp]:
// GQ 0 = e4m3(256 g), 1 = e5m2(256 g), 2 = bf16(g), 3 = the reference-precision
// bf16 planes hi | mid | lo (row stride 3 Bp, hi + mid + lo = g exactly)
template <int GQ>
__global__ void g_quant_kernel(const float* __restrict__ G, int64_t ld, int64_t rows, int B, int Bp,
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
    if constexpr (GQ == 0) out[i] = enc_e4m3(v * 256.0f);
    else if constexpr (GQ == 1) out[i] = enc_e5m2(v * 256.0f);
    else if constexpr (GQ == 2) reinterpret_cast<uint16_t*>(out)[i] = enc_bf16(v);
    else {
      uint16_t* o = reinterpret_cast<uint16_t*>(out) + r * 3 * Bp + s;
      const uint16_t hi = enc_bf16(v);
      const float r1 = v - dec_bf16(hi);
      const uint16_t mid = enc_bf16(r1);
      o[0] = hi;
      o[Bp] = mid;
      o[2 * Bp] = enc_bf16(r1 - dec_bf16(mid));
    }
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

}  // namespace xmc
