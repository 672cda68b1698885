// TMA load-throughput probe (measurement tool, not product code).  Every CTA
// (one per SM) streams boxes of a [rows][pitch] uint8 matrix into a ring of
// smem stages with one thread; a stage is re-issued once its previous load
// landed.  Reports bytes/clk/SM and chip TB/s for several box shapes, from a
// DRAM-sized buffer and from an L2-resident one.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_tma tools/probe_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#include "../paper_2510_11168_b200/csrc/xmc_ptx.cuh"

using namespace xmc;

XMC_DEV void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// mode 0: 2-D boxes [box_rows][128 B] at column chunk `chunk`, rows advance
// mode 1: 3-D box [nchunk][box_rows][128 B] (all column chunks of box_rows rows)
__global__ void __launch_bounds__(256, 1) stream(const __grid_constant__ CUtensorMap tm, int mode, int box_rows,
                                                int nchunk, int stages, int box_bytes, int64_t rows, int iters,
                                                long long* clk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[16];
  // lanes_mode: producers are lanes 0..nprod-1 of warp 0 instead of one lane per warp
  const bool lanes_mode = gridDim.y >= 2;
  const int nprod = lanes_mode ? static_cast<int>(gridDim.y) : blockDim.x / 32,
            w = lanes_mode ? (threadIdx.x & 31) : threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 16; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (lanes_mode ? (static_cast<int>(threadIdx.x) >= nprod) : ((threadIdx.x & 31) != 0)) return;
  if (blockIdx.y != 0) return;
  // warp w of nprod issues every nprod-th box into its own share of the stages
  stages /= nprod;
  smem += w * stages * box_bytes;
  uint64_t* mybars = bars + w * stages;
  iters /= nprod;
  const int64_t row_tiles = rows / box_rows;
  int64_t t = blockIdx.x * nprod + w;
  int chunk = 0;
  long long t0 = 0;
  for (int i = 0; i < iters + stages; ++i) {
    const int s = i % stages;
    if (mode == 2) {   // TMA stores of smem stage s, at most `stages` groups outstanding
      if (i == stages) t0 = clock64();
      if (i >= iters) break;
      if (i >= stages) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(7) : "memory");
      tma_store_2d(&tm, smem + s * box_bytes, chunk * 128, static_cast<int32_t>(t * box_rows));
      bulk_commit();
      if (++chunk == nchunk) { chunk = 0; t = (t + gridDim.x * nprod) % row_tiles; }
      continue;
    }
    if (i >= stages) mbar_wait(&mybars[s], ((i / stages) - 1) & 1);
    if (i == stages) t0 = clock64();
    if (i >= iters) continue;
    mbar_arrive_expect_tx(&mybars[s], box_bytes);
    uint8_t* dst = smem + s * box_bytes;
    if (mode == 0) {
      tma_load_2d(dst, &tm, &mybars[s], chunk * 128, static_cast<int32_t>(t * box_rows));
      if (++chunk == nchunk) { chunk = 0; t = (t + gridDim.x * nprod) % row_tiles; }
    } else {
      tma_load_3d(dst, &tm, &mybars[s], 0, static_cast<int32_t>(t * box_rows), 0);
      t = (t + gridDim.x * nprod) % row_tiles;
    }
  }
  if (mode == 2) bulk_wait<0>();
  if (w == 0) clk[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int sweep(PFN_encodeTiled enc, uint8_t* buf, long long* clk, int sms);
int main(int argc, char** argv) {
  if (argc > 1) {
    void* p0 = nullptr;
    cudaDriverEntryPointQueryResult q0;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p0, cudaEnableDefault, &q0);
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* b;
    cudaMalloc(&b, 2000000ll * 768);
    cudaMemset(b, 0x11, 2000000ll * 768);
    long long* c;
    cudaMalloc(&c, n * 8);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    return sweep(reinterpret_cast<PFN_encodeTiled>(p0), b, c, n);
  }
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN_encodeTiled enc = reinterpret_cast<PFN_encodeTiled>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t pitch = 768;
  const int64_t big_rows = 2000000, small_rows = 32768;   // 1.5 GB (DRAM) and 24 MB (L2)
  uint8_t* buf;
  cudaMalloc(&buf, big_rows * pitch);
  cudaMemset(buf, 0x11, big_rows * pitch);
  long long* clk;
  cudaMalloc(&clk, sms * 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Case { int mode, box_rows, nchunk, stages; int64_t rows; const char* what; int nprod; };
  const Case cases[] = {
      {0, 128, 6, 12, small_rows, "L2: 2D 128Bx128 rows, 6 chunks, 1 producer", 1},
      {0, 128, 6, 12, small_rows, "L2: 2D 128Bx128 rows, 6 chunks, 4 LANES of one warp", -4},
      {0, 32, 6, 16, small_rows, "L2: 2D 128Bx32 rows, 4 LANES of one warp", -4},
      {0, 128, 6, 12, small_rows, "L2: 2D 128Bx128 rows, 6 chunks, 2 producers", 2},
      {0, 128, 6, 12, small_rows, "L2: 2D 128Bx128 rows, 6 chunks, 4 producers", 4},
      {0, 32, 6, 16, small_rows, "L2: 2D 128Bx32 rows, 1 producer", 1},
      {0, 32, 6, 16, small_rows, "L2: 2D 128Bx32 rows, 4 producers", 4},
      {1, 128, 2, 6, small_rows, "L2: 3D 2x128x128B (32 KB: a G tile)", 1},
      {1, 128, 6, 2, small_rows, "L2: 3D 6x128x128B", 1},
      {1, 128, 6, 2, small_rows, "L2: 3D 6x128x128B, 2 producers", 2},
      {0, 128, 6, 12, big_rows, "DRAM: 2D 128Bx128 rows, 1 producer", 1},
      {0, 128, 6, 12, big_rows, "DRAM: 2D 128Bx128 rows, 4 producers", 4},
      {1, 128, 6, 2, big_rows, "DRAM: 3D 6x128x128B", 1},
      {1, 128, 2, 6, big_rows, "DRAM: 3D 2x128x128B", 1},
      {2, 32, 6, 8, big_rows, "DRAM store: 2D 128Bx32 rows (4 KB)", 1},
      {2, 128, 6, 8, big_rows, "DRAM store: 2D 128Bx128 rows (16 KB)", 1},
      {2, 32, 6, 8, big_rows, "DRAM store: 2D 128Bx32 rows (4 KB), 4 producers", 4},
  };
  for (const Case& c : cases) {
    CUtensorMap tm;
    CUresult r;
    int box_bytes;
    if (c.mode != 1) {
      cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)c.rows};
      cuuint64_t strides[1] = {(cuuint64_t)pitch};
      cuuint32_t box[2] = {128, (cuuint32_t)c.box_rows};
      cuuint32_t es[2] = {1, 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      box_bytes = 128 * c.box_rows;
    } else {
      cuuint64_t dims[3] = {128, (cuuint64_t)c.rows, (cuuint64_t)(pitch / 128)};
      cuuint64_t strides[2] = {(cuuint64_t)pitch, 128};
      cuuint32_t box[3] = {128, (cuuint32_t)c.box_rows, (cuuint32_t)c.nchunk};
      cuuint32_t es[3] = {1, 1, 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      box_bytes = 128 * c.box_rows * c.nchunk;
    }
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.what, (int)r); continue; }
    const int iters = static_cast<int>((64ll << 20) / box_bytes);   // 64 MB per CTA
    const int smem = c.stages * box_bytes + 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const dim3 grid(sms, c.nprod < 0 ? 2 : 1);
    const int thr = c.nprod < 0 ? 32 : 32 * c.nprod;
    stream<<<grid, thr, smem>>>(tm, c.mode, c.box_rows, c.nchunk, c.stages, box_bytes, c.rows, iters / 8, clk);
    cudaEventRecord(a);
    stream<<<grid, thr, smem>>>(tm, c.mode, c.box_rows, c.nchunk, c.stages, box_bytes, c.rows, iters, clk);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long hc[256];
    cudaMemcpy(hc, clk, sms * 8, cudaMemcpyDeviceToHost);
    long long mc = 0;
    for (int i = 0; i < sms; ++i) mc = hc[i] > mc ? hc[i] : mc;
    const double bytes = (double)iters * box_bytes;
    printf("%-70s stages %2d: %6.1f B/clk/SM, %6.2f TB/s chip %s\n", c.what, c.stages, bytes / mc,
           bytes * sms / (ms * 1e-3) / 1e12, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}

// in-flight sweep: per-SM bytes/clk for 1..16 concurrently issuing lanes with a
// 12-deep ring of 16 KB boxes, on 1 SM and on all SMs, L2-resident and DRAM
int sweep(PFN_encodeTiled enc, uint8_t* buf, long long* clk, int sms) {
  for (int src = 0; src < 2; ++src) {
    const int64_t rows = src == 0 ? 2000000 : 32768;
    CUtensorMap tm;
    cuuint64_t dims[2] = {768, (cuuint64_t)rows};
    cuuint64_t strides[1] = {768};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int g : {1, 16, 74, sms})
      for (int lanes : {2, 4, 8, 12}) {
        const int stages = 12, box_bytes = 16384;
        const int iters = 4096;
        const dim3 grid(g, lanes);
        stream<<<grid, 32, stages * box_bytes + 1024>>>(tm, 0, 128, 6, stages, box_bytes, rows, iters / 8, clk);
        stream<<<grid, 32, stages * box_bytes + 1024>>>(tm, 0, 128, 6, stages, box_bytes, rows, iters, clk);
        cudaError_t e = cudaDeviceSynchronize();
        long long hc[256];
        cudaMemcpy(hc, clk, g * 8, cudaMemcpyDeviceToHost);
        long long mc = 0;
        for (int i = 0; i < g; ++i) mc = hc[i] > mc ? hc[i] : mc;
        const double bytes = (double)(iters / lanes) * lanes * box_bytes;
        printf("%-4s grid %3d lanes %2d (<= %3d KB in flight): %6.1f B/clk/SM, %6.2f TB/s chip-equiv %s\n",
               src == 0 ? "DRAM" : "L2", g, lanes, lanes * 16, bytes / mc, bytes / mc * g * 1.9e9 / 1e12,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  }
  return 0;
}
