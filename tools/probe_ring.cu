// Producer/consumer ring probe (measurement tool, not product code): how long
// does one slot cycle of the backward's pipeline take without its math?
// One CTA per SM; warp 0 = TMA producer (one 16 KB box per slot), warp 1 =
// "MMA" consumer, warps 2..17 = "epilogue" consumers.  Modes:
//   0  consumer waits full, releases the slot with a plain mbarrier arrive
//   1  consumer releases with tcgen05.commit (no MMAs issued)
//   2  mode 1 + the 16 epilogue warps wait a commit-signalled t_full and
//      also arrive on the slot's empty barrier (1 + 16 arrivals, as the bwd)
//   3  mode 2 + real MMAs per slot (M=128 N=128 K=256 fp8, 8 instructions)
// Reports cycles per slot (clock64 on the producer) for ring depths 3 and 6,
// from a DRAM-sized buffer and an L2-resident one.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_ring tools/probe_ring.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#include "../paper_2510_11168_b200/csrc/xmc_ptx.cuh"

using namespace xmc;

constexpr int kEpi = 16;

__global__ void __launch_bounds__(64 + kEpi * 32, 1) ring(const __grid_constant__ CUtensorMap tm, int mode, int S,
                                                          int iters, int64_t row_tiles, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mode >= 2 ? 1 + kEpi : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpi);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // B operand for the MMAs: a fixed 32 KB region after the ring
  uint8_t* bsm = smem + S * 16384;
  if (warp == 0) {
    if (lane == 0) {
      long long t0 = 0;
      int64_t t = blockIdx.x;
      for (int i = 0; i < iters; ++i) {
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
        if (i == 2 * S) t0 = clock64();
        mbar_arrive_expect_tx(&full[s], 16384);
        tma_load_2d(smem + s * 16384, &tm, &full[s], 0, static_cast<int32_t>(t * 128));
        t = (t + gridDim.x) % row_tiles;
      }
      out[blockIdx.x] = (clock64() - t0) / (iters - 2 * S);
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = umma_idesc(0, 0, false, false, 128, 128);
    for (int i = 0; i < iters; ++i) {
      const int s = i % S, ds = i & 1;
      mbar_wait(&full[s], (i / S) & 1);
      if (mode >= 2) mbar_wait(&tempty[ds], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        if (mode == 0) {
          mbar_arrive(&empty[s]);
        } else {
          if (mode == 3) {
            const uint32_t a = smem_u32(smem + s * 16384), b = smem_u32(bsm);
            for (int k = 0; k < 8; ++k)
              mma_f8(tmem + ds * 128, umma_desc_sw128(a + (k & 3) * 32, 16, 1024),
                     umma_desc_sw128(b + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024), idesc, k != 0);
          }
          if (mode >= 2) mma_commit(&tfull[ds]);
          mma_commit(&empty[s]);
        }
      }
      __syncwarp();
    }
  } else if (mode >= 2) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % S, ds = i & 1;
      mbar_wait(&full[s], (i / S) & 1);
      mbar_wait(&tfull[ds], (i >> 1) & 1);
      tc_fence_after();
      if (mode == 3) {
        uint32_t r[32];
        tmem_ld32(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + ds * 128 + ((warp - 2) >> 2) * 32, r);
        tmem_ld_wait();
        if (r[0] == 0x7fffffffu && r[31] == 1u) out[gridDim.x] = r[5];   // keep the load alive
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty[ds]);
        mbar_arrive(&empty[s]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN_encodeTiled enc = reinterpret_cast<PFN_encodeTiled>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t pitch = 768;
  uint8_t* buf;
  const int64_t big = 2000000, small = 16384;
  cudaMalloc(&buf, big * pitch);
  cudaMemset(buf, 0x11, big * pitch);
  long long* out;
  cudaMalloc(&out, (sms + 1) * 8);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[4] = {"plain arrive", "tcgen05.commit", "commit + 16 epi warps", "commit + epi + MMAs"};
  for (int src = 0; src < 2; ++src) {
    const int64_t rows = src == 0 ? big : small;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 0; mode < 4; ++mode) {
      for (int S : {3, 6}) {
        const int smem = S * 16384 + 32768 + 1024;
        ring<<<sms, 64 + kEpi * 32, smem>>>(tm, mode, S, 200, rows / 128, out);
        ring<<<sms, 64 + kEpi * 32, smem>>>(tm, mode, S, 2000, rows / 128, out);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[256];
        cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        printf("%-5s %-24s S=%d: %6.0f cycles per slot (%5.1f B/clk/SM) %s\n", src == 0 ? "DRAM" : "L2", names[mode],
               S, avg, 16384.0 / avg, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
