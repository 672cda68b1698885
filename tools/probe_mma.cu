// Throughput probe for tcgen05.mma operand majorness on sm_100a (measurement
// tool, not product code).  One CTA per SM, one thread issues `iters` MMAs into
// one TMEM accumulator from shared-memory operands; clock64 / globaltimer
// around issue + commit wait.  Compares K-major vs MN-major A/B for
// kind::f8f6f4 (K = 32) and kind::f16 (K = 16) at several N.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_mma tools/probe_mma.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2510_11168_b200/csrc/xmc_ptx.cuh"

using namespace xmc;

template <int KIND>  // 0: f8f6f4, 1: f16
__global__ void __launch_bounds__(128, 1) probe(int iters, uint32_t idesc, int a_mn, int b_mn, int n_blocks,
                                                long long* out_clk, unsigned long long* out_ns) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  // operand bytes: fill with small finite values (0x38 = e4m3 1.0 / bf16 pattern)
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x30383038u ^ (i * 2654435761u & 0x01010101u);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 64 * 1024);
  long long t0 = 0, t1 = 0;
  unsigned long long g0 = 0, g1 = 0;
  if (threadIdx.x < 32) {
    if (elect_one()) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        const int k = i & 3;
        // K-major: advance 32 B inside the 128-B atom; MN-major: advance
        // 8-row (K) groups of 1024 B  (layouts only need to be in range)
        const uint32_t ao = a_mn ? (k * 4096) : (k * 32);
        const uint32_t bo = b_mn ? (k * 4096) : (k * 32);
        const uint64_t ad = umma_desc_sw128(a0 + ao, a_mn ? 16384 : 16, 1024);
        const uint64_t bd = umma_desc_sw128(b0 + bo, b_mn ? 16384 : 16, 1024);
        if (KIND == 0) mma_f8(tmem, ad, bd, idesc, i != 0);
        else mma_f16(tmem, ad, bd, idesc, i != 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (elect_one()) {
      t1 = clock64();
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
      out_clk[blockIdx.x] = t1 - t0;
      out_ns[blockIdx.x] = g1 - g0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk;
  unsigned long long* ns;
  cudaMalloc(&clk, sms * 8);
  cudaMalloc(&ns, sms * 8);
  const int smem = 161 * 1024;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Case { int kind, M, N, amn, bmn; };
  const Case cases[] = {
      {0, 128, 256, 0, 0}, {0, 128, 256, 1, 0}, {0, 128, 256, 0, 1}, {0, 128, 256, 1, 1},
      {0, 128, 128, 0, 0}, {0, 128, 128, 1, 1}, {0, 128, 64, 0, 0},  {0, 128, 32, 0, 0},
      {1, 128, 256, 0, 0}, {1, 128, 256, 1, 1}, {1, 128, 128, 0, 0}, {1, 128, 128, 1, 1},
  };
  const int iters = 8192;
  for (const Case& c : cases) {
    const uint32_t idesc = c.kind == 0 ? umma_idesc(0, 0, c.amn, c.bmn, c.M, c.N) : umma_idesc(1, 1, c.amn, c.bmn, c.M, c.N);
    for (int rep = 0; rep < 2; ++rep) {
      if (c.kind == 0) probe<0><<<sms, 128, smem>>>(iters, idesc, c.amn, c.bmn, 1, clk, ns);
      else probe<1><<<sms, 128, smem>>>(iters, idesc, c.amn, c.bmn, 1, clk, ns);
    }
    cudaError_t e = cudaDeviceSynchronize();
    long long hc[256];
    unsigned long long hn[256];
    cudaMemcpy(hc, clk, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hn, ns, sms * 8, cudaMemcpyDeviceToHost);
    long long mc = 0;
    unsigned long long mn = 0;
    for (int i = 0; i < sms; ++i) { if (hc[i] > mc) mc = hc[i]; if (hn[i] > mn) mn = hn[i]; }
    const int K = c.kind == 0 ? 32 : 16;
    const double flop = 2.0 * c.M * c.N * K * iters;
    printf("%s M=%d N=%3d A%s B%s: %.0f flop/clk/SM, %.1f TFLOP/s (148 SMs, %.2f GHz eff) %s\n",
           c.kind == 0 ? "f8 " : "f16", c.M, c.N, c.amn ? "-MN" : "-K ", c.bmn ? "-MN" : "-K ",
           flop / mc, flop * sms / (mn * 1e-9) / 1e12, (double)mc / mn, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
