// Probe the sm_100a hardware stochastic-rounding conversion (cvt.rs) to learn
// which bits of `rbits` drive which lane, and how many of them are used.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe tools/probe_cvt_rs.cu && ./probe
#include <cstdio>
#include <cstdint>

__global__ void k_e4m3(const float* x, const uint32_t* rb, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t r;
  asm("cvt.rs.satfinite.e4m3x4.f32 %0, {%1, %2, %3, %4}, %5;"
      : "=r"(r) : "f"(x[4 * i]), "f"(x[4 * i + 1]), "f"(x[4 * i + 2]), "f"(x[4 * i + 3]), "r"(rb[i]));
  out[i] = r;
}
__global__ void k_bf16(const float* x, const uint32_t* rb, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t r;
  asm("cvt.rs.satfinite.bf16x2.f32 %0, %1, %2, %3;" : "=r"(r) : "f"(x[2 * i]), "f"(x[2 * i + 1]), "r"(rb[i]));
  out[i] = r;
}

int main() {
  const int N = 1 << 20;
  float *x, *dx;
  uint32_t *rb, *drb, *o, *dout;
  cudaMallocHost(&x, 4 * N * 4);
  cudaMallocHost(&rb, N * 4);
  cudaMallocHost(&o, N * 4);
  cudaMalloc(&dx, 4 * N * 4);
  cudaMalloc(&drb, N * 4);
  cudaMalloc(&dout, N * 4);
  // e4m3 grid around 1.0: ulp 0.125.  x = 1 + f*0.125 in each of the 4 lanes,
  // lane l gets fraction f_l so results identify the lane.
  const float fr[4] = {0.5f, 0.5f, 0.5f, 0.5f};
  printf("e4m3x4 lane byte order and rbits bit usage (x = 1 + 0.5 ulp in all lanes):\n");
  for (int p = 0; p < 32; ++p) {
    for (int l = 0; l < 4; ++l) x[l] = 1.0f + fr[l] * 0.125f;
    rb[0] = 1u << p;
    cudaMemcpy(dx, x, 16, cudaMemcpyHostToDevice);
    cudaMemcpy(drb, rb, 4, cudaMemcpyHostToDevice);
    k_e4m3<<<1, 1>>>(dx, drb, dout, 1);
    cudaMemcpy(o, dout, 4, cudaMemcpyDeviceToHost);
    printf("  bit %2d -> result %08x\n", p, o[0]);
  }
  // distinct x per lane with rbits = 0 to identify byte order (round-down values)
  x[0] = 1.0f; x[1] = 2.0f; x[2] = 4.0f; x[3] = 8.0f;
  rb[0] = 0;
  cudaMemcpy(dx, x, 16, cudaMemcpyHostToDevice);
  cudaMemcpy(drb, rb, 4, cudaMemcpyHostToDevice);
  k_e4m3<<<1, 1>>>(dx, drb, dout, 1);
  cudaMemcpy(o, dout, 4, cudaMemcpyDeviceToHost);
  printf("  {a,b,c,d}={1,2,4,8}, rbits=0 -> %08x (e4m3 1=0x38 2=0x40 4=0x48 8=0x50)\n", o[0]);

  // statistical: fraction f in lane 0 (x = 1 + f ulp), uniform random rbits; P(up) vs f
  printf("e4m3 P(round up) vs fraction (lane a), 2^20 random rbits:\n");
  const double fs[] = {0.5, 0.25, 1.0 / 3, 0.01, 0.001, 1.0 / 256, 1.0 / 512, 1.0 / 4096, 1.0 / 65536};
  uint64_t s = 88172645463325252ull;
  for (double f : fs) {
    for (int i = 0; i < N; ++i) {
      for (int l = 0; l < 4; ++l) x[4 * i + l] = (float)(1.0 + f * 0.125);
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      rb[i] = (uint32_t)(s >> 11);
    }
    cudaMemcpy(dx, x, 16 * N, cudaMemcpyHostToDevice);
    cudaMemcpy(drb, rb, 4 * N, cudaMemcpyHostToDevice);
    k_e4m3<<<N / 256, 256>>>(dx, drb, dout, N);
    cudaMemcpy(o, dout, 4 * N, cudaMemcpyDeviceToHost);
    long up[4] = {0, 0, 0, 0};
    for (int i = 0; i < N; ++i)
      for (int l = 0; l < 4; ++l) up[l] += ((o[i] >> (8 * l)) & 0xFF) == 0x39;
    printf("  f=%.6g  P(up) bytes[0..3] = %.6f %.6f %.6f %.6f\n", f, up[0] / (double)N, up[1] / (double)N,
           up[2] / (double)N, up[3] / (double)N);
  }
  printf("bf16x2 rbits bit usage (x = 1 + 0.5 ulp, ulp 2^-7):\n");
  for (int p = 0; p < 32; ++p) {
    x[0] = x[1] = 1.0f + 0.5f / 128.0f;
    rb[0] = 1u << p;
    cudaMemcpy(dx, x, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(drb, rb, 4, cudaMemcpyHostToDevice);
    k_bf16<<<1, 1>>>(dx, drb, dout, 1);
    cudaMemcpy(o, dout, 4, cudaMemcpyDeviceToHost);
    printf("  bit %2d -> result %08x\n", p, o[0]);
  }
  printf("bf16 P(up) vs fraction, random rbits:\n");
  for (double f : fs) {
    for (int i = 0; i < N; ++i) {
      x[2 * i] = x[2 * i + 1] = (float)(1.0 + f / 128.0);
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      rb[i] = (uint32_t)(s >> 11);
    }
    cudaMemcpy(dx, x, 8 * N, cudaMemcpyHostToDevice);
    cudaMemcpy(drb, rb, 4 * N, cudaMemcpyHostToDevice);
    k_bf16<<<N / 256, 256>>>(dx, drb, dout, N);
    cudaMemcpy(o, dout, 4 * N, cudaMemcpyDeviceToHost);
    long up[2] = {0, 0};
    for (int i = 0; i < N; ++i)
      for (int l = 0; l < 2; ++l) up[l] += ((o[i] >> (16 * l)) & 0xFFFF) == 0x3F81;
    printf("  f=%.6g  P(up) halves[0,1] = %.6f %.6f\n", f, up[0] / (double)N, up[1] / (double)N);
  }
  return 0;
}
