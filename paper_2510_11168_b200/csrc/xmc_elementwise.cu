// Elementwise numeric core of the C ABI (formats.py / optimizers.py / rng.py
// restated bit-exactly on the GPU) plus the standalone logit_gradient,
// dropout_mask and native RTN cast entry points.  Every kernel here is a
// grid-stride loop over independent elements; the fp64 grid arithmetic and
// the splitmix64 draws reproduce the reference's numbers exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "xmc_common.cuh"
#include "xmc_round.cuh"

using namespace xmc;

#define fail xmc_fail

static int ew_blocks(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8192))); }

constexpr uint64_t kDropoutTag = 0xbfe79d70c7098ab2ull;   // tensor_tag("head.dropout"), head.py:43

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
  dropout_mask_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      row0, row1 - row0, num_cols, sm64_base(seed, step, kDropoutTag),
      static_cast<uint64_t>(std::ceil(p * 9007199254740992.0)), keep);
  CUDA_TRY(cudaGetLastError());
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
  int32_t* status = xmc_device_scratch_status();
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
  int32_t* status = xmc_device_scratch_status();
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
  int32_t* stw = status ? status : xmc_device_scratch_status();
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
  int32_t* status = xmc_device_scratch_status();
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
  int32_t* status = xmc_device_scratch_status();
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
