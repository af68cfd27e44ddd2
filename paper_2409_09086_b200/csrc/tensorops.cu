// Single-row attention primitives of the reference's tensorops module
// (/root/reference/pkg/src/streamkv/tensorops.py:26-111) on the device, with
// the reference's float32 operation order:
//   softmax_row  (26-35):  z = x - max(x); e = exp(z); e / sum(e)  (f32 sum)
//   attn_probs   (86-102): logits = (K @ q) * f32(scale); softmax_row(logits)
//   weighted_sum (105-111): p @ V
//   rope_apply   (38-64):  pair i rotated by f32(cos/sin(position * base^(-2i/dim))),
//                          angles in float64
// These back the drop-in functions (tensorops.py of this package); the engine's
// hot path fuses the same arithmetic into K1.  Input validation (shapes,
// non-finite entries) happens on the host, exactly where the reference raises.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/streamkv_b200.h"
#include "skv_internal.h"

namespace skv {

constexpr int kRowThreads = 1024;

__device__ float block_reduce(float v, float* red, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float y = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, y) : __fadd_rn(v, y);
  }
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? red[lane] : (is_max ? -INFINITY : 0.f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float y = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, y) : __fadd_rn(v, y);
    }
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const float r = red[0];
  __syncthreads();
  return r;
}

// logits (optional: computed as (K @ q) * scale first), then softmax in place
// into out[0, n).  One CTA; n is small (one attention row).
__global__ void __launch_bounds__(kRowThreads) softmax_row_kernel(const float* __restrict__ x, const float* __restrict__ q,
                                                                 const float* __restrict__ keys, int n, int dim,
                                                                 float scale, float* __restrict__ out) {
  __shared__ float red[32];
  if (keys) {  // logits[i] = dot(K[i], q) (sequential f32 over dim) * scale
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const float* k = keys + (int64_t)i * dim;
      float acc = 0.f;
      for (int d = 0; d < dim; ++d) acc = __fmaf_rn(k[d], q[d], acc);
      out[i] = __fmul_rn(acc, scale);
    }
    __syncthreads();
    x = out;
  }
  float m = -INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, x[i]);
  m = block_reduce(m, red, true);
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float e = expf(__fsub_rn(x[i], m));
    out[i] = e;
    s = __fadd_rn(s, e);
  }
  s = block_reduce(s, red, false);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = __fdiv_rn(out[i], s);
}

// out[d] = sum_i p[i] * V[i][d]: thread d walks the rows (coalesced across d).
__global__ void weighted_sum_kernel(const float* __restrict__ p, const float* __restrict__ v, int n, int dim,
                                    float* __restrict__ out) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= dim) return;
  float acc = 0.f;
  for (int i = 0; i < n; ++i) acc = __fmaf_rn(p[i], v[(int64_t)i * dim + d], acc);
  out[d] = acc;
}

// rope_apply: freqs (f64, from the host's libm like numpy) -> angle in f64 ->
// f32 cos / sin -> the reference's even/odd pair products in f32.
__global__ void rope_apply_kernel(const float* __restrict__ v, int half, const double* __restrict__ freqs,
                                  double position, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= half) return;
  const double ang = position * freqs[i];
  const float c = (float)cos(ang), s = (float)sin(ang);
  const float e = v[2 * i], o = v[2 * i + 1];
  out[2 * i] = __fsub_rn(__fmul_rn(e, c), __fmul_rn(o, s));
  out[2 * i + 1] = __fadd_rn(__fmul_rn(e, s), __fmul_rn(o, c));
}

// aggregate_heads (policies.py:259-265): mean = sequential f32 head sum / f32(H)
// (numpy's axis-0 reduction order), max = elementwise max over heads.
__global__ void aggregate_heads_kernel(const float* __restrict__ p, int H, int n, int mode, float* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float acc = p[j];
  for (int h = 1; h < H; ++h) {
    const float x = p[(int64_t)h * n + j];
    acc = mode ? fmaxf(acc, x) : __fadd_rn(acc, x);
  }
  out[j] = mode ? acc : __fdiv_rn(acc, (float)H);
}

// bias_vector (policies.py:150-162): d = f32(b) / f32(cols), out[c] = (-d) * f32(cols - 1 - c).
__global__ void bias_vector_kernel(int cols, float b, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const float d = __fdiv_rn(b, (float)cols);
  out[c] = __fmul_rn(-d, (float)(cols - 1 - c));
}

}  // namespace skv

using namespace skv;

namespace {
int tfail(int code, const char* msg) { return set_error(code, msg); }  // skv_last_error()
}  // namespace

extern "C" {

int skv_softmax_row(const float* logits_dev, int n, float* out_dev, void* stream) {
  if (n < 1 || !logits_dev || !out_dev) return tfail(SKV_EINVAL, "logits must be a non-empty 1-D vector");
  softmax_row_kernel<<<1, kRowThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(logits_dev, nullptr, nullptr, n,
                                                                                     0, 1.f, out_dev);
  return cudaGetLastError() == cudaSuccess ? SKV_OK : tfail(SKV_ECUDA, "softmax kernel launch");
}

int skv_attn_probs(const float* q_dev, const float* keys_dev, int n, int dim, float scale, float* out_dev,
                   void* stream) {
  if (n < 1 || dim < 1 || !q_dev || !keys_dev || !out_dev)
    return tfail(SKV_EINVAL, "keys must be a non-empty sequence of vectors");
  if (!(scale > 0.f)) return tfail(SKV_EINVAL, "scale must be positive");
  softmax_row_kernel<<<1, kRowThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(nullptr, q_dev, keys_dev, n, dim,
                                                                                     scale, out_dev);
  return cudaGetLastError() == cudaSuccess ? SKV_OK : tfail(SKV_ECUDA, "attn_probs kernel launch");
}

int skv_weighted_sum(const float* probs_dev, const float* values_dev, int n, int dim, float* out_dev, void* stream) {
  if (n < 1 || dim < 1 || !probs_dev || !values_dev || !out_dev) return tfail(SKV_EINVAL, "bad weighted_sum shapes");
  weighted_sum_kernel<<<(dim + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(probs_dev, values_dev, n,
                                                                                              dim, out_dev);
  return cudaGetLastError() == cudaSuccess ? SKV_OK : tfail(SKV_ECUDA, "weighted_sum kernel launch");
}

int skv_aggregate_heads(const float* probs_dev, int heads, int n, int mode, float* out_dev, void* stream) {
  if (heads < 1 || n < 1 || !probs_dev || !out_dev) return tfail(SKV_EINVAL, "per-head block must be non-empty");
  if (mode != SKV_AGG_MEAN && mode != SKV_AGG_MAX) return tfail(SKV_EINVAL, "unknown head aggregation");
  aggregate_heads_kernel<<<(n + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(probs_dev, heads, n,
                                                                                               mode, out_dev);
  return cudaGetLastError() == cudaSuccess ? SKV_OK : tfail(SKV_ECUDA, "aggregate kernel launch");
}

int skv_bias_vector(int n, int recent_len, float bias, float* out_dev, void* stream) {
  if (n <= recent_len) return tfail(SKV_EINVAL, "no scorable columns: n <= l");
  if (!(bias >= 0.f)) return tfail(SKV_EINVAL, "bias must be >= 0");
  const int cols = n - recent_len;
  bias_vector_kernel<<<(cols + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(cols, bias, out_dev);
  return cudaGetLastError() == cudaSuccess ? SKV_OK : tfail(SKV_ECUDA, "bias kernel launch");
}

int skv_rope_apply(const float* v_dev, int dim, int64_t position, double base, float* out_dev, void* stream) {
  if (dim < 2 || dim % 2) return tfail(SKV_EINVAL, "rope_apply requires an even-dimensional vector");
  if (position < 0) return tfail(SKV_EINVAL, "position must be non-negative");
  if (!(base > 1.0)) return tfail(SKV_EINVAL, "base must be > 1");
  const int half = dim / 2;
  std::vector<double> f(half);
  for (int i = 0; i < half; ++i) f[i] = std::pow(base, -2.0 * i / dim);  // base ** (-2 i / dim), f64
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double* fd = nullptr;
  if (cudaMallocAsync(&fd, half * sizeof(double), st) != cudaSuccess) return tfail(SKV_ENOMEM, "rope scratch");
  cudaMemcpyAsync(fd, f.data(), half * sizeof(double), cudaMemcpyHostToDevice, st);
  rope_apply_kernel<<<(half + 127) / 128, 128, 0, st>>>(v_dev, half, fd, (double)position, out_dev);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(fd, st);
  if (cudaStreamSynchronize(st) != cudaSuccess || e != cudaSuccess) return tfail(SKV_ECUDA, "rope_apply kernel");
  return SKV_OK;
}

}  // extern "C"
