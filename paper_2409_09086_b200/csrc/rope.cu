// Rotary positions (the reference Session's rotary helpers, engine.py:198-233,
// and _refresh_rotations, engine.py:339-342) for the RoPE-enabled engine.
//
// The cache keeps two key stores: the raw keys (KvCache's storage, what
// cache.keys() returns) and the rotated keys the decode and prefill kernels
// attend over (the Session's `_rot` store).  Rotation is the reference's
// interleaved pairing with f32 products and a separate f32 add/sub (NumPy
// `even * cos - odd * sin`, no FMA contraction); cos/sin come from the f64
// angle `pos * inv_freq[i]` rounded to f32, inv_freq = base^(-2i/D) in f64
// (engine.py:176-178, 200-207).
//
//   * rope_tokens_kernel: q and the new k of a decode step / prefill chunk,
//     at the cache-relative slot (n-1, engine.py:266) or the original
//     position (global stream position);
//   * rope_rows_kernel: rows [r0, r1) of every (block, head) segment from the
//     raw store into the rotated store -- the cache-relative re-rotation after
//     a compaction (positions = slot index, fused after K3's raw gather) and
//     state injection.
#include <cuda_bf16.h>

#include <algorithm>

#include "skv_common.cuh"
#include "skv_internal.h"

namespace skv {

template <typename T>
__device__ __forceinline__ void rot_store(T* dst, float e, float o, float c, float s);

template <>
__device__ __forceinline__ void rot_store<float>(float* dst, float e, float o, float c, float s) {
  dst[0] = __fsub_rn(__fmul_rn(e, c), __fmul_rn(o, s));
  dst[1] = __fadd_rn(__fmul_rn(e, s), __fmul_rn(o, c));
}

template <>
__device__ __forceinline__ void rot_store<__nv_bfloat16>(__nv_bfloat16* dst, float e, float o, float c, float s) {
  const float re = __fsub_rn(__fmul_rn(e, c), __fmul_rn(o, s));
  const float ro = __fadd_rn(__fmul_rn(e, s), __fmul_rn(o, c));
  *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(re, ro);
}

// cos/sin of pair i at position p: the cache-relative table when p < tab_rows
// (positions are slot indices there), else f64 on the fly
__device__ __forceinline__ void rope_cs(const RopeArgs& a, int64_t p, int i, float& c, float& s) {
  if (a.tcos && p < a.tab_rows) {
    c = a.tcos[p * (a.D / 2) + i];
    s = a.tsin[p * (a.D / 2) + i];
  } else {
    double sd, cd;
    sincos((double)p * a.inv_freq[i], &sd, &cd);
    c = (float)cd;
    s = (float)sd;
  }
}

// grid (T tokens, S streams); q/k inputs [S][T][H][D] (stream stride q_ss/k_ss
// elements), outputs with the same layout
template <typename T>
__global__ void rope_tokens_kernel(const RopeArgs a) {
  const int t = blockIdx.x, s = blockIdx.y;
  const int half = a.D / 2;
  int64_t p;
  if (a.mode == 1) {
    p = a.pos0 + t;
  } else {
    p = (a.pos_in ? a.pos_in[s] : a.next_pos[s * a.np_ss]) + t;
  }
  const int pairs = (a.Hq + a.Hkv) * half;
  for (int x = threadIdx.x; x < pairs; x += blockDim.x) {
    const int hh = x / half, i = x - hh * half;
    float c, sn;
    rope_cs(a, p, i, c, sn);
    const T* src;
    T* dst;
    if (hh < a.Hq) {
      const int64_t off = s * a.q_ss + ((int64_t)t * a.Hq + hh) * a.D + 2 * i;
      src = static_cast<const T*>(a.q) + off;
      dst = static_cast<T*>(a.qr) + off;
    } else {
      const int64_t off = s * a.k_ss + ((int64_t)t * a.Hkv + (hh - a.Hq)) * a.D + 2 * i;
      src = static_cast<const T*>(a.k) + off;
      dst = static_cast<T*>(a.kr) + off;
    }
    rot_store<T>(dst, to_f32(src[0]), to_f32(src[1]), c, sn);
  }
}

// grid (heads, blocks); rows [r0_b, r1) of segment (b, h): rotated[row] =
// rope(raw[row], position), position = row (cache-relative) or pos[b][row]
template <typename T>
__global__ void rope_rows_kernel(const RopeRowsArgs a) {
  const int h = blockIdx.x, b = blockIdx.y;
  const int r0 = a.first ? min(a.first[b], a.r1) : a.r0;
  const int half = a.D / 2;
  const T* raw = static_cast<const T*>(a.raw) + b * a.bs + h * a.hs;
  T* rot = static_cast<T*>(a.rot) + b * a.bs + h * a.hs;
  const int64_t total = (int64_t)(a.r1 - r0) * half;
  for (int64_t x = threadIdx.x; x < total; x += blockDim.x) {
    const int row = r0 + (int)(x / half), i = (int)(x % half);
    const int64_t p = a.pos ? a.pos[b * a.pos_bs + row] : row;
    float c, sn;
    rope_cs(a.ra, p, i, c, sn);
    const T* src = raw + (int64_t)row * a.D + 2 * i;
    rot_store<T>(rot + (int64_t)row * a.D + 2 * i, to_f32(src[0]), to_f32(src[1]), c, sn);
  }
}

cudaError_t launch_rope_tokens(int dtype, int tokens, int streams, const RopeArgs& a, cudaStream_t st) {
  dim3 grid(tokens, streams);
  if (dtype == 1)
    rope_tokens_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(a);
  else
    rope_tokens_kernel<float><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rope_rows(int dtype, int heads, int blocks, const RopeRowsArgs& a, cudaStream_t st) {
  dim3 grid(heads, blocks);
  if (dtype == 1)
    rope_rows_kernel<__nv_bfloat16><<<grid, 512, 0, st>>>(a);
  else
    rope_rows_kernel<float><<<grid, 512, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace skv
