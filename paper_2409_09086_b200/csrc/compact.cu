// K3: in-place stable compaction, dst[i] = src[kept[i]] for i in [first, m).
//
// Replaces KvCache.gather_keep (reference cache.py:136-156: k, v, orig_pos,
// modality, round_id) and AttentionWindow.remap (policies.py:117-124).
// `kept` is strictly ascending, so kept[i] >= i: a CTA walking destination
// chunks in ascending order, loading a whole chunk's sources into registers
// before a barrier and storing after it, never overwrites a row it still has
// to read.  One CTA per (block, head) for the K/V rows (16-byte vectors, 4 per
// thread per array in flight); one extra CTA per block for token metadata and
// the window rows.  The identity prefix [0, first) is skipped.
#include "skv_common.cuh"
#include "skv_internal.h"

namespace skv {

constexpr int kCmpThreads = 512;
constexpr int kCmpUnroll = 4;

__device__ __forceinline__ int64_t kept_at(const CompactArgs& a, int b, int i) {
  return a.kept32 ? (int64_t)a.kept32[b * a.k_bs + i] : a.kept64[b * a.k_bs + i];
}

// Gather rows of `units` 16-byte vectors; two arrays moved in lockstep (y may be null).
__device__ void gather_rows16(uint4* x, uint4* y, int units, const CompactArgs& a, int b, int first, int m) {
  const int tid = threadIdx.x;
  const int rows_per_chunk = max(1, kCmpThreads * kCmpUnroll / units);
  for (int i0 = first; i0 < m; i0 += rows_per_chunk) {
    uint4 xr[kCmpUnroll], yr[kCmpUnroll];
    int dst[kCmpUnroll];
#pragma unroll
    for (int u = 0; u < kCmpUnroll; ++u) {
      const int idx = tid + u * kCmpThreads;
      const int row = i0 + idx / units;
      dst[u] = -1;
      if (idx < rows_per_chunk * units && row < m) {
        const int64_t src = kept_at(a, b, row);
        const int64_t off = src * units + idx % units;
        xr[u] = x[off];
        if (y) yr[u] = y[off];
        dst[u] = row * units + idx % units;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kCmpUnroll; ++u) {
      if (dst[u] >= 0) {
        x[dst[u]] = xr[u];
        if (y) y[dst[u]] = yr[u];
      }
    }
    __syncthreads();
  }
}

template <typename E>
__device__ void gather_elems(E* x, const CompactArgs& a, int b, int first, int m) {
  const int tid = threadIdx.x;
  const int per = kCmpThreads * kCmpUnroll;
  for (int i0 = first; i0 < m; i0 += per) {
    E r[kCmpUnroll];
#pragma unroll
    for (int u = 0; u < kCmpUnroll; ++u) {
      const int i = i0 + tid + u * kCmpThreads;
      if (i < m) r[u] = x[kept_at(a, b, i)];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kCmpUnroll; ++u) {
      const int i = i0 + tid + u * kCmpThreads;
      if (i < m) x[i] = r[u];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCmpThreads) compact_kernel(const CompactArgs a) {
  const int h = blockIdx.x, b = blockIdx.y;
  const int first = a.first_moved ? min(a.first_moved[b], a.m) : 0;
  if (h < a.heads) {
    if (first >= a.m) return;
    const int units = a.row_bytes / 16;
    uint4* kx = reinterpret_cast<uint4*>(a.k + b * a.kv_bs + h * a.kv_hs);
    uint4* vx = a.v ? reinterpret_cast<uint4*>(a.v + b * a.kv_bs + h * a.kv_hs) : nullptr;
    if (a.k_raw) {
      uint4* rx = reinterpret_cast<uint4*>(a.k_raw + b * a.kv_bs + h * a.kv_hs);
      if (a.rope_cr) {
        // cache-relative RoPE: the moved keys change position, so only the raw
        // rows move here; rope_rows_kernel re-rotates them at their new slots
        gather_rows16(rx, vx, units, a, b, first, a.m);
        return;
      }
      gather_rows16(rx, nullptr, units, a, b, first, a.m);  // original positions: rotations move as-is
    }
    gather_rows16(kx, vx, units, a, b, first, a.m);
    return;
  }
  // metadata + window rows + lengths
  if (first < a.m) {
    if (a.acc) gather_elems<float>(a.acc + b * a.acc_bs, a, b, first, a.m);  // accumulators[kept] (engine.py:335)
    if (a.pos) gather_elems<int64_t>(a.pos + b * a.m_bs, a, b, first, a.m);
    if (a.modality) gather_elems<int8_t>(a.modality + b * a.m_bs, a, b, first, a.m);
    if (a.round_id) gather_elems<int32_t>(a.round_id + b * a.m_bs, a, b, first, a.m);
  }
  if (a.rows) {
    for (int w = 0; w < a.W; ++w) {
      const int nl = a.newlen[b * a.w_bs + w];
      if (first < nl) gather_elems<float>(a.rows + b * a.r_bs + (int64_t)w * a.row_stride, a, b, first, nl);
    }
    __syncthreads();
    for (int w = threadIdx.x; w < a.W; w += blockDim.x) a.wlen[b * a.w_bs + w] = a.newlen[b * a.w_bs + w];
  }
  if (threadIdx.x == 0 && a.len) a.len[b * a.len_bs] = a.m;
}

cudaError_t launch_compact(int blocks, const CompactArgs& a, cudaStream_t st) {
  if (a.row_bytes % 16) return cudaErrorInvalidValue;
  dim3 grid(a.heads + 1, blocks);
  compact_kernel<<<grid, kCmpThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace skv
