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
//
// Slot-map engines (CompactArgs::moves) skip the stable shift altogether: the
// selection kernel planned which kept rows must move (at most the tokens
// appended since the last eviction), each row moves once from a source row
// >= m to a free destination row < m, and the logical order lives in the slot
// map.  Token metadata and window lengths are still gathered in logical order.
#include <algorithm>

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

// Planned row moves (src -> dst, disjoint): each thread copies 16-byte units of
// the listed rows of up to three arrays of one head segment.
__device__ void move_rows16(uint4* x, uint4* y, uint4* z, int units, const int32_t* trip, int count) {
  for (int idx = threadIdx.x; idx < count * units; idx += kCmpThreads) {
    const int j = idx / units, u = idx - j * units;
    const int64_t src = (int64_t)trip[3 * j] * units + u, dst = (int64_t)trip[3 * j + 1] * units + u;
    const uint4 xv = x[src];
    const uint4 yv = y ? y[src] : uint4{};
    const uint4 zv = z ? z[src] : uint4{};
    x[dst] = xv;
    if (y) y[dst] = yv;
    if (z) z[dst] = zv;
  }
}

__global__ void __launch_bounds__(kCmpThreads) compact_kernel(const CompactArgs a) {
  const int h = blockIdx.x, b = blockIdx.y;
  if (a.moves) {
    // ---- slot-map compaction: planned moves only
    const int32_t* trip = a.moves + b * a.mv_bs + a.row_stride;  // after the [capacity] planning scratch
    const int count = a.mcount[b * a.mc_bs];
    if (h < a.heads) {
      const int units = a.row_bytes / 16;
      uint4* kx = reinterpret_cast<uint4*>(a.k + b * a.kv_bs + h * a.kv_hs);
      uint4* vx = reinterpret_cast<uint4*>(a.v + b * a.kv_bs + h * a.kv_hs);
      uint4* rx = a.k_raw ? reinterpret_cast<uint4*>(a.k_raw + b * a.kv_bs + h * a.kv_hs) : nullptr;
      move_rows16(kx, vx, rx, units, trip, count);
      return;
    }
    const int first = a.first_moved ? min(a.first_moved[b], a.m) : 0;
    if (first < a.m) {  // token metadata: logical order (cache.py:154-156)
      if (a.pos) gather_elems<int64_t>(a.pos + b * a.m_bs, a, b, first, a.m);
      if (a.modality) gather_elems<int8_t>(a.modality + b * a.m_bs, a, b, first, a.m);
      if (a.round_id) gather_elems<int32_t>(a.round_id + b * a.m_bs, a, b, first, a.m);
    }
    // accumulators (engine.py:335) and window-row values sit at physical rows:
    // a row keeps the mover's value when the mover lies inside its new length
    if (a.acc) {
      float* acc = a.acc + b * a.acc_bs;
      for (int j = threadIdx.x; j < count; j += kCmpThreads) acc[trip[3 * j + 1]] = acc[trip[3 * j]];
    }
    if (a.rows) {
      for (int idx = threadIdx.x; idx < a.W * count; idx += kCmpThreads) {
        const int w = idx / count, j = idx - w * count;
        if (trip[3 * j + 2] < a.newlen[b * a.w_bs + w]) {
          float* row = a.rows + b * a.r_bs + (int64_t)w * a.row_stride;
          row[trip[3 * j + 1]] = row[trip[3 * j]];
        }
      }
      __syncthreads();
      for (int w = threadIdx.x; w < a.W; w += blockDim.x) a.wlen[b * a.w_bs + w] = a.newlen[b * a.w_bs + w];
    }
    if (threadIdx.x == 0 && a.len) a.len[b * a.len_bs] = a.m;
    return;
  }
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

namespace skv {

// p[i] = i % period for i < count (identity slot maps).
__global__ void iota_kernel(int32_t* p, int64_t count, int period) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)(i % period);
}

cudaError_t launch_iota(int32_t* p, int64_t count, int period, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(4096, (count + 255) / 256);
  if (blocks <= 0) return cudaSuccess;
  iota_kernel<<<blocks, 256, 0, st>>>(p, count, period);
  return cudaGetLastError();
}

}  // namespace skv
