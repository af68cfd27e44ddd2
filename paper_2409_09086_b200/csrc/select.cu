// K2: Algorithm-1 selection on device, one 1024-thread CTA per window.
//
//   window_mean_scores (reference policies.py:130-147): column sums over the
//     window rows oldest -> newest in float32 (__fadd_rn, a column absent from a
//     shorter row contributes nothing), then IEEE division by f32(rows held);
//   bias_vector (policies.py:150-162): d = f32(b)/f32(cols),
//     bias[c] = (-d) * f32(cols-1-c) with __fmul_rn (no FMA contraction), added
//     with a separate __fadd_rn exactly like `scores + bias` (policies.py:197);
//   top_k_indices (policies.py:165-181): 4-pass 8-bit radix select on the
//     order-preserving uint32 image of the float (-0.0 == +0.0), ties resolved
//     toward the larger index, ascending output by a block-wide scan;
//   inf_mllm_decide (policies.py:184-201): keep-all when n <= r+l, otherwise
//     kept = relevant ++ [n-l, n).
// It also emits what compaction needs: the first moved index (kept[i] != i),
// the window row lengths after AttentionWindow.remap (policies.py:117-124)
// and, for engines with a slot map, the plan of the compaction (plan_moves).
#include <algorithm>

#include "skv_common.cuh"
#include "skv_internal.h"
#include "skv_topk.cuh"

namespace skv {

constexpr int kSelThreads = 1024;

// Slot-map compaction plan for one (stream, layer).  Logical slot c lives in
// physical row perm[c]; rows [0, n) hold exactly the live tokens.  After the
// decision keeps `kept` (ascending, m entries) the kept tokens must occupy rows
// [0, m) again.  Those already there stay put; each kept token whose row is
// >= m moves into a row of [0, m) freed by an evicted token (the i-th such
// mover, in logical order, to the i-th free row, ascending).  Sources (>= m)
// and destinations (< m) are disjoint, so the moves are hazard-free and
// independent.  The logical order (cache.py:151-156: stable, ascending) is
// carried by the new perm; token metadata and window lengths stay logical.
// At most n - m rows move -- the tokens appended since the last eviction that
// survive it -- instead of every row after the first evicted one.
__device__ void plan_moves(const SelectArgs& a, int b, int n, int m, const int32_t* k32, const int64_t* k64,
                           unsigned* used, ScanSmem& scan) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int32_t* perm = a.perm + b * a.pm_bs;
  int32_t* pk = a.moves + b * a.mv_bs;     // [m] physical row of kept[i]
  int32_t* trip = pk + a.row_stride;       // [count][3] (src, dst, logical index); region = 4 x capacity
  const int words = (m + 31) / 32;
  for (int w = tid; w < words; w += nt) used[w] = 0;
  __syncthreads();
  for (int i = tid; i < m; i += nt) {
    const int c = k32 ? k32[i] : (int)k64[i];
    const int p = perm[c];
    pk[i] = p;
    if (p < m) atomicOr(&used[p >> 5], 1u << (p & 31));
  }
  __syncthreads();
  // free rows of [0, m), ascending: contiguous word ranges per thread
  const int wseg = (words + nt - 1) / nt;
  const int w0 = min(tid * wseg, words), w1 = min(w0 + wseg, words);
  auto free_bits = [&](int w) {
    const unsigned valid = (w == words - 1 && (m & 31)) ? ((1u << (m & 31)) - 1u) : 0xffffffffu;
    return ~used[w] & valid;
  };
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(free_bits(w));
  int holes_total;
  int rank = block_excl_scan(cnt, scan, holes_total);
  for (int w = w0; w < w1; ++w) {
    unsigned f = free_bits(w);
    while (f) {
      const int bit = __ffs(f) - 1;
      f &= f - 1;
      trip[3 * rank + 1] = 32 * w + bit;
      ++rank;
    }
  }
  __syncthreads();
  // movers in logical order take the free rows in ascending order
  const int seg = (m + nt - 1) / nt;
  const int i0 = min(tid * seg, m), i1 = min(i0 + seg, m);
  int mv = 0;
  for (int i = i0; i < i1; ++i) mv += pk[i] >= m;
  int movers_total;
  int j = block_excl_scan(mv, scan, movers_total);
  for (int i = i0; i < i1; ++i) {
    const int p = pk[i];
    if (p >= m) {
      const int dst = trip[3 * j + 1];
      trip[3 * j] = p;
      trip[3 * j + 2] = i;
      perm[i] = dst;
      ++j;
    } else {
      perm[i] = p;
    }
  }
  for (int i = m + tid; i < n; i += nt) perm[i] = i;  // appends land at their logical slot
  if (tid == 0) a.mcount[b * a.mc_bs] = movers_total;  // == holes_total
  __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectArgs a) {
  __shared__ TopkSmem sm;
  __shared__ int slot_of[1024];
  __shared__ int len_of[1024];
  __shared__ unsigned used_rows[kMaxMapRows / 32];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, l = a.l, r = a.r;
  int32_t* k32 = a.kept32 ? a.kept32 + b * a.k_bs : nullptr;
  int64_t* k64 = a.kept64 ? a.kept64 + b * a.k_bs : nullptr;

  for (int k = tid; k < a.count; k += blockDim.x) {
    const int slot = ((a.ring_head - a.count + k) % a.W + a.W) % a.W;
    slot_of[k] = slot;
    len_of[k] = a.wlen[b * a.w_bs + slot];
  }
  __syncthreads();

  const bool keep_all = !a.scores_only && n <= r + l;
  if (!keep_all) {
    const int cols = n - l;
    float* sc = a.scores + b * a.s_bs;
    if (a.policy == 1 || a.policy == 2) {
      // sliding_window_decide / sink_recent_decide (policies.py:204-231):
      // kept = [0, s) ++ [n - (B - s), n), s = 0 for the sliding window
      const int B = r + l, s0 = a.policy == 2 ? a.sink : 0;
      for (int i = tid; i < B; i += blockDim.x) {
        const int v = i < s0 ? i : n - B + i;
        if (k32) k32[i] = v;
        if (k64) k64[i] = v;
      }
      if (tid == 0 && a.first_moved) a.first_moved[b] = s0;
    } else {
      if (a.policy == 3) {
        // heavy_hitter_decide (policies.py:246-256): top-r of the accumulated
        // mass acc[:n-l], no averaging, no bias
        const float* acc = a.acc + b * a.acc_bs;
        const int32_t* pm = a.perm ? a.perm + b * a.pm_bs : nullptr;
        for (int c = tid; c < cols; c += blockDim.x) sc[c] = acc[pm ? pm[c] : c];
      } else {
        // ---- window-mean scores (+ bias), policies.py:130-162
        const float d = __fdiv_rn(a.bias, (float)cols);
        const float negd = -d;
        const float inv_m = (float)a.count;
        const float* rows = a.rows + b * a.r_bs;
        const float* sin = a.scores_in ? a.scores_in + b * a.si_bs : nullptr;
        const int32_t* pm = a.perm ? a.perm + b * a.pm_bs : nullptr;
        for (int c = tid; c < cols; c += blockDim.x) {
          float v;
          if (sin) {
            v = sin[c];
          } else {
            // row values sit at the column's physical row (slot map)
            const int pc = pm ? pm[c] : c;
            float acc = 0.f;
            for (int k = 0; k < a.count; ++k)
              if (c < len_of[k]) acc = __fadd_rn(acc, rows[(int64_t)slot_of[k] * a.row_stride + pc]);
            v = __fdiv_rn(acc, inv_m);
          }
          if (a.apply_bias) v = __fadd_rn(v, __fmul_rn(negd, (float)(cols - 1 - c)));
          sc[c] = v;
        }
      }
      __syncthreads();
      if (a.scores_only) return;

      // ---- top-r + recent merge
      int first = 0;
      if (r > 0) {
        topk_block(sc, cols, r, k32, k64, sm);
        first = sm.first_unsel;
      }
      for (int i = tid; i < l; i += blockDim.x) {
        if (k32) k32[r + i] = n - l + i;
        if (k64) k64[r + i] = n - l + i;
      }
      if (tid == 0 && a.first_moved) a.first_moved[b] = first;
    }
    __syncthreads();
    if (a.moves) plan_moves(a, b, n, r + l, k32, k64, used_rows, sm.scan);
    // ---- window lengths after remap: #{i : kept[i] < len}
    if (a.newlen) {
      for (int k = tid; k < a.count; k += blockDim.x) {
        const int len = len_of[k];
        int lo = 0, hi = r + l;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const int64_t kv = k32 ? (int64_t)k32[mid] : k64[mid];
          if (kv < len) lo = mid + 1;
          else hi = mid;
        }
        a.newlen[b * a.w_bs + slot_of[k]] = lo;
      }
    }
  } else {
    for (int i = tid; i < n; i += blockDim.x) {
      if (k32) k32[i] = i;
      if (k64) k64[i] = i;
    }
    for (int i = n + tid; i < a.pad; i += blockDim.x) {
      if (k32) k32[i] = -1;
      if (k64) k64[i] = -1;
    }
    if (tid == 0 && a.first_moved) a.first_moved[b] = n;
    if (tid == 0 && a.moves) a.mcount[b * a.mc_bs] = 0;  // keep-all: nothing moves
    if (a.newlen)
      for (int k = tid; k < a.count; k += blockDim.x) a.newlen[b * a.w_bs + slot_of[k]] = len_of[k];
  }
}

__global__ void __launch_bounds__(kSelThreads) topk_kernel(const float* scores, int n, int k, int64_t* out) {
  __shared__ TopkSmem sm;
  if (k >= n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = i;
    return;
  }
  if (k <= 0) return;
  topk_block(scores, n, k, nullptr, out, sm);
}

cudaError_t launch_select(int batches, const SelectArgs& a, cudaStream_t st) {
  if (a.W > 1024) return cudaErrorInvalidValue;
  select_kernel<<<batches, kSelThreads, 0, st>>>(a);
  return cudaGetLastError();
}

__global__ void hh_accumulate_kernel(const float* __restrict__ acc, int na, const float* __restrict__ row, int n,
                                     float* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    out[j] = j < na ? __fadd_rn(row[j], acc[j]) : row[j];
}

cudaError_t launch_hh_accumulate(const float* acc, int na, const float* row, int n, float* out, cudaStream_t st) {
  const int blocks = std::min(1024, (n + 255) / 256);
  hh_accumulate_kernel<<<blocks, 256, 0, st>>>(acc, na, row, n, out);
  return cudaGetLastError();
}

// replay_trace's projection (replay.py:139-142): out[i] = f32(f64(probs[live[i]]) / sum),
// sum = the f64 total of the projected values (one block).
__global__ void __launch_bounds__(1024) project_row_kernel(const float* __restrict__ probs, int n,
                                                           const int64_t* __restrict__ live, int m,
                                                           float* __restrict__ out) {
  __shared__ double part[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int64_t c = live[i];
    acc += (c >= 0 && c < n) ? (double)probs[c] : 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) part[0] = v;
  }
  __syncthreads();
  const double total = part[0];
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int64_t c = live[i];
    const double p = (c >= 0 && c < n) ? (double)probs[c] : 0.0;
    out[i] = total > 0.0 ? (float)(p / total) : (float)p;
  }
}

// retained_mass's per-row sums (metrics.py:46-62): out[r] = f64 sum of
// rows[r][kept[i]] over kept[i] < lens[r].  One block per row.
__global__ void __launch_bounds__(256) masked_row_sums_kernel(const float* __restrict__ rows, int row_stride,
                                                              const int32_t* __restrict__ lens,
                                                              const int64_t* __restrict__ kept, int k,
                                                              double* __restrict__ out) {
  __shared__ double part[8];
  const int r = blockIdx.x;
  const int len = lens[r];
  const float* row = rows + (int64_t)r * row_stride;
  double acc = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int64_t c = kept[i];
    if (c >= 0 && c < len) acc += (double)row[c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += part[w];
    out[r] = v;
  }
}

cudaError_t launch_project_row(const float* probs, int n, const int64_t* live, int m, float* out, cudaStream_t st) {
  project_row_kernel<<<1, 1024, 0, st>>>(probs, n, live, m, out);
  return cudaGetLastError();
}

cudaError_t launch_masked_row_sums(const float* rows, int row_stride, const int32_t* lens, int m, const int64_t* kept,
                                   int k, double* out, cudaStream_t st) {
  masked_row_sums_kernel<<<m, 256, 0, st>>>(rows, row_stride, lens, kept, k, out);
  return cudaGetLastError();
}

cudaError_t launch_topk(const float* scores, int n, int k, int64_t* out, cudaStream_t st) {
  topk_kernel<<<1, kSelThreads, 0, st>>>(scores, n, k, out);
  return cudaGetLastError();
}

}  // namespace skv
