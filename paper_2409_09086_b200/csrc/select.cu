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
// It also emits what compaction needs: the first moved index (kept[i] != i) and
// the window row lengths after AttentionWindow.remap (policies.py:117-124).
#include <algorithm>

#include "skv_common.cuh"
#include "skv_internal.h"

namespace skv {

constexpr int kSelThreads = 1024;

struct ScanSmem {
  int warp_sums[32];
  int total;
};

// Block-wide exclusive scan of one int per thread.  All threads must call.
__device__ int block_excl_scan(int v, ScanSmem& sm, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? sm.warp_sums[lane] : 0;
    int incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < nw) sm.warp_sums[lane] = incl - w;
    if (lane == 31) sm.total = incl;
  }
  __syncthreads();
  const int excl = sm.warp_sums[warp] + x - v;
  total = sm.total;
  __syncthreads();
  return excl;
}

struct TopkSmem {
  unsigned hist[256];
  unsigned prefix;
  int krem;
  int first_unsel;
  ScanSmem scan;
};

// Select the k largest of scores[0, cols) (ties -> larger index) and write their
// indices ascending to out32/out64[0, k).  Requires 0 < k < cols.  Returns
// (through smem) the smallest unselected index.
__device__ void topk_block(const float* scores, int cols, int k, int32_t* out32, int64_t* out64, TopkSmem& sm) {
  const int tid = threadIdx.x, nt = blockDim.x;
  unsigned prefix = 0, mask = 0;
  int krem = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += nt) sm.hist[i] = 0;
    __syncthreads();
    for (int c = tid; c < cols; c += nt) {
      const unsigned u = orderable(scores[c]);
      if ((u & mask) == prefix) atomicAdd(&sm.hist[(u >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane L owns bins [8L, 8L+8); find the digit holding the krem-th largest
      unsigned local[8];
      unsigned lsum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        local[i] = sm.hist[8 * tid + i];
        lsum += local[i];
      }
      unsigned suffix = lsum;  // inclusive suffix sum over lanes >= tid
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_down_sync(0xffffffffu, suffix, o);
        if (tid + o < 32) suffix += y;
      }
      const unsigned above = suffix - lsum;  // count in lanes > tid
      if (above < (unsigned)krem && suffix >= (unsigned)krem) {
        unsigned acc = above;
        int digit = 8 * tid;
        for (int i = 7; i >= 0; --i) {
          if (acc + local[i] >= (unsigned)krem) {
            digit = 8 * tid + i;
            break;
          }
          acc += local[i];
        }
        sm.prefix = prefix | ((unsigned)digit << shift);
        sm.krem = krem - (int)acc;
      }
    }
    __syncthreads();
    prefix = sm.prefix;
    krem = sm.krem;
    mask |= 255u << shift;
    __syncthreads();
  }
  const unsigned thr = prefix;  // key of the k-th largest; take krem of its ties

  // contiguous segment per thread so scans preserve index order
  const int seg = (cols + nt - 1) / nt;
  const int c0 = min(tid * seg, cols), c1 = min(c0 + seg, cols);
  int eq = 0;
  for (int c = c0; c < c1; ++c) eq += orderable(scores[c]) == thr;
  int eq_total;
  const int eq_before = block_excl_scan(eq, sm.scan, eq_total);
  if (tid == 0) sm.first_unsel = cols;
  __syncthreads();
  int nsel = 0, r = eq_before, first_un = cols;
  for (int c = c0; c < c1; ++c) {
    const unsigned u = orderable(scores[c]);
    bool sel = u > thr;
    if (u == thr) {
      sel = (eq_total - 1 - r) < krem;  // newest ties win
      ++r;
    }
    nsel += sel;
    if (!sel && first_un == cols) first_un = c;
  }
  if (first_un < cols) atomicMin(&sm.first_unsel, first_un);
  int sel_total;
  int pos = block_excl_scan(nsel, sm.scan, sel_total);
  r = eq_before;
  for (int c = c0; c < c1; ++c) {
    const unsigned u = orderable(scores[c]);
    bool sel = u > thr;
    if (u == thr) {
      sel = (eq_total - 1 - r) < krem;
      ++r;
    }
    if (sel) {
      if (out32) out32[pos] = c;
      if (out64) out64[pos] = c;
      ++pos;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectArgs a) {
  __shared__ TopkSmem sm;
  __shared__ int slot_of[1024];
  __shared__ int len_of[1024];
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
        for (int c = tid; c < cols; c += blockDim.x) sc[c] = acc[c];
      } else {
        // ---- window-mean scores (+ bias), policies.py:130-162
        const float d = __fdiv_rn(a.bias, (float)cols);
        const float negd = -d;
        const float inv_m = (float)a.count;
        const float* rows = a.rows + b * a.r_bs;
        const float* sin = a.scores_in ? a.scores_in + b * a.si_bs : nullptr;
        for (int c = tid; c < cols; c += blockDim.x) {
          float v;
          if (sin) {
            v = sin[c];
          } else {
            float acc = 0.f;
            for (int k = 0; k < a.count; ++k)
              if (c < len_of[k]) acc = __fadd_rn(acc, rows[(int64_t)slot_of[k] * a.row_stride + c]);
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
