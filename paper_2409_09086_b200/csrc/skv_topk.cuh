// Block-wide scan and radix top-k shared by the selection kernel (select.cu)
// and the trace replay (replay.cu): top_k_indices (policies.py:165-181) as a
// 4-pass 8-bit radix select on the order-preserving uint32 image of the
// float (-0.0 == +0.0), ties resolved toward the larger index, ascending
// output by a block-wide scan.
#pragma once

#include <stdint.h>

#include "skv_common.cuh"

namespace skv {

struct ScanSmem {
  int warp_sums[32];
  int total;
};

// Block-wide exclusive scan of one int per thread.  All threads must call.
__device__ inline int block_excl_scan(int v, ScanSmem& sm, int& total) {
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
__device__ inline void topk_block(const float* scores, int cols, int k, int32_t* out32, int64_t* out64, TopkSmem& sm) {
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


}  // namespace skv
