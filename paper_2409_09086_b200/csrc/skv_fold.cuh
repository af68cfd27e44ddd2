// Window-row fold shared by the decode and prefill paths: materialises
// head-aggregated probability rows from recorded logits and per-head
// (max, sum) -- aggregate_heads (reference policies.py:259-263) applied to
// Session._attend's probabilities (engine.py:240-244).
#pragma once

#include "skv_common.cuh"
#include "skv_internal.h"

namespace skv {

// row[j] = agg_h p[h][j] with p = expf(x - M_h) / L_h, for j in [c0, c1).
// Head order is sequential h = 0..Hq-1 in float32 (aggregate_heads, policies.py:262).
__device__ __forceinline__ void fold_columns(const FoldArgs& f, int s, int c0, int c1, int Hq, int tid, int nthreads,
                             const float* stt = nullptr) {
  const float* lg = f.logits + s * f.l_ss;
  if (!stt) stt = f.stats + s * f.st_ss;
  float* row = f.rows ? f.rows + s * f.r_ss : nullptr;
  for (int j = c0 + tid; j < c1; j += nthreads) {
    float acc = f.mode == 1 ? -INFINITY : 0.f;
#pragma unroll 16
    for (int h = 0; h < Hq; ++h) {
      const float M = stt[2 * h];
      const float L = stt[2 * h + 1];
      const float p = __fdiv_rn(expf(__fsub_rn(__ldcs(lg + h * f.l_hs + j), M)), L);
      if (f.mode == 2) {
        f.probs[s * f.p_ss + h * f.p_hs + j] = p;
      } else if (f.mode == 1) {
        acc = fmaxf(acc, p);
      } else {
        acc = __fadd_rn(acc, p);
      }
    }
    if (f.mode == 0) row[j] = __fdiv_rn(acc, (float)(f.agg_div ? f.agg_div : Hq));
    else if (f.mode == 1) row[j] = acc;
  }
}

__device__ __forceinline__ void fold_piece(const FoldArgs& f, int s, int piece, int pieces, int Hq, int tid,
                                           int nthreads) {
  if (f.n <= 0) return;
  const int w = (f.n + pieces - 1) / pieces;
  const int c0 = piece * w;
  const int c1 = min(c0 + w, f.n);
  if (c0 < c1) fold_columns(f, s, c0, c1, Hq, tid, nthreads);
  if (piece == 0 && tid == 0 && f.wlen) f.wlen[s * f.w_ss] = f.n;
}

}  // namespace skv
