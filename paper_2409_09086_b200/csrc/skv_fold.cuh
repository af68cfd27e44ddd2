// Window-row fold shared by the decode and prefill paths: materialises
// head-aggregated probability rows from recorded logits and per-head
// (max, sum) -- aggregate_heads (reference policies.py:259-263) applied to
// Session._attend's probabilities (engine.py:240-244).
#pragma once

#include "skv_common.cuh"
#include "skv_internal.h"

namespace skv {

// p = expf(x - M) * (1/L): the row sum's reciprocal (__frcp_rn, IEEE) is
// formed once per (row, head) and staged next to M, so the per-column cost is
// one expf and one multiply (within 1.5 ulp of expf(x - M) / L).
__device__ __forceinline__ float fold_prob(float x, float M, float rL) { return __fmul_rn(expf(__fsub_rn(x, M)), rL); }

// row[j] = agg_h p[h][j] with p = fold_prob(x, M_h, 1/L_h), for j in [c0, c1).
// Head order is sequential h = 0..Hq-1 in float32 (aggregate_heads, policies.py:262).
// stt: staged (M_h, 1/L_h) pairs, or null to read (M_h, L_h) from f.stats.
// The logits of HB heads are loaded before any is used: the per-head stores of
// mode 2 may alias the logits as far as the compiler knows, so without the
// explicit batch every load waited for the previous head's store (a 64-column
// piece of 32 heads took ~30 us in a decode kernel's fold warp).
// Few heads (a KV-head group as a stream): CB columns per thread per pass, all
// their CB x Hq logit loads in flight together (same per-column arithmetic).
template <int CB, int HMAX>
__device__ __forceinline__ void fold_columns_few(const FoldArgs& f, int s, const float* lg, const float* stt,
                                                 bool staged, float* row, int c0, int c1, int Hq, int tid,
                                                 int nthreads) {
  for (int jb = c0 + tid; jb < c1; jb += nthreads * CB) {
    float x[CB][HMAX];
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int j = jb + c * nthreads;
#pragma unroll
      for (int h = 0; h < HMAX; ++h) x[c][h] = (h < Hq && j < c1) ? __ldcs(lg + (int64_t)h * f.l_hs + j) : 0.f;
    }
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int j = jb + c * nthreads;
      if (j >= c1) continue;
      float acc = f.mode == 1 ? -INFINITY : 0.f;
#pragma unroll
      for (int h = 0; h < HMAX; ++h) {
        if (h < Hq) {
          const float M = stt[2 * h];
          const float rL = staged ? stt[2 * h + 1] : __frcp_rn(stt[2 * h + 1]);
          const float p = fold_prob(x[c][h], M, rL);
          if (f.mode == 2) {
            f.probs[s * f.p_ss + h * f.p_hs + j] = p;
          } else if (f.mode == 1) {
            acc = fmaxf(acc, p);
          } else {
            acc = __fadd_rn(acc, p);
          }
        }
      }
      if (f.mode != 2) {
        const float v = f.mode == 0 ? __fdiv_rn(acc, (float)(f.agg_div ? f.agg_div : Hq)) : acc;
        row[j] = (f.accum && j < f.n - 1) ? __fadd_rn(row[j], v) : v;
      }
    }
  }
}

// columns one pass of fold_columns covers per thread (pieces of a fold warp)
__host__ __device__ __forceinline__ int fold_cols_per_pass(int Hq) { return Hq <= 4 ? 4 : Hq <= 8 ? 2 : 1; }

template <int HB = 16>
__device__ __forceinline__ void fold_columns(const FoldArgs& f, int s, int c0, int c1, int Hq, int tid, int nthreads,
                                             const float* stt = nullptr) {
  const bool staged = stt != nullptr;
  const float* lg = f.logits + s * f.l_ss;
  if (!stt) stt = f.stats + s * f.st_ss;
  float* row = f.rows ? f.rows + s * f.r_ss : nullptr;
  if (Hq <= 4) return fold_columns_few<4, 4>(f, s, lg, stt, staged, row, c0, c1, Hq, tid, nthreads);
  if (Hq <= 8) return fold_columns_few<2, 8>(f, s, lg, stt, staged, row, c0, c1, Hq, tid, nthreads);
  for (int j = c0 + tid; j < c1; j += nthreads) {
    float acc = f.mode == 1 ? -INFINITY : 0.f;
    for (int h0 = 0; h0 < Hq; h0 += HB) {
      float x[HB];
#pragma unroll
      for (int b = 0; b < HB; ++b) x[b] = h0 + b < Hq ? __ldcs(lg + (int64_t)(h0 + b) * f.l_hs + j) : 0.f;
#pragma unroll
      for (int b = 0; b < HB; ++b) {
        const int h = h0 + b;
        if (h < Hq) {
          const float M = stt[2 * h];
          const float rL = staged ? stt[2 * h + 1] : __frcp_rn(stt[2 * h + 1]);
          const float p = fold_prob(x[b], M, rL);
          if (f.mode == 2) {
            f.probs[s * f.p_ss + h * f.p_hs + j] = p;
          } else if (f.mode == 1) {
            acc = fmaxf(acc, p);
          } else {
            acc = __fadd_rn(acc, p);
          }
        }
      }
    }
    if (f.mode != 2) {
      const float v = f.mode == 0 ? __fdiv_rn(acc, (float)(f.agg_div ? f.agg_div : Hq)) : acc;
      row[j] = (f.accum && j < f.n - 1) ? __fadd_rn(row[j], v) : v;
    }
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

// Throughput version for stand-alone fold launches: each thread owns four
// consecutive columns (16-byte logit loads, four independent head-sum
// chains), the per-head (M, 1/L) are staged in shared memory, and the heads
// are walked in batches of eight loads in flight.  Same arithmetic per column
// as fold_columns (sequential head order, fold_prob) -- bit-identical.
// MODE 0: mean over heads (divisor agg), MODE 1: max over heads.
template <int MODE, int HB = 8>
__device__ __forceinline__ void fold_vec4(const float* __restrict__ lg, int64_t l_hs, const float* __restrict__ stt,
                                          float* __restrict__ row, int j0, int n, int Hq, float agg, int accum = 0) {
  float acc[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) acc[e] = MODE == 1 ? -INFINITY : 0.f;
  if (j0 + 3 < n) {
    for (int h0 = 0; h0 < Hq; h0 += HB) {
      float4 x[HB];
#pragma unroll
      for (int b = 0; b < HB; ++b)
        if (h0 + b < Hq) x[b] = __ldcs(reinterpret_cast<const float4*>(lg + (int64_t)(h0 + b) * l_hs + j0));
#pragma unroll
      for (int b = 0; b < HB; ++b) {
        if (h0 + b < Hq) {
          const float M = stt[2 * (h0 + b)], rL = stt[2 * (h0 + b) + 1];
          const float v[4] = {x[b].x, x[b].y, x[b].z, x[b].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float p = fold_prob(v[e], M, rL);
            acc[e] = MODE == 1 ? fmaxf(acc[e], p) : __fadd_rn(acc[e], p);
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float v = MODE == 1 ? acc[e] : __fdiv_rn(acc[e], agg);
      row[j0 + e] = (accum && j0 + e < n - 1) ? __fadd_rn(row[j0 + e], v) : v;
    }
  } else {
    for (int e = 0; e < 4 && j0 + e < n; ++e) {
      float a = MODE == 1 ? -INFINITY : 0.f;
      for (int h = 0; h < Hq; ++h) {
        const float p = fold_prob(__ldcs(lg + (int64_t)h * l_hs + j0 + e), stt[2 * h], stt[2 * h + 1]);
        a = MODE == 1 ? fmaxf(a, p) : __fadd_rn(a, p);
      }
      const float v = MODE == 1 ? a : __fdiv_rn(a, agg);
      row[j0 + e] = (accum && j0 + e < n - 1) ? __fadd_rn(row[j0 + e], v) : v;
    }
  }
}

}  // namespace skv
