// K1: split-KV flash-decode for one layer of S independent streams (sm_100a).
//
// Replaces, per (stream, layer) and decode step, the body of
// Session.decode_step (reference engine.py:264-273):
//   KvCache.append (cache.py:112-134)   -> the new k/v row is bulk-copied from the
//                                          input straight into the last tile and
//                                          written to the cache slot n_old;
//   Session._attend (engine.py:235-246) -> split-KV online softmax, warp-shuffle
//                                          reductions, P.V in fp32;
//   aggregate_heads + AttentionWindow.push (policies.py:259-263, 107-115)
//                                       -> each CTA records its tile logits; the
//                                          head-aggregated row is materialised
//                                          ("folded") by the NEXT launch of the
//                                          layer, spread over all its CTAs, once
//                                          the global per-head (max, sum) exist.
//
// Grid (splits, Hkv, S); 4 consumer warps + 1 producer warp.  The producer
// streams 32-token K and V tiles (contiguous rows of one head) into a 4-stage
// shared-memory ring with 1-D bulk async copies (TMA engine) completing on
// mbarriers.  The last CTA of each (stream, kv-head) merges the split partials
// (fixed split order => deterministic) and publishes per-head (M, L).
#include "skv_common.cuh"
#include "skv_internal.h"

namespace skv {

template <typename T, int D>
struct Geo {
  static constexpr int ELT = sizeof(T);
  static constexpr int RB = D * ELT;      // bytes per cached row
  static constexpr int LPR = RB / 16;     // lanes per row (16 B each)
  static constexpr int EPL = 16 / ELT;    // elements per lane
  static constexpr int RPW = 32 / LPR;    // rows per warp load
  static constexpr int TT = 32;           // tokens per tile
  static constexpr int NW = 4;            // consumer warps
  static constexpr int RPWARP = TT / NW;  // rows per warp per tile
  static constexpr int ITERS = RPWARP / RPW;
  static constexpr int TILE = TT * RB;    // bytes per K (or V) tile
  static constexpr int STAGES = TILE > 8192 ? 3 : 4;
  static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "row geometry");
  static_assert(ITERS >= 1, "tile geometry");
};

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

__device__ __forceinline__ float rescale(float m, float M) {
  return m == -INFINITY ? 0.f : exp2f((m - M) * kLog2e);
}

// row[j] = agg_h p[h][j] with p = expf(x - M_h) / L_h, for j in [c0, c1).
// Head order is sequential h = 0..Hq-1 in float32 (aggregate_heads, policies.py:262).
__device__ void fold_columns(const FoldArgs& f, int s, int c0, int c1, int Hq, int tid, int nthreads) {
  const float* lg = f.logits + s * f.l_ss;
  const float* stt = f.stats + s * f.st_ss;
  float* row = f.rows ? f.rows + s * f.r_ss : nullptr;
  for (int j = c0 + tid; j < c1; j += nthreads) {
    float acc = f.mode == 1 ? -INFINITY : 0.f;
#pragma unroll 8
    for (int h = 0; h < Hq; ++h) {
      const float M = __ldg(stt + 2 * h);
      const float L = __ldg(stt + 2 * h + 1);
      const float p = __fdiv_rn(expf(__fsub_rn(__ldcs(lg + h * f.l_hs + j), M)), L);
      if (f.mode == 2) {
        f.probs[s * f.p_ss + h * f.p_hs + j] = p;
      } else if (f.mode == 1) {
        acc = fmaxf(acc, p);
      } else {
        acc = __fadd_rn(acc, p);
      }
    }
    if (f.mode == 0) row[j] = __fdiv_rn(acc, (float)Hq);
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

template <typename T, int D, int G>
__global__ void __launch_bounds__(160) decode_kernel(const AttnArgs a) {
  using Gm = Geo<T, D>;
  constexpr int TT = Gm::TT, RB = Gm::RB, LPR = Gm::LPR, EPL = Gm::EPL, RPW = Gm::RPW;
  constexpr int NW = Gm::NW, ITERS = Gm::ITERS, STAGES = Gm::STAGES, TILE = Gm::TILE;

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* tiles = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * 2 * TILE);
  uint64_t* empty = full + STAGES;
  float* wm = reinterpret_cast<float*>(empty + STAGES);  // [NW][G]
  float* wl = wm + NW * G;                               // [NW][G]
  float* wo = wl + NW * G;                               // [NW][G][D]
  float* fin = wo + NW * G * D;                          // [G][2] merged (M, L)
  int* flag = reinterpret_cast<int*>(fin + 2 * G);

  const int split = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_old + a.append;
  const int t0 = split * a.chunk;
  const int t1 = min(t0 + a.chunk, n);
  const int ntiles = t1 > t0 ? (t1 - t0 + TT - 1) / TT : 0;

  const T* kbase = static_cast<const T*>(a.kc) + s * a.c_ss + (int64_t)g * a.c_hs;
  const T* vbase = static_cast<const T*>(a.vc) + s * a.c_ss + (int64_t)g * a.c_hs;
  const T* knew = static_cast<const T*>(a.kin) + s * a.in_ss + (int64_t)g * D;
  const T* vnew = static_cast<const T*>(a.vin) + s * a.in_ss + (int64_t)g * D;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int it = 0; it < ntiles; ++it) {
        const int st = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        const int ts = t0 + it * TT;
        const int rows = min(TT, t1 - ts);
        const int rc = max(0, min(rows, a.n_old - ts));
        unsigned char* ks = tiles + (2 * st) * TILE;
        unsigned char* vs = ks + TILE;
        mbar_arrive_expect_tx(&full[st], 2u * rows * RB);
        if (rc > 0) {
          bulk_g2s(ks, kbase + (int64_t)ts * D, rc * RB, &full[st]);
          bulk_g2s(vs, vbase + (int64_t)ts * D, rc * RB, &full[st]);
        }
        if (rc < rows) {  // the appended token: straight from the step input
          bulk_g2s(ks + rc * RB, knew, RB, &full[st]);
          bulk_g2s(vs + rc * RB, vnew, RB, &full[st]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int rsub = lane / LPR, c16 = lane % LPR;
  float qf[G][EPL];
#pragma unroll
  for (int h = 0; h < G; ++h)
    Vec16<T>::load(qf[h], static_cast<const T*>(a.q) + s * a.q_ss + (int64_t)(g * G + h) * D + c16 * EPL);

  float m_run[G], l_run[G], o[G][EPL];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    m_run[h] = -INFINITY;
    l_run[h] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) o[h][e] = 0.f;
  }
  float* lg = a.logits ? a.logits + s * a.l_ss + (int64_t)(g * G) * a.l_hs : nullptr;

  for (int it = 0; it < ntiles; ++it) {
    const int st = it % STAGES;
    const uint32_t ph = (it / STAGES) & 1;
    const int ts = t0 + it * TT;
    const int rows = min(TT, t1 - ts);
    const unsigned char* ks = tiles + (2 * st) * TILE;
    const unsigned char* vs = ks + TILE;
    mbar_wait(&full[st], ph);

    float sc[ITERS][G];
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int row = warp * Gm::RPWARP + i * RPW + rsub;
      float kf[EPL];
      Vec16<T>::load(kf, ks + row * RB + c16 * 16);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) d = fmaf(qf[h][e], kf[e], d);
#pragma unroll
        for (int off = LPR / 2; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        sc[i][h] = row < rows ? d * a.scale : -INFINITY;
      }
    }
    if (lg && c16 == 0) {
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        const int row = warp * Gm::RPWARP + i * RPW + rsub;
        if (row < rows) {
#pragma unroll
          for (int h = 0; h < G; ++h) lg[h * a.l_hs + ts + row] = sc[i][h];
        }
      }
    }
    float p[ITERS][G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float mt = -INFINITY;
#pragma unroll
      for (int i = 0; i < ITERS; ++i) mt = fmaxf(mt, sc[i][h]);
#pragma unroll
      for (int off = LPR; off < 32; off <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
      const float mn = fmaxf(m_run[h], mt);
      const float alpha = rescale(m_run[h], mn);
      float ps = 0.f;
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        p[i][h] = mn == -INFINITY ? 0.f : exp2f((sc[i][h] - mn) * kLog2e);
        ps += p[i][h];
      }
      l_run[h] = l_run[h] * alpha + ps;
#pragma unroll
      for (int e = 0; e < EPL; ++e) o[h][e] *= alpha;
      m_run[h] = mn;
    }
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const int row = warp * Gm::RPWARP + i * RPW + rsub;
      if (row < rows) {
        float vf[EPL];
        Vec16<T>::load(vf, vs + row * RB + c16 * 16);
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int e = 0; e < EPL; ++e) o[h][e] = fmaf(p[i][h], vf[e], o[h][e]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // ---- warp -> CTA partial
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float l = l_run[h];
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      float v = o[h][e];
#pragma unroll
      for (int off = LPR; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      o[h][e] = v;
    }
    if (rsub == 0) {
#pragma unroll
      for (int e = 0; e < EPL; ++e) wo[(warp * G + h) * D + c16 * EPL + e] = o[h][e];
    }
    if (lane == 0) {
      wm[warp * G + h] = m_run[h];
      wl[warp * G + h] = l;
    }
  }
  consumers_sync();
  {
    float* part = a.part + ((int64_t)s * a.Hq + g * G) * a.splits * (D + 2);
    for (int idx = tid; idx < G * (D + 2); idx += 128) {
      const int h = idx / (D + 2), d = idx % (D + 2);
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w * G + h]);
      float acc = 0.f;
      if (d < D) {
#pragma unroll
        for (int w = 0; w < NW; ++w) acc += rescale(wm[w * G + h], M) * wo[(w * G + h) * D + d];
      } else if (d == D) {
        acc = M;
      } else {
#pragma unroll
        for (int w = 0; w < NW; ++w) acc += rescale(wm[w * G + h], M) * wl[w * G + h];
      }
      part[((int64_t)h * a.splits + split) * (D + 2) + d] = acc;
    }
  }

  // ---- append: the new row and its metadata go to cache slot n_old
  if (a.append && a.n_old >= t0 && a.n_old < t1) {
    T* kdst = static_cast<T*>(a.kc) + s * a.c_ss + (int64_t)g * a.c_hs + (int64_t)a.n_old * D;
    T* vdst = static_cast<T*>(a.vc) + s * a.c_ss + (int64_t)g * a.c_hs + (int64_t)a.n_old * D;
    for (int i = tid; i < RB / 16; i += 128) {
      reinterpret_cast<uint4*>(kdst)[i] = reinterpret_cast<const uint4*>(knew)[i];
      reinterpret_cast<uint4*>(vdst)[i] = reinterpret_cast<const uint4*>(vnew)[i];
    }
    if (g == 0 && tid == 0) {
      int64_t* np = a.next_pos + s * a.len_ss;
      const int64_t pv = a.pos_in ? a.pos_in[s] : *np;
      a.pos[s * a.m_ss + a.n_old] = pv;
      a.modality[s * a.m_ss + a.n_old] = 0;
      a.round_id[s * a.m_ss + a.n_old] = a.round_value;
      *np = pv + 1;
      a.len[s * a.len_ss] = n;
    }
  }

  // ---- previous step's window row, spread over every CTA of the launch
  fold_piece(a.fold, s, split * a.Hkv + g, a.splits * a.Hkv, a.Hq, tid, 128);

  // ---- split combine by the last CTA of (stream, kv-head)
  __threadfence();
  consumers_sync();
  if (tid == 0) {
    const int prev = atomicAdd(&a.counters[s * a.Hkv + g], 1);
    *flag = prev == a.splits - 1;
  }
  consumers_sync();
  if (!*flag) return;
  __threadfence();
  const float* part = a.part + ((int64_t)s * a.Hq + g * G) * a.splits * (D + 2);
  if (tid < G) {
    const float* ph = part + (int64_t)tid * a.splits * (D + 2);
    float M = -INFINITY;
    for (int c = 0; c < a.splits; ++c) M = fmaxf(M, __ldcg(ph + c * (D + 2) + D));
    float L = 0.f;
    for (int c = 0; c < a.splits; ++c) L += rescale(__ldcg(ph + c * (D + 2) + D), M) * __ldcg(ph + c * (D + 2) + D + 1);
    fin[2 * tid] = M;
    fin[2 * tid + 1] = L;
    if (a.stats) {
      a.stats[s * a.st_ss + (g * G + tid) * 2] = M;
      a.stats[s * a.st_ss + (g * G + tid) * 2 + 1] = L;
    }
  }
  consumers_sync();
  for (int idx = tid; idx < G * D; idx += 128) {
    const int h = idx / D, d = idx % D;
    const float* ph = part + (int64_t)h * a.splits * (D + 2);
    const float M = fin[2 * h], L = fin[2 * h + 1];
    float acc = 0.f;
    for (int c = 0; c < a.splits; ++c) acc += rescale(__ldcg(ph + c * (D + 2) + D), M) * __ldcg(ph + c * (D + 2) + d);
    a.out[s * a.o_ss + (int64_t)(g * G + h) * D + d] = acc / L;
  }
  if (tid == 0) a.counters[s * a.Hkv + g] = 0;
}

__global__ void fold_kernel(const FoldArgs f, int Hq) {
  fold_piece(f, blockIdx.y, blockIdx.x, gridDim.x, Hq, threadIdx.x, blockDim.x);
}

template <typename T, int D, int G>
static size_t decode_smem() {
  using Gm = Geo<T, D>;
  return (size_t)Gm::STAGES * 2 * Gm::TILE + 2 * Gm::STAGES * sizeof(uint64_t) +
         sizeof(float) * (2 * Gm::NW * G + Gm::NW * G * D + 2 * G) + 16;
}

template <typename T, int D, int G>
static cudaError_t launch_decode_t(int streams, const AttnArgs& a, cudaStream_t st) {
  const size_t smem = decode_smem<T, D, G>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(a.splits, a.Hkv, streams);
  decode_kernel<T, D, G><<<grid, 160, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t dispatch_group(int group, int streams, const AttnArgs& a, cudaStream_t st) {
  switch (group) {
    case 1: return launch_decode_t<T, D, 1>(streams, a, st);
    case 2: return launch_decode_t<T, D, 2>(streams, a, st);
    case 4: return launch_decode_t<T, D, 4>(streams, a, st);
    case 8: return launch_decode_t<T, D, 8>(streams, a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_decode(int dtype, int head_dim, int group, int streams, const AttnArgs& a, cudaStream_t st) {
  if (dtype == 1) {
    if (head_dim == 128) return dispatch_group<__nv_bfloat16, 128>(group, streams, a, st);
    if (head_dim == 64) return dispatch_group<__nv_bfloat16, 64>(group, streams, a, st);
  } else {
    if (head_dim == 128) return dispatch_group<float, 128>(group, streams, a, st);
    if (head_dim == 64) return dispatch_group<float, 64>(group, streams, a, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fold(int streams, int pieces, const FoldArgs& f, int Hq, cudaStream_t st) {
  if (f.n <= 0) return cudaSuccess;
  dim3 grid(pieces, streams);
  fold_kernel<<<grid, 128, 0, st>>>(f, Hq);
  return cudaGetLastError();
}

}  // namespace skv
