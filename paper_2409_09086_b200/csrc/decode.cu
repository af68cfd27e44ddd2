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
__device__ void fold_columns(const FoldArgs& f, int s, int c0, int c1, int Hq, int tid, int nthreads,
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

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// CTA that owns global tile t under the even split [c*T/P, (c+1)*T/P).
__device__ __forceinline__ int tile_owner(int64_t t, int64_t T, int P) {
  return (int)(((t + 1) * P + T - 1) / T) - 1;
}

// Persistent stream-K decode: CTA c streams the global tile range
// [c*T/P, (c+1)*T/P) of the (segment, tile) space, crossing segment (stream,
// kv-head) boundaries without draining its TMA pipeline.  At the end of each
// segment piece it publishes a partial (m, l, o) and the last contributor of
// the segment merges the pieces in CTA order (deterministic).
template <typename T, int D, int G>
__global__ void __launch_bounds__(192) decode_kernel(const AttnArgs a) {
  using Gm = Geo<T, D>;
  constexpr int TT = Gm::TT, RB = Gm::RB, LPR = Gm::LPR, EPL = Gm::EPL, RPW = Gm::RPW;
  constexpr int NW = Gm::NW, ITERS = Gm::ITERS, STAGES = Gm::STAGES, TILE = Gm::TILE;
  constexpr int PW = D + 2;  // floats per head in a partial

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* tiles = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * 2 * TILE);
  uint64_t* empty = full + STAGES;
  float* wm = reinterpret_cast<float*>(empty + STAGES);  // [NW][G]
  float* wl = wm + NW * G;                               // [NW][G]
  float* wo = wl + NW * G;                               // [NW][G][D]
  float* fin = wo + NW * G * D;                          // [G][2] merged (M, L)
  int* flag = reinterpret_cast<int*>(fin + 2 * G);
  float* fstats = fin + 2 * G + 4;                        // [Hq][2] fold warp

  const int c = blockIdx.x, P = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_old + a.append;
  const int64_t a0 = (int64_t)c * a.T / P, a1 = (int64_t)(c + 1) * a.T / P;

  griddep_launch();
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW + 1) {
    // ---------------------------------------------------------- fold warp
    // Materialises the previous recorded step's window row (64-column pieces,
    // pieces c, c+P, ...) while the other warps stream K/V: its load latency
    // is hidden behind the main loop.
    const FoldArgs& f = a.fold;
    if (f.n > 0) {
      if (!a.prefetch) griddep_wait();  // same layer back to back: wait for its logits
      const int ppc = (f.n + 63) / 64;
      for (int piece = c; piece < a.S * ppc; piece += P) {
        const int s = piece / ppc, col0 = (piece - s * ppc) * 64;
        const float* stt = f.stats + s * f.st_ss;
        for (int h = lane; h < a.Hq; h += 32) {
          fstats[2 * h] = __ldg(stt + 2 * h);
          fstats[2 * h + 1] = __ldg(stt + 2 * h + 1);
        }
        __syncwarp();
        fold_columns(f, s, col0, min(col0 + 64, f.n), a.Hq, lane, 32, fstats);
        __syncwarp();
        if (col0 == 0 && lane == 0 && f.wlen) f.wlen[s * f.w_ss] = f.n;
      }
    }
    return;
  }
  if (warp == NW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      bool waited = false;
      if (!a.prefetch) {
        griddep_wait();
        waited = true;
      }
      int i = 0;
      for (int64_t t = a0; t < a1; ++t, ++i) {
        const int sigma = (int)(t / a.nt);
        const int ts = (int)(t - (int64_t)sigma * a.nt) * TT;
        const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
        const int rows = min(TT, n - ts);
        const int rc = max(0, min(rows, a.n_old - ts));
        const int st = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        unsigned char* ks = tiles + (2 * st) * TILE;
        unsigned char* vs = ks + TILE;
        mbar_arrive_expect_tx(&full[st], 2u * rows * RB);
        const int64_t base = s * a.c_ss + (int64_t)g * a.c_hs + (int64_t)ts * D;
        if (rc > 0) {
          bulk_g2s(ks, static_cast<const T*>(a.kc) + base, rc * RB, &full[st]);
          bulk_g2s(vs, static_cast<const T*>(a.vc) + base, rc * RB, &full[st]);
        }
        if (rc < rows) {  // the appended token: straight from the step input
          if (!waited) {
            griddep_wait();
            waited = true;
          }
          const int64_t in = s * a.in_ss + (int64_t)g * D;
          bulk_g2s(ks + rc * RB, static_cast<const T*>(a.kin) + in, RB, &full[st]);
          bulk_g2s(vs + rc * RB, static_cast<const T*>(a.vin) + in, RB, &full[st]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  griddep_wait();  // q, out, logits, partials and counters cross launches
  const int rsub = lane / LPR, c16 = lane % LPR;
  float qf[G][EPL];
  float m_run[G], l_run[G], o[G][EPL];
  float* lg = nullptr;
  int cur = -1;
  int i = 0;
  for (int64_t t = a0; t < a1; ++t, ++i) {
    const int sigma = (int)(t / a.nt);
    const int tt = (int)(t - (int64_t)sigma * a.nt);
    const int ts = tt * TT;
    const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
    if (sigma != cur) {
      cur = sigma;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        Vec16<T>::load(qf[h], static_cast<const T*>(a.q) + s * a.q_ss + (int64_t)(g * G + h) * D + c16 * EPL);
        m_run[h] = -INFINITY;
        l_run[h] = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) o[h][e] = 0.f;
      }
      lg = a.logits ? a.logits + s * a.l_ss + (int64_t)(g * G) * a.l_hs : nullptr;
    }
    const int st = i % STAGES;
    const uint32_t ph = (i / STAGES) & 1;
    const int rows = min(TT, n - ts);
    const unsigned char* ks = tiles + (2 * st) * TILE;
    const unsigned char* vs = ks + TILE;
    mbar_wait(&full[st], ph);

    float sc[ITERS][G];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int row = warp * Gm::RPWARP + it * RPW + rsub;
      float kf[EPL];
      Vec16<T>::load(kf, ks + row * RB + c16 * 16);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) d = fmaf(qf[h][e], kf[e], d);
#pragma unroll
        for (int off = LPR / 2; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        sc[it][h] = row < rows ? d * a.scale : -INFINITY;
      }
    }
    if (lg && c16 == 0) {
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        const int row = warp * Gm::RPWARP + it * RPW + rsub;
        if (row < rows) {
#pragma unroll
          for (int h = 0; h < G; ++h) lg[h * a.l_hs + ts + row] = sc[it][h];
        }
      }
    }
    float p[ITERS][G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float mt = -INFINITY;
#pragma unroll
      for (int it = 0; it < ITERS; ++it) mt = fmaxf(mt, sc[it][h]);
#pragma unroll
      for (int off = LPR; off < 32; off <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
      const float mn = fmaxf(m_run[h], mt);
      const float alpha = rescale(m_run[h], mn);
      float ps = 0.f;
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        p[it][h] = mn == -INFINITY ? 0.f : exp2f((sc[it][h] - mn) * kLog2e);
        ps += p[it][h];
      }
      l_run[h] = l_run[h] * alpha + ps;
#pragma unroll
      for (int e = 0; e < EPL; ++e) o[h][e] *= alpha;
      m_run[h] = mn;
    }
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int row = warp * Gm::RPWARP + it * RPW + rsub;
      if (row < rows) {
        float vf[EPL];
        Vec16<T>::load(vf, vs + row * RB + c16 * 16);
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int e = 0; e < EPL; ++e) o[h][e] = fmaf(p[it][h], vf[e], o[h][e]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);

    if (tt != a.nt - 1 && t != a1 - 1) continue;

    // ================= end of this CTA's piece of segment sigma =================
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
      float* part = a.part + (int64_t)(sigma + c) * G * PW;
      for (int idx = tid; idx < G * PW; idx += 128) {
        const int h = idx / PW, d = idx - h * PW;
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
        part[idx] = acc;
      }
    }
    // append: the new row and (once per stream) its metadata go to slot n_old
    if (a.append && tt == a.nt - 1) {
      const int64_t dst = s * a.c_ss + (int64_t)g * a.c_hs + (int64_t)a.n_old * D;
      const int64_t in = s * a.in_ss + (int64_t)g * D;
      for (int u = tid; u < RB / 16; u += 128) {
        reinterpret_cast<uint4*>(static_cast<T*>(a.kc) + dst)[u] =
            reinterpret_cast<const uint4*>(static_cast<const T*>(a.kin) + in)[u];
        reinterpret_cast<uint4*>(static_cast<T*>(a.vc) + dst)[u] =
            reinterpret_cast<const uint4*>(static_cast<const T*>(a.vin) + in)[u];
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
    __threadfence();
    consumers_sync();
    const int64_t seg0 = (int64_t)sigma * a.nt;
    const int c_lo = tile_owner(seg0, a.T, P);
    const int c_hi = tile_owner(seg0 + a.nt - 1, a.T, P);
    if (tid == 0) {
      const int prev = atomicAdd(&a.counters[sigma], 1);
      *flag = prev == c_hi - c_lo;
    }
    consumers_sync();
    if (*flag) {
      __threadfence();
      if (tid < G) {
        float M = -INFINITY;
        for (int cc = c_lo; cc <= c_hi; ++cc) M = fmaxf(M, __ldcg(a.part + ((int64_t)(sigma + cc) * G + tid) * PW + D));
        float L = 0.f;
        for (int cc = c_lo; cc <= c_hi; ++cc) {
          const float* pp = a.part + ((int64_t)(sigma + cc) * G + tid) * PW;
          L += rescale(__ldcg(pp + D), M) * __ldcg(pp + D + 1);
        }
        fin[2 * tid] = M;
        fin[2 * tid + 1] = L;
        if (a.stats) {
          a.stats[s * a.st_ss + (g * G + tid) * 2] = M;
          a.stats[s * a.st_ss + (g * G + tid) * 2 + 1] = L;
        }
      }
      consumers_sync();
      for (int idx = tid; idx < G * D; idx += 128) {
        const int h = idx / D, d = idx - h * D;
        const float M = fin[2 * h], L = fin[2 * h + 1];
        float acc = 0.f;
        for (int cc = c_lo; cc <= c_hi; ++cc) {
          const float* pp = a.part + ((int64_t)(sigma + cc) * G + h) * PW;
          acc += rescale(__ldcg(pp + D), M) * __ldcg(pp + d);
        }
        a.out[s * a.o_ss + (int64_t)(g * G + h) * D + d] = acc / L;
      }
      if (tid == 0) a.counters[sigma] = 0;
    }
    consumers_sync();
  }
}

__global__ void fold_kernel(const FoldArgs f, int Hq) {
  fold_piece(f, blockIdx.y, blockIdx.x, gridDim.x, Hq, threadIdx.x, blockDim.x);
}

template <typename T, int D, int G>
static size_t decode_smem() {
  using Gm = Geo<T, D>;
  return (size_t)Gm::STAGES * 2 * Gm::TILE + 2 * Gm::STAGES * sizeof(uint64_t) +
         sizeof(float) * (2 * Gm::NW * G + Gm::NW * G * D + 2 * G + 4);
}

template <typename T, int D, int G>
static cudaError_t launch_decode_t(int ctas, const AttnArgs& a, cudaStream_t st) {
  const size_t smem = decode_smem<T, D, G>() + 8 * (size_t)a.Hq;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(decode_smem<T, D, G>() + 8 * 1024));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_kernel<T, D, G>, a);
}

template <typename T, int D, int G>
static int occupancy_t() {
  static int occ = 0;
  if (!occ) {
    const size_t smem = decode_smem<T, D, G>() + 8 * 64;
    cudaFuncSetAttribute(decode_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(decode_smem<T, D, G>() + 8 * 1024));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decode_kernel<T, D, G>, 192, smem) != cudaSuccess ||
        occ < 1)
      occ = 1;
  }
  return occ;
}

template <typename T, int D>
static cudaError_t dispatch_group(int group, int ctas, const AttnArgs& a, cudaStream_t st) {
  switch (group) {
    case 1: return launch_decode_t<T, D, 1>(ctas, a, st);
    case 2: return launch_decode_t<T, D, 2>(ctas, a, st);
    case 4: return launch_decode_t<T, D, 4>(ctas, a, st);
    case 8: return launch_decode_t<T, D, 8>(ctas, a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int D>
static int occ_group(int group) {
  switch (group) {
    case 1: return occupancy_t<T, D, 1>();
    case 2: return occupancy_t<T, D, 2>();
    case 4: return occupancy_t<T, D, 4>();
    case 8: return occupancy_t<T, D, 8>();
    default: return 1;
  }
}

int decode_ctas_per_sm(int dtype, int head_dim, int group) {
  if (dtype == 1) return head_dim == 128 ? occ_group<__nv_bfloat16, 128>(group) : occ_group<__nv_bfloat16, 64>(group);
  return head_dim == 128 ? occ_group<float, 128>(group) : occ_group<float, 64>(group);
}

cudaError_t launch_decode(int dtype, int head_dim, int group, int ctas, const AttnArgs& a, cudaStream_t st) {
  if (dtype == 1) {
    if (head_dim == 128) return dispatch_group<__nv_bfloat16, 128>(group, ctas, a, st);
    if (head_dim == 64) return dispatch_group<__nv_bfloat16, 64>(group, ctas, a, st);
  } else {
    if (head_dim == 128) return dispatch_group<float, 128>(group, ctas, a, st);
    if (head_dim == 64) return dispatch_group<float, 64>(group, ctas, a, st);
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
