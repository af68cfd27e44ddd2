// K1 small-batch GQA variant: the decode of a latency-bound launch (one
// chunk per CTA, the static schedule of config 3) on the tensor cores with
// warp-level mma.sync, so each CTA's math fits in a few hundred instructions
// per warp instead of ~1000 CUDA-core instructions per 64-token tile.
//
// Same contract as decode_kernel (Session._attend + KvCache.append, reference
// engine.py:235-246, 264): per (stream, kv-head) segment the chunk's partial
// (o, m, l) per query head, published to merge_kernel.  Per CTA:
//   * the producer warp loads the chunk's K and V tiles (64 rows x 128 dims,
//     bf16) with cp.async.bulk.tensor into 128-byte-swizzled shared memory,
//     before griddepcontrol.wait (PDL prefetch); if the chunk holds the
//     appended token, the new k/v row is written into its slot after release;
//   * consumer warp w owns 32 keys: S = Q K^T with mma.m16n8k16 (M = the
//     group's query heads padded to 16, N = 8 keys, K = 16 dims; B fragments
//     by ldmatrix from the swizzled tile, conflict-free), softmax over its 32
//     keys in registers, then O = P V with P taken straight from the S
//     accumulators (the flash-attention register trick) as two bf16 terms
//     (hi + lo: a single bf16 P would carry 2^-8 relative error) and V
//     fragments by ldmatrix.trans;
//   * the warps' (m, l, o) are merged in chunk order by all consumer threads
//     and published like the CUDA-core kernel's static path.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "skv_common.cuh"
#include "skv_append.cuh"
#include "skv_fold.cuh"
#include "skv_internal.h"

namespace skv {
namespace tcd {

constexpr int D = 128;
constexpr int TT = 64;                 // rows per tile
constexpr int REGION = TT * 128;       // [64 rows][64 bf16] swizzled, 8 KB
constexpr int TILE = 2 * REGION;       // 64 rows x 128 dims, 16 KB
constexpr int MAXT = 4;                // tiles per chunk (8 warps x 32 keys)
constexpr int NW = 8;                  // consumer warps
constexpr int CT = NW * 32;
constexpr int THREADS = CT + 96;       // + producer, (idle) epilogue, fold warps
constexpr int PW = D + 2;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D = A(16x16, rows 8..15 zero) . B(16x8) + D, bf16 inputs, f32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// byte offset of (row r of a 64-row tile, 16-byte dim chunk cd in 0..15)
__device__ __forceinline__ uint32_t swz(int r, int cd) {
  return (uint32_t)((cd >> 3) * REGION + r * 128 + (((cd & 7) ^ (r & 7)) << 4));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(CT) : "memory"); }
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ float rescale(float m, float M) { return m == -INFINITY ? 0.f : exp2f((m - M) * kLog2e); }
__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int G>
struct Smem {
  static constexpr size_t tiles = (size_t)2 * MAXT * TILE;  // K tiles then V tiles
  static constexpr size_t slot_floats = 4 + 2 * NW * G + NW * G * D;
  static constexpr size_t bytes = tiles + slot_floats * 4 + 64 + 1024 + 8 * 1024;  // + bars, align, fold stats
};

// decode_tc_kernel's shared memory for chunks of MT tiles (2 MT consumer warps);
// Hq query heads' fold stats
template <int G, int MT>
struct SmemT {
  static constexpr int NWK = 2 * MT;
  static constexpr int THREADS = NWK * 32 + 96;
  static constexpr size_t tiles = (size_t)2 * MT * TILE;
  static constexpr size_t slot_floats = 4 + 2 * NWK * G + NWK * G * D;
  static size_t bytes(int Hq) { return tiles + slot_floats * 4 + 64 + 1024 + (size_t)Hq * 8; }
};

}  // namespace tcd

namespace tcd {

// D = A(16x16) . B(16x8) + D, bf16 inputs, f32 accumulate (all four A registers)
__device__ __forceinline__ void mma16816_a4(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Transpose of an 8x8 b16 matrix held in the accumulator layout (row lane/4,
// columns 2(lane%4), +1) into the same layout.
__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

// One consumer warp's 32 keys [wk0, wk0 + 32) of the chunk in shared memory,
// keys along the MMA's M dimension and the group's query heads along N (8
// columns: G of them real), so no MMA row is padding:
//   S^T (16 keys x 8 heads) = K (16 keys x 16 dims, ldmatrix from the swizzled
//   tile) . Q^T (16 dims x 8 heads, the q fragments qb, fixed for the launch),
// then the softmax over the warp's keys per head: p = exp2((x - m) log2e), head
// max m and sum l.  Lane (gid, tig) holds keys wk0 + 16 mt + gid (+8) of heads
// 2 tig, 2 tig + 1 (m[e], l[e] for head 2 tig + e).  Recorded steps store the
// raw logits x = s * scale to lg + head * lg_hs (null: not recorded).
__device__ __forceinline__ void warp_scores(const uint32_t (&qb)[8][2], uint32_t kbase, int wk0, int lane, int k0,
                                            int kend, float scale, float* lg, int64_t lg_hs, int G, float (&p)[2][4],
                                            float (&m)[2], float (&l)[2]) {
  const int gid = lane >> 2, tig = lane & 3;
  float sacc[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    sacc[mt][0] = sacc[mt][1] = sacc[mt][2] = sacc[mt][3] = 0.f;
    const int kk = wk0 + 16 * mt + (lane & 7) + 8 * ((lane >> 3) & 1);  // key row this lane addresses
    const int t = kk >> 6, r = kk & 63;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(kbase + t * TILE + swz(r, 2 * ks + (lane >> 4)), a0, a1, a2, a3);
      mma16816_a4(sacc[mt], a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
    }
  }
  float x[2][4];
  float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int key = k0 + wk0 + 16 * mt + gid + (c >> 1) * 8;
      x[mt][c] = key < kend ? sacc[mt][c] * scale : -INFINITY;
      mx[c & 1] = fmaxf(mx[c & 1], x[mt][c]);
    }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
#pragma unroll
    for (int sh = 4; sh < 32; sh <<= 1) mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], sh));
    m[e] = mx[e];
  }
  float ls[2] = {0.f, 0.f};
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      p[mt][c] = m[c & 1] == -INFINITY ? 0.f : fast_exp2((x[mt][c] - m[c & 1]) * kLog2e);
      ls[c & 1] += p[mt][c];
    }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
#pragma unroll
    for (int sh = 4; sh < 32; sh <<= 1) ls[e] += __shfl_xor_sync(0xffffffffu, ls[e], sh);
    l[e] = ls[e];
  }
  if (lg) {  // recorded steps: raw f32 logits for the window fold
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * tig + e;
      if (h >= G) continue;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {
          const int key = k0 + wk0 + 16 * mt + gid + 8 * hi;
          if (key < kend) lg[h * lg_hs + key] = x[mt][2 * hi + e];
        }
    }
  }
}

// O^T (16 dims x 8 heads) += V^T (16 dims x 16 keys, ldmatrix.trans) . P^T
// (16 keys x 8 heads) over the warp's 32 keys: P^T fragments are the score
// accumulators transposed in registers (movmatrix), as two bf16 terms (hi + lo).
// Lane (gid, tig) holds o[md] = dims 16 md + gid (c 0, 1) and + 8 (c 2, 3) of
// heads 2 tig + (c & 1).
__device__ __forceinline__ void warp_pv(const float (&p)[2][4], uint32_t vbase, int wk0, int lane, float (&o)[8][4]) {
#pragma unroll
  for (int kq = 0; kq < 2; ++kq) {
    const uint32_t h0 = pack_bf16(p[kq][0], p[kq][1]), h1 = pack_bf16(p[kq][2], p[kq][3]);
    const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h0));
    const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h1));
    const uint32_t l0 = pack_bf16(p[kq][0] - f0.x, p[kq][1] - f0.y), l1 = pack_bf16(p[kq][2] - f1.x, p[kq][3] - f1.y);
    const uint32_t bh0 = movtrans(h0), bh1 = movtrans(h1), bl0 = movtrans(l0), bl1 = movtrans(l1);
    // lane's ldmatrix.trans row: key 16 kq + (lane & 7) + 8 (lane >> 4), dim chunk 2 md + ((lane >> 3) & 1)
    const int kk = wk0 + 16 * kq + (lane & 7) + 8 * (lane >> 4);
    const int t = kk >> 6, r = kk & 63;
#pragma unroll
    for (int md = 0; md < 8; ++md) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4_t(vbase + t * TILE + swz(r, 2 * md + ((lane >> 3) & 1)), a0, a1, a2, a3);
      mma16816_a4(o[md], a0, a1, a2, a3, bh0, bh1);
      mma16816_a4(o[md], a0, a1, a2, a3, bl0, bl1);
    }
  }
}

// The warp's partial into shared memory: wo[h][D] (h < G), wm[h], wl[h].
__device__ __forceinline__ void warp_stage(const float (&o)[8][4], const float (&m)[2], const float (&l)[2], int lane,
                                           int G, float* wo, float* wm, float* wl) {
  const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int h = 2 * tig + e;
    if (h >= G) continue;
#pragma unroll
    for (int md = 0; md < 8; ++md) {
      wo[h * D + 16 * md + gid] = o[md][e];
      wo[h * D + 16 * md + gid + 8] = o[md][2 + e];
    }
    if (gid == 0) {
      wm[h] = m[e];
      wl[h] = l[e];
    }
  }
}

}  // namespace tcd


// One CTA = chunk blockIdx.x (static schedule): segment sigma = c / nc,
// tiles [j*ch, min((j+1)*ch, nt)).
template <int G, int MT>
__global__ void __launch_bounds__(tcd::SmemT<G, MT>::THREADS, (MT <= 2 ? 3 : 1))
    decode_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                     const AttnArgs a) {
  using namespace tcd;
  constexpr int MAXT = MT, NW = 2 * MT, CT = NW * 32;  // chunk tiles, consumer warps / threads
  using Smem = tcd::SmemT<G, MT>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align up by offset from the array (keeps the shared state space: LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  unsigned char* ktiles = smem;
  unsigned char* vtiles = smem + MAXT * TILE;
  float* slot = reinterpret_cast<float*>(smem + Smem::tiles);
  uint64_t* bars = reinterpret_cast<uint64_t*>(slot + Smem::slot_floats);
  uint64_t* full = bars;      // TMA of every tile
  uint64_t* row_ok = bars + 1;  // appended row written (chunks that hold it)
  float* fstats = reinterpret_cast<float*>(bars + 4);  // fold warp: [Hq][2]

  const int c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_old + a.append;
  const int sigma = c / a.nc, j = c - sigma * a.nc;
  const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
  const int tt0 = j * a.ch, tt1 = min(tt0 + a.ch, a.nt);
  const int ntile = tt1 - tt0;
  const int k0 = tt0 * TT;                       // first key of the chunk
  const int kend = min(tt1 * TT, n);             // keys [k0, kend) are valid
  const bool has_new = a.append && a.n_old >= k0 && a.n_old < kend;
  const int seg_row = (int)(((int64_t)s * a.L + a.layer) * a.Hkv + g) * a.cap;

  if (a.tstamp && tid == 0) atomicMin(&a.tstamp[0], gtimer());
  if (a.ctat && tid == 0) a.ctat[8 * blockIdx.x] = gtimer();
  if (tid == 0) {
    mbar_init(full, 1);
    mbar_init(row_ok, 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------------------------------------------------- producer
    if (!a.prefetch) griddep_wait();  // same layer back to back: its appended row
    if (lane == 0) {
      mbar_arrive_expect_tx(full, 2u * ntile * TILE);
      for (int t = 0; t < ntile; ++t) {
        const int y = seg_row + (tt0 + t) * TT;
        tma_load_2d(ktiles + t * TILE, &kmap, 0, y, full);
        tma_load_2d(ktiles + t * TILE + REGION, &kmap, 64, y, full);
        tma_load_2d(vtiles + t * TILE, &vmap, 0, y, full);
        tma_load_2d(vtiles + t * TILE + REGION, &vmap, 64, y, full);
      }
    }
    if (has_new) {
      // the new token's k/v (a real model's previous-layer output) cross the
      // launch: after release, over the TMA copy of its (stale) cache slot
      griddep_wait();
      mbar_wait(full, 0);
      const int kk = a.n_old - k0, t = kk / TT, r = kk % TT;
      const int cd = lane & 15;
      const uint4* in = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(lane < 16 ? a.kin : a.vin) +
                                                       s * a.in_ss + (int64_t)g * D);
      unsigned char* dst = (lane < 16 ? ktiles : vtiles) + t * TILE + swz(r, cd);
      *reinterpret_cast<uint4*>(dst) = in[cd];
      __syncwarp();
      if (lane == 0) mbar_arrive(row_ok);
    }
    return;
  }

  if (warp == NW + 2) {
    // ------------------------------------------------- window-row fold warp
    const FoldArgs& f = a.fold;
    if (f.n <= 0) return;
    if (!a.prefetch) griddep_wait();
    const int P = gridDim.x;
    const int ppc = (f.n + 63) / 64;
    for (int piece = c; piece < a.S * ppc; piece += P) {
      const int s2 = piece / ppc, col0 = (piece - s2 * ppc) * 64;
      const float* stt = f.stats + s2 * f.st_ss;
      for (int h = lane; h < a.Hq; h += 32) {
        fstats[2 * h] = __ldg(stt + 2 * h);
        fstats[2 * h + 1] = __frcp_rn(__ldg(stt + 2 * h + 1));  // staged as 1/L
      }
      __syncwarp();
      fold_columns(f, s2, col0, min(col0 + 64, f.n), a.Hq, lane, 32, fstats);
      __syncwarp();
      if (col0 == 0 && lane == 0 && f.wlen) f.wlen[s2 * f.w_ss] = f.n;
    }
    if (a.ctat && lane == 0) a.ctat[8 * c + 6] = gtimer();  // instrumentation: fold warp done
    return;
  }

  if (warp == NW + 1) return;  // (the append is done by the consumers before they publish)

  // ------------------------------------------------------------ consumers
  griddep_wait();
  if (tid == 0) griddep_launch();
  if (a.ctat && tid == 0) a.ctat[8 * c + 1] = gtimer();
  const int gid = lane >> 2, tig = lane & 3;
  const bool real = gid < G;  // rows >= G of the 16-row MMA are padding
  // q A-fragments (row gid = head g*G + gid): a0 = q[16ks + 2tig..+1], a2 = q[16ks + 8 + 2tig..+1]
  uint32_t qa[8][2];
  {
    const uint32_t* qrow =
        reinterpret_cast<const uint32_t*>(static_cast<const __nv_bfloat16*>(a.q) + s * a.q_ss + (int64_t)(g * G + (real ? gid : 0)) * D);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = real ? qrow[8 * ks + tig] : 0u;
      qa[ks][1] = real ? qrow[8 * ks + 4 + tig] : 0u;
    }
  }
  mbar_wait(full, 0);
  if (has_new) mbar_wait(row_ok, 0);

  const int wk0 = warp * 32;  // this warp's keys [wk0, wk0 + 32) of the chunk
  const uint32_t kbase = smem_u32(ktiles), vbase = smem_u32(vtiles);
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float* lg = a.logits ? a.logits + s * a.l_ss + (int64_t)(g * G) * a.l_hs : nullptr;
  if (wk0 < ntile * TT) {
    float p[2][4];
    warp_scores(qa, kbase, wk0, lane, k0, kend, a.scale, lg, a.l_hs, G, p, m, l);
    warp_pv(p, vbase, wk0, lane, o);
  }
  // ---- warp partials to the slot: wm[NW][G], wl[NW][G], wo[NW][G][D]
  float* wm = slot + 4;
  float* wl = wm + NW * G;
  float* wo = wl + NW * G;
  warp_stage(o, m, l, lane, G, wo + warp * G * D, wm + warp * G, wl + warp * G);
  bar_sync_n(1, CT);
  if (a.ctat && tid == 0) a.ctat[8 * c + 3] = gtimer();
  // ---- merge the warp partials in warp order and publish the chunk partial
  // KvCache.append: the segment's last chunk stores the new row and its
  // metadata before publishing (the merge, and so the next launch, sees them)
  if (a.append && j == a.nc - 1) append_row<__nv_bfloat16, D>(a, sigma, n, tid, CT);
  float* part = a.part + ((int64_t)sigma * a.nc + j) * G * PW;
  for (int idx = tid; idx < G * D; idx += CT) {
    const int h = idx / D, d = idx - h * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w * G + h]);
    float f[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) f[w] = rescale(wm[w * G + h], M);
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) acc = fmaf(f[w], wo[(w * G + h) * D + d], acc);
    part[h * PW + d] = acc;
    if (d == 0) {
      float xs[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) xs[w] = f[w] * wl[w * G + h];
#pragma unroll
      for (int off = NW / 2; off > 0; off >>= 1)
#pragma unroll
        for (int w = 0; w < off; ++w) xs[w] = xs[w] + xs[w + off];
      part[h * PW + D] = M;
      part[h * PW + D + 1] = xs[0];
    }
  }
  bar_sync_n(1, CT);
  if (tid == 0) {
    red_release_add(&a.counters[sigma], 1);
    if (a.tstamp) atomicMax(&a.tstamp[1], gtimer());
    if (a.ctat) a.ctat[8 * c + 2] = gtimer();
  }
}

// ---------------------------------------------------------------------------
// All layers of one token in one persistent launch (static schedule: CTA c
// owns chunk j of segment sigma in every layer).  Per layer l the producer
// streams the chunk's K tiles as soon as the consumers are done with layer
// l-1's K (and V likewise), so layer l's cache is in shared memory before its
// queries are released; the consumers wait for layer l-1's outputs
// (layer_done[l-1], the model's dependency; griddepcontrol.wait for layer 0),
// compute the chunk exactly like decode_tc_kernel and publish its partial;
// the CTA whose publication completes the segment merges it (merge_kernel's
// arithmetic and order) and releases layer_done[l].  No launch or grid
// completion sits on the layer-to-layer chain.  All CTAs must be co-resident
// (grid <= SMs at one CTA per SM); dependents launch only after every CTA has
// started (griddepcontrol.launch_dependents after layer 0's release).
template <int G>
__global__ void __launch_bounds__(tcd::THREADS, 1)
    decode_tc_layers_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                            const AttnArgs a, const LayerSteps ls) {
  using namespace tcd;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align up by offset from the array (keeps the shared state space: LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  unsigned char* ktiles = smem;
  unsigned char* vtiles = smem + MAXT * TILE;
  float* slot = reinterpret_cast<float*>(smem + Smem<G>::tiles);
  uint64_t* bars = reinterpret_cast<uint64_t*>(slot + Smem<G>::slot_floats);
  uint64_t* kfull = bars;      // layer l's K tiles landed (phase l & 1)
  uint64_t* vfull = bars + 1;
  uint64_t* kfree = bars + 2;  // consumers done with layer l's K
  uint64_t* vfree = bars + 3;
  float* fstats = reinterpret_cast<float*>(bars + 4);  // fold warp: [Hq][2]
  int* merger = reinterpret_cast<int*>(slot);          // slot[0]: this CTA merges the segment

  const int c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_old + a.append;
  const int sigma = c / a.nc, j = c - sigma * a.nc;
  const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
  const int segs = a.S * a.Hkv;
  const int tt0 = j * a.ch, tt1 = min(tt0 + a.ch, a.nt);
  const int ntile = tt1 - tt0;
  const int k0 = tt0 * TT;
  const int kend = min(tt1 * TT, n);
  const bool has_new = a.append && a.n_old >= k0 && a.n_old < kend;
  // the previous token's row (appended by the preceding launch) lies in this chunk
  const bool has_prev = a.n_old - 1 >= k0 && a.n_old - 1 < kend;

  if (tid == 0) {
    mbar_init(kfull, 1);
    mbar_init(vfull, 1);
    mbar_init(kfree, NW);
    mbar_init(vfree, NW);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      if (!ls.prefetch0 || has_prev) griddep_wait();  // rows the preceding launch wrote
      for (int l = 0; l < ls.L; ++l) {
        const int seg_row = (int)(((int64_t)s * a.L + a.layer + l) * a.Hkv + g) * a.cap;
        if (l > 0) mbar_wait(kfree, (l - 1) & 1);
        mbar_arrive_expect_tx(kfull, (uint32_t)ntile * TILE);
        for (int t = 0; t < ntile; ++t) {
          const int y = seg_row + (tt0 + t) * TT;
          tma_load_2d(ktiles + t * TILE, &kmap, 0, y, kfull);
          tma_load_2d(ktiles + t * TILE + REGION, &kmap, 64, y, kfull);
        }
        if (l > 0) mbar_wait(vfree, (l - 1) & 1);
        mbar_arrive_expect_tx(vfull, (uint32_t)ntile * TILE);
        for (int t = 0; t < ntile; ++t) {
          const int y = seg_row + (tt0 + t) * TT;
          tma_load_2d(vtiles + t * TILE, &vmap, 0, y, vfull);
          tma_load_2d(vtiles + t * TILE + REGION, &vmap, 64, y, vfull);
        }
      }
    }
    return;
  }

  if (warp == NW + 2) {
    // ------------------------------------------------- window-row fold warp
    // the previous token's recorded rows of every layer (written by the
    // preceding launch) materialise into their ring slots
    if (a.fold.n <= 0) return;
    griddep_wait();
    const int P = gridDim.x;
    const int ppc = (a.fold.n + 63) / 64;
    for (int l = 0; l < ls.L; ++l) {
      FoldArgs f = a.fold;
      f.logits += l * ls.lg_ls;
      f.stats += l * ls.st_ls;
      f.rows += l * ls.fr_ls;
      if (f.wlen) f.wlen += l * ls.fw_ls;
      for (int piece = c; piece < a.S * ppc; piece += P) {
        const int s2 = piece / ppc, col0 = (piece - s2 * ppc) * 64;
        const float* stt = f.stats + s2 * f.st_ss;
        for (int h = lane; h < a.Hq; h += 32) {
          fstats[2 * h] = __ldg(stt + 2 * h);
          fstats[2 * h + 1] = __frcp_rn(__ldg(stt + 2 * h + 1));  // staged as 1/L
        }
        __syncwarp();
        fold_columns(f, s2, col0, min(col0 + 64, f.n), a.Hq, lane, 32, fstats);
        __syncwarp();
        if (col0 == 0 && lane == 0 && f.wlen) f.wlen[s2 * f.w_ss] = f.n;
      }
    }
    return;
  }

  if (warp == NW + 1) return;

  // ------------------------------------------------------------ consumers
  const int gid = lane >> 2, tig = lane & 3;
  const bool real = gid < G;  // rows >= G of the 16-row MMA are padding
  const uint32_t kbase = smem_u32(ktiles), vbase = smem_u32(vtiles);
  const int wk0 = warp * 32;
  float* wm = slot + 4;
  float* wl = wm + NW * G;
  float* wo = wl + NW * G;
  for (int l = 0; l < ls.L; ++l) {
    // ---- layer l's inputs are the previous layer's outputs in a real model
    if (l == 0) {
      griddep_wait();
      if (tid == 0) griddep_launch();  // every CTA has started: dependents cannot starve this grid
    } else {
      if (tid == 0)
        while (ld_acquire(&ls.layer_done[l - 1]) < segs) {
        }
      consumers_sync();
    }
    unsigned long long* tl = ls.tl && c < 148 ? ls.tl + ((int64_t)l * 148 + c) * 16 : nullptr;
    if (tl && tid == 0) tl[0] = gtimer();  // released
    const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(a.q) + l * ls.q_ls;
    uint32_t qa[8][2];
    {
      const uint32_t* qrow =
          reinterpret_cast<const uint32_t*>(q + s * a.q_ss + (int64_t)(g * G + (real ? gid : 0)) * D);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qa[ks][0] = real ? qrow[8 * ks + tig] : 0u;
        qa[ks][1] = real ? qrow[8 * ks + 4 + tig] : 0u;
      }
    }
    const uint32_t ph = l & 1;
    if (tl && tid == 0) tl[1] = gtimer();  // q loaded
    mbar_wait(kfull, ph);
    if (tl && tid == 0) tl[2] = gtimer();  // K tiles in
    if (has_new) {
      // the new token's k/v replace their (stale) cache slot in the tiles
      if (warp == 0) {
        if (lane >= 16) mbar_wait(vfull, ph);
        const int kk = a.n_old - k0, t = kk / TT, r = kk % TT;
        const int cd = lane & 15;
        const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(lane < 16 ? a.kin : a.vin) + l * ls.in_ls;
        const uint4* in = reinterpret_cast<const uint4*>(src + s * a.in_ss + (int64_t)g * D);
        *reinterpret_cast<uint4*>((lane < 16 ? ktiles : vtiles) + t * TILE + swz(r, cd)) = in[cd];
      }
      consumers_sync();
    }
    float m[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
    float o[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float* lg = a.logits ? a.logits + l * ls.lg_ls + s * a.l_ss + (int64_t)(g * G) * a.l_hs : nullptr;
    float p[2][4];
    const bool active = wk0 < ntile * TT;
    if (active) warp_scores(qa, kbase, wk0, lane, k0, kend, a.scale, lg, a.l_hs, G, p, m, lsum);
    __syncwarp();
    if (lane == 0) mbar_arrive(kfree);
    mbar_wait(vfull, ph);
    if (active) warp_pv(p, vbase, wk0, lane, o);
    __syncwarp();
    if (lane == 0) mbar_arrive(vfree);
    if (tl && tid == 0) tl[3] = gtimer();  // warp 0 math done
    // ---- warp partials -> chunk partial (decode_tc_kernel's order)
    warp_stage(o, m, lsum, lane, G, wo + warp * G * D, wm + warp * G, wl + warp * G);
    consumers_sync();
    if (a.append && j == a.nc - 1) {
      AttnArgs al = a;  // layer l's cache rows and token metadata
      al.kc = static_cast<__nv_bfloat16*>(a.kc) + l * ls.kv_ls;
      al.vc = static_cast<__nv_bfloat16*>(a.vc) + l * ls.kv_ls;
      al.kin = static_cast<const __nv_bfloat16*>(a.kin) + l * ls.in_ls;
      al.vin = static_cast<const __nv_bfloat16*>(a.vin) + l * ls.in_ls;
      al.pos = a.pos + l * ls.m_ls;
      al.modality = a.modality + l * ls.m_ls;
      al.round_id = a.round_id + l * ls.m_ls;
      al.len = a.len + l;
      al.next_pos = a.next_pos + l;
      append_row<__nv_bfloat16, D>(al, sigma, n, tid, CT);
    }
    float* part = a.part + ((int64_t)sigma * a.nc + j) * G * PW;
    for (int idx = tid; idx < G * D; idx += CT) {
      const int h = idx / D, d = idx - h * D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w * G + h]);
      float f[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) f[w] = rescale(wm[w * G + h], M);
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc = fmaf(f[w], wo[(w * G + h) * D + d], acc);
      part[h * PW + d] = acc;
      if (d == 0) {
        float xs[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) xs[w] = f[w] * wl[w * G + h];
#pragma unroll
        for (int off = NW / 2; off > 0; off >>= 1)
#pragma unroll
          for (int w = 0; w < off; ++w) xs[w] = xs[w] + xs[w + off];
        part[h * PW + D] = M;
        part[h * PW + D + 1] = xs[0];
      }
    }
    consumers_sync();
    if (tid == 0) {
      int old;  // publish; the chunk completing the segment merges it
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;\n" : "=r"(old) : "l"(&ls.seg_count[sigma]) : "memory");
      *merger = old == a.nc - 1;
      if (tl) tl[4] = gtimer();  // published
    }
    consumers_sync();
    if (*merger) {
      // ---- segment merge (merge_kernel's arithmetic): chunk weights per head
      // by warp h, then each output element over the chunks in order
      const int nc = a.nc;
      const float* seg = a.part + (int64_t)sigma * nc * G * PW;
      float* fac = wo;  // the warp partials are consumed
      float* stats = a.stats + l * ls.st_ls;
      if (warp < G) {
        const int hh = warp;
        float mj[4], lj[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int jj = lane + 32 * k;
          mj[k] = jj < nc ? __ldcg(seg + (jj * G + hh) * PW + D) : -INFINITY;
          lj[k] = jj < nc ? __ldcg(seg + (jj * G + hh) * PW + D + 1) : 0.f;
        }
        float M = fmaxf(fmaxf(mj[0], mj[1]), fmaxf(mj[2], mj[3]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        float L = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int jj = lane + 32 * k;
          if (jj < nc) {
            const float w = rescale(mj[k], M);
            fac[hh * nc + jj] = w;
            L += w * lj[k];
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
        if (lane == 0) {
          fac[G * nc + hh] = L;
          stats[s * a.st_ss + (g * G + hh) * 2] = M;
          stats[s * a.st_ss + (g * G + hh) * 2 + 1] = L;
        }
      }
      consumers_sync();
      float* out = a.out + l * ls.o_ls + s * a.o_ss + (int64_t)(g * G) * D;
      for (int idx = tid; idx < G * D; idx += CT) {
        const int h = idx / D, d = idx - h * D;
        const float* wf = fac + h * nc;
        const float* pp = seg + h * PW + d;
        float acc = 0.f;
        for (int jj = 0; jj < nc; ++jj) acc = fmaf(wf[jj], __ldcg(pp + jj * G * PW), acc);
        out[idx] = acc / fac[G * nc + h];
      }
      consumers_sync();
      if (tid == 0) {
        ls.seg_count[sigma] = 0;
        red_release_add(&ls.layer_done[l], 1);
        if (tl) tl[5] = gtimer();  // segment merged + released
      }
    }
  }
  if (tid == 0) {
    // the last CTA out resets the layer counters for the next launch (the
    // next launch's consumers read them only after griddepcontrol.wait)
    if (atomicAdd(ls.exit_count, 1) == (int)gridDim.x - 1) {
      for (int l = 0; l < ls.L; ++l) ls.layer_done[l] = 0;
      *ls.exit_count = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// All layers of one token, one thread-block cluster per (stream, kv-head)
// segment: cluster rank j owns chunk j (tiles [j ch, (j+1) ch)) in every layer,
// so the cluster's CTAs are co-resident for the whole token and the segment
// merge runs over distributed shared memory instead of a global round trip:
//   * every rank combines its warps' partials (staged in the K rows each warp
//     scored) and pushes the chunk partial of each output element straight
//     into the owning rank's receive buffer (st.async, completing bytes on that
//     rank's `ready` mbarrier), and its (m, l) per head to every rank;
//   * every rank waits on its own `ready` (its expected byte count), merges its
//     slice of the segment's outputs from local shared memory (merge_kernel's
//     arithmetic: chunk weights rescale(m_j, M), L = sum w_j l_j,
//     out = sum_j w_j o_j / L in chunk order), stores them and releases
//     layer_done[l] (target: segments x ranks);
//   * layer l+1's consumers wait for layer_done[l] (the model's dependency),
//     while the producer has already streamed layer l+1's K/V into the tiles
//     freed by layer l, and its warp appends layer l's token.
template <int G, int MT>
struct ClSmem {
  static constexpr int NWC = 2 * MT;                        // consumer warps (32 keys each)
  static constexpr int THREADS = NWC * 32 + 64;             // + producer and fold warps
  static constexpr size_t tiles = (size_t)2 * MT * tcd::TILE;
  // Each warp's partial (o [G][D], then m [G], l [G]) is staged in the K rows it
  // alone has just scored (its 32 rows: 4 KB in each half of the swizzled tile),
  // so no shared memory is set aside for it.
  static_assert(G * tcd::D * 4 <= 4096, "warp partial must fit the warp's consumed K rows");
  // receive buffer (one: layer l+1's pushes follow every rank's layer-l merge):
  // [CS][per] chunk-partial values of the elements this rank owns, then
  // [CS][G][2] every rank's (m, l) per head, then the merge's [CS][G] chunk
  // weights and [G] maxima
  __host__ __device__ static int per(int cs) { return ((G * tcd::D + cs - 1) / cs + 3) / 4 * 4; }
  __host__ __device__ static int recv_floats(int cs) { return cs * per(cs) + 2 * G * cs + (cs + 1) * G; }
  __device__ static uint32_t recv_bytes(int cs, int rank) {
    const int cnt = max(0, min(per(cs), G * tcd::D - rank * per(cs)));
    return (uint32_t)(cs * cnt + cs * G * 2) * 4;
  }
  // tiles + receive buffer + barriers + the fold warp's (M, 1/L) per query head;
  // the launcher adds up to 1 KB of alignment slack where the SM has room
  __host__ __device__ static size_t bytes(int Hq, int cs) { return tiles + (size_t)recv_floats(cs) * 4 + 128 + (size_t)Hq * 8; }
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Asynchronous stores into a cluster peer's shared memory, completing bytes
// on that peer's mbarrier (visible to it once the barrier phase completes).
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(raddr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, float x, float y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];\n" ::"r"(raddr), "f"(x),
               "f"(y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int G, int MT>
__global__ void __launch_bounds__(ClSmem<G, MT>::THREADS, 1) decode_tc_cluster_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                                         const AttnArgs a, const LayerSteps ls) {
  using namespace tcd;
  using Sm = ClSmem<G, MT>;
  constexpr int NWC = Sm::NWC, CTC = NWC * 32;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align up by offset from the array (keeps the shared state space: LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  const int CS = a.nc;  // cluster size == chunks per segment
  unsigned char* ktiles = smem;
  unsigned char* vtiles = smem + MT * TILE;
  float* recv = reinterpret_cast<float*>(smem + Sm::tiles);  // [recv_floats(CS)]
  uint64_t* bars = reinterpret_cast<uint64_t*>(recv + Sm::recv_floats(CS));
  uint64_t* kfull = bars;
  uint64_t* vfull = bars + 1;
  uint64_t* kfree = bars + 2;  // K rows free: every warp's partial consumed by the chunk combine
  uint64_t* vfree = bars + 3;
  uint64_t* ready = bars + 4;  // own arrive + every rank's pushed bytes, one phase per layer
  uint64_t* mdone = bars + 5;  // (late_prefetch) this rank's merge of the layer is done
  volatile int* relc = reinterpret_cast<volatile int*>(bars + 6);  // layers released to the consumers
  float* fstats = reinterpret_cast<float*>(bars + 16);  // fold warp: [Hq][2]
  {
    uint32_t dyn;  // the tight layout needs the aligned base inside the allocation
    asm("mov.u32 %0, %%dynamic_smem_size;\n" : "=r"(dyn));
    if ((size_t)(smem - smem_raw) + Sm::bytes(a.Hq, CS) > dyn) {
      if (threadIdx.x == 0 && a.err) atomicOr(a.err, 1 << 30);
      return;  // same offset in every CTA of the launch: all leave, no barrier is left waiting
    }
  }

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = (int)cluster_rank();
  const int sigma = blockIdx.x / CS;
  const int n = a.n_old + a.append;
  const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
  const int segs = a.S * a.Hkv;
  const int tt0 = min(j * a.ch, a.nt), tt1 = min(tt0 + a.ch, a.nt);
  const int ntile = tt1 - tt0;
  const int k0 = tt0 * TT;
  const int kend = min(tt1 * TT, n);
  const bool has_new = a.append && a.n_old >= k0 && a.n_old < kend;
  const bool has_prev = a.n_old - 1 >= k0 && a.n_old - 1 < kend;

  if (tid == 0) {
    mbar_init(kfull, 1);
    mbar_init(vfull, 1);
    mbar_init(kfree, NWC);
    mbar_init(vfree, NWC);
    mbar_init(ready, 1);
    mbar_init(mdone, 1);
    *relc = 0;
    mbar_fence_init();
    mbar_arrive_expect_tx(ready, Sm::recv_bytes(CS, j));  // layer 0's pushes
  }
  cluster_sync_all();  // every rank's barriers exist before any remote arrive

  if (warp == NWC) {
    // ---------------------------------------------------------- producer
    // (lane 0 streams the tiles; the whole warp appends the token's row once
    // its layer is released, off the consumers' critical path)
    if (ntile > 0) {
      if (!ls.prefetch0 || has_prev) griddep_wait();
      for (int l = 0; l < ls.L; ++l) {
        const int seg_row = (int)(((int64_t)s * a.L + a.layer + l) * a.Hkv + g) * a.cap;
        // layer l > 0: V as soon as layer l-1's P V is done, K once the chunk
        // combine has consumed the warp partials staged in the K rows
        for (int kv = 0; kv < 2; ++kv) {
          const bool isk = (kv == 0) == (l == 0);
          if (lane == 0) {
            if (l > 0) {
              const bool late = ls.late_prefetch == 1 || (ls.late_prefetch == 2 && isk);
              mbar_wait(late ? mdone : isk ? kfree : vfree, (l - 1) & 1);
            }
            uint64_t* full = isk ? kfull : vfull;
            unsigned char* dst = isk ? ktiles : vtiles;
            const CUtensorMap* map = isk ? &kmap : &vmap;
            mbar_arrive_expect_tx(full, (uint32_t)ntile * TILE);
            for (int t = 0; t < ntile; ++t) {
              const int y = seg_row + (tt0 + t) * TT;
              tma_load_2d(dst + t * TILE, map, 0, y, full);
              tma_load_2d(dst + t * TILE + REGION, map, 64, y, full);
            }
          }
          __syncwarp();
        }
        if (has_new) {  // KvCache.append of layer l's token, after layer l's release
          while (*relc < l + 1) {
          }
          AttnArgs al = a;  // layer l's cache rows and token metadata
          al.kc = static_cast<__nv_bfloat16*>(a.kc) + l * ls.kv_ls;
          al.vc = static_cast<__nv_bfloat16*>(a.vc) + l * ls.kv_ls;
          al.kin = static_cast<const __nv_bfloat16*>(a.kin) + l * ls.in_ls;
          al.vin = static_cast<const __nv_bfloat16*>(a.vin) + l * ls.in_ls;
          al.pos = a.pos + l * ls.m_ls;
          al.modality = a.modality + l * ls.m_ls;
          al.round_id = a.round_id + l * ls.m_ls;
          al.len = a.len + l;
          al.next_pos = a.next_pos + l;
          append_row<__nv_bfloat16, D>(al, sigma, n, lane, 32);
        }
      }
    }
  } else if (warp == NWC + 1) {
    // ------------------------------------------------- window-row fold warp
    if (a.fold.n > 0) {
      griddep_wait();
      const int P = gridDim.x, c = blockIdx.x;
      const int pw = 64 * fold_cols_per_pass(a.Hq);  // (wider pieces for few heads per stream)
      const int ppc = (a.fold.n + pw - 1) / pw;
      for (int l = 0; l < ls.L; ++l) {
        FoldArgs f = a.fold;
        f.logits += l * ls.lg_ls;
        f.stats += l * ls.st_ls;
        f.rows += l * ls.fr_ls;
        if (f.wlen) f.wlen += l * ls.fw_ls;
        for (int piece = c; piece < a.S * ppc; piece += P) {
          const int s2 = piece / ppc, col0 = (piece - s2 * ppc) * pw;
          const float* stt = f.stats + s2 * f.st_ss;
          for (int h = lane; h < a.Hq; h += 32) {
            fstats[2 * h] = __ldg(stt + 2 * h);
            fstats[2 * h + 1] = __frcp_rn(__ldg(stt + 2 * h + 1));  // staged as 1/L
          }
          __syncwarp();
          fold_columns(f, s2, col0, min(col0 + pw, f.n), a.Hq, lane, 32, fstats);
          __syncwarp();
          if (col0 == 0 && lane == 0 && f.wlen) f.wlen[s2 * f.w_ss] = f.n;
        }
      }
    }
  } else if (warp < NWC) {
    // ------------------------------------------------------------ consumers
    const int gid = lane >> 2, tig = lane & 3;
    const bool real = gid < G;
    const uint32_t kbase = smem_u32(ktiles), vbase = smem_u32(vtiles);
    const int wk0 = warp * 32;
    // warp w's partial lives in the 32 K rows it scored: o in the first half of
    // the swizzled tile, (m, l) in the second
    auto wpart = [&](int w) { return reinterpret_cast<float*>(ktiles + (w >> 1) * TILE + (w & 1) * 4096); };
    constexpr int HALF = REGION / 4;  // floats
    for (int l = 0; l < ls.L; ++l) {
      if (l == 0) {
        griddep_wait();
        if (tid == 0) griddep_launch();
      } else {
        // layer l-1 released: four pollers (lane 0 of warps 0-3) staggered by a
        // quarter of an L2 round trip, so some read reaches L2 soon after the
        // last release lands; the first to see it tells the others
        if (lane == 0 && warp < 4) {
          if (warp) __nanosleep(160 * warp);
          while (*relc < l + 1) {
            if (ld_acquire(&ls.layer_done[l - 1]) >= segs * CS) {
              *relc = l + 1;  // (also lets the producer warp append layer l's token)
              break;
            }
          }
        }
        bar_sync_n(1, CTC);
      }
      if (l == 0 && tid == 0) *relc = 1;  // the producer warp may append layer 0's token
      unsigned long long* tl = ls.tl && blockIdx.x < 148 ? ls.tl + ((int64_t)l * 148 + blockIdx.x) * 16 : nullptr;
      // instrumentation: release in %globaltimer ns, later stamps by SM cycles (ns at 1965 MHz)
      const unsigned long long tg0 = tl && tid == 0 ? gtimer() : 0ull;
      const long long tc0 = clock64();
      auto stamp = [&](int i) { tl[i] = i == 0 ? tg0 : tg0 + (unsigned long long)((clock64() - tc0) * 1000 / 1965); };
      if (tl && tid == 0) stamp(0);
      const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(a.q) + l * ls.q_ls;
      uint32_t qa[8][2];
      {
        const uint32_t* qrow =
            reinterpret_cast<const uint32_t*>(q + s * a.q_ss + (int64_t)(g * G + (real ? gid : 0)) * D);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          qa[ks][0] = real ? qrow[8 * ks + tig] : 0u;
          qa[ks][1] = real ? qrow[8 * ks + 4 + tig] : 0u;
        }
      }
      const uint32_t ph = l & 1;
      const bool any = ntile > 0;
      // the token's new k/v row: loaded together with q by the one warp whose
      // 32 keys hold slot n_old (lanes 0-15 k, 16-31 v) and written into its
      // own tile rows -- no other warp reads them, so no CTA barrier
      const int kk_new = a.n_old - k0;
      const bool own_new = has_new && warp == (kk_new >> 5);
      uint4 nrow = make_uint4(0u, 0u, 0u, 0u);
      const uint32_t nrow_off = own_new ? (uint32_t)((kk_new / TT) * TILE) + swz(kk_new % TT, lane & 15) : 0u;
      if (own_new) {
        const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(lane < 16 ? a.kin : a.vin) + l * ls.in_ls;
        nrow = reinterpret_cast<const uint4*>(src + s * a.in_ss + (int64_t)g * D)[lane & 15];
      }
      if (any) mbar_wait(kfull, ph);
      if (tl && tid == 0) stamp(1);
      if (own_new) {
        if (lane < 16) *reinterpret_cast<uint4*>(ktiles + nrow_off) = nrow;
        __syncwarp();
      }
      float m[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
      float o[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float* lg = a.logits ? a.logits + l * ls.lg_ls + s * a.l_ss + (int64_t)(g * G) * a.l_hs : nullptr;
      float p[2][4];
      const bool active = wk0 < ntile * TT;
      if (active) warp_scores(qa, kbase, wk0, lane, k0, kend, a.scale, lg, a.l_hs, G, p, m, lsum);
      if (any) mbar_wait(vfull, ph);
      if (own_new) {
        if (lane >= 16) *reinterpret_cast<uint4*>(vtiles + nrow_off) = nrow;
        // (generic writes into tiles the async proxy refills next layer)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
      }
      if (active) warp_pv(p, vbase, wk0, lane, o);
      __syncwarp();
      if (lane == 0 && any) mbar_arrive(vfree);
      if (tl && tid == 0) stamp(2);
      {  // into this warp's own K rows (every lane's ldmatrix reads are done)
        float* wp = wpart(warp);
        warp_stage(o, m, lsum, lane, G, wp, wp + HALF, wp + HALF + G);
      }
      bar_sync_n(1, CTC);
      if (tl && tid == 0) stamp(5);  // every warp's partial staged
      if (tl && tid == 0) stamp(8);  // (append done)
      const int per = Sm::per(CS);
      float* rv = recv;
      const uint32_t rv_local = smem_u32(rv), rbar_local = smem_u32(ready);
      // warp weights rescale(m_w, M) once per (warp, head), next to the warp's
      // (m, l); the head maxima next to warp 0's
      if (tid < NWC * G) {
        const int w = tid / G, h = tid - (tid / G) * G;
        float M = -INFINITY;
#pragma unroll
        for (int w2 = 0; w2 < NWC; ++w2) M = fmaxf(M, wpart(w2)[HALF + h]);
        wpart(w)[HALF + 2 * G + h] = rescale(wpart(w)[HALF + h], M);
        if (w == 0) wpart(0)[HALF + 3 * G + h] = M;
      }
      bar_sync_n(1, CTC);
      static_assert(G * D / 4 <= 2 * MT * 32, "one 4-element group per consumer thread");
      if (tid < G * D / 4) {
        const int idx = tid * 4, h = idx / D, d = idx - h * D;
        const float M = wpart(0)[HALF + 3 * G + h];
        float f[NWC];
#pragma unroll
        for (int w = 0; w < NWC; ++w) f[w] = wpart(w)[HALF + 2 * G + h];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < NWC; ++w) {
          const float4 o4 = *reinterpret_cast<const float4*>(wpart(w) + h * D + d);
          acc.x = fmaf(f[w], o4.x, acc.x);
          acc.y = fmaf(f[w], o4.y, acc.y);
          acc.z = fmaf(f[w], o4.z, acc.z);
          acc.w = fmaf(f[w], o4.w, acc.w);
        }
        const int owner = idx / per, e = idx - owner * per;
        st_async_v4(map_rank(rv_local + (j * per + e) * 4, owner), acc, map_rank(rbar_local, owner));
        // (every lane of this warp works on head h: G*D/4 groups fit the consumer
        // threads, 32 groups per head) -- lane r sends (M, L) to rank r
        float xs = 0.f;  // warps in order (NWC need not be a power of two)
#pragma unroll
        for (int w = 0; w < NWC; ++w) xs += f[w] * wpart(w)[HALF + G + h];
        if (lane < CS) {
          const uint32_t so = rv_local + (CS * per + (j * G + h) * 2) * 4;
          st_async_v2(map_rank(so, lane), M, xs, map_rank(rbar_local, lane));
        }
      }
      if (tl && tid == 0) stamp(9);  // (combine + pushes issued)
      __syncwarp();
      if (lane == 0 && any) mbar_arrive(kfree);  // this warp's reads of the staged partials are done
      if (tl && tid == 0) stamp(3);
      wait_cluster(ready, l & 1);
      if (tl && tid == 0) stamp(6);  // every rank's partial received
      // ---- merge this rank's elements from local shared memory (merge_kernel's
      // arithmetic: weights rescale(m_r, M), L = sum w_r l_r, out = sum_r w_r o_r / L)
      float* out = a.out + l * ls.o_ls + s * a.o_ss + (int64_t)(g * G) * D;
      float* stats = a.stats + l * ls.st_ls;
      const int cnt = min(per, G * D - j * per);
      float* mw = rv + CS * per + 2 * G * CS;  // [CS][G] chunk weights, [G] maxima
      if (tid < CS * G) {
        const int r = tid / G, h = tid - (tid / G) * G;
        const float* sm = rv + CS * per + h * 2;
        float M = -INFINITY;
        for (int r2 = 0; r2 < CS; ++r2) M = fmaxf(M, sm[r2 * G * 2]);
        mw[r * G + h] = rescale(sm[r * G * 2], M);
        if (r == 0) mw[CS * G + h] = M;
      }
      bar_sync_n(1, CTC);
      for (int e4 = tid * 4; e4 < cnt; e4 += CTC * 4) {
        const int idx = j * per + e4, h = idx / D;
        const float* sm = rv + CS * per + h * 2;  // [src][G][2]
        const float M = mw[CS * G + h];
        float L = 0.f;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < CS; ++r) {
          const float w = mw[r * G + h];
          L += w * sm[r * G * 2 + 1];
          const float4 o4 = *reinterpret_cast<const float4*>(rv + r * per + e4);
          acc.x = fmaf(w, o4.x, acc.x);
          acc.y = fmaf(w, o4.y, acc.y);
          acc.z = fmaf(w, o4.z, acc.z);
          acc.w = fmaf(w, o4.w, acc.w);
        }
        *reinterpret_cast<float4*>(out + idx) = make_float4(acc.x / L, acc.y / L, acc.z / L, acc.w / L);
        if (idx - h * D == 0) {
          stats[s * a.st_ss + (g * G + h) * 2] = M;
          stats[s * a.st_ss + (g * G + h) * 2 + 1] = L;
        }
      }
      if (tl && tid == 0) stamp(7);  // thread 0's elements merged
      // layer l+1's expected bytes (its pushes follow every rank's release of
      // layer_done[l], hence this rank's merge above: one buffer suffices)
      if (tid == 0) mbar_arrive_expect_tx(ready, Sm::recv_bytes(CS, j));
      bar_sync_n(1, CTC);
      if (tid == 0 && any) mbar_arrive(mdone);
      if (tid == 0) {
        red_release_add(&ls.layer_done[l], 1);
        if (tl) stamp(4);
      }
    }
    if (tid == 0) {
      if (atomicAdd(ls.exit_count, 1) == (int)gridDim.x - 1) {
        for (int l = 0; l < ls.L; ++l) ls.layer_done[l] = 0;
        *ls.exit_count = 0;
      }
    }
  }
  // no rank leaves while a push into it may be in flight (every rank has
  // received all its bytes before it arrives: no memory ordering needed)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// Throughput launches (many segments: dynamic chunk tickets) on the tensor
// cores.  decode_kernel's schedule -- ticket producer with a 3-stage ring, the
// epilogue warp merging each chunk's warp partials in the background, the fold
// warp, merge_kernel after it -- with 2-D TMA tiles in the 128-byte swizzle and
// the keys-as-M MMA math: 4 consumer warps take 16 keys of every 64-token tile
// and keep a running (max, sum, O^T) per query head over the chunk.  The
// segment's new token is appended to the cache by the producer warp before
// the tile that holds it streams in (a proxy fence orders the row stores
// before the tensor copy), so the tile arrives complete.
namespace tcd {
template <int G>
struct DynSmem {
  static constexpr int NWD = 4;                  // consumer warps
  static constexpr int THREADS = NWD * 32 + 96;  // + producer, epilogue, fold warps
  static constexpr int STAGES = 3;
  static constexpr size_t tiles = (size_t)STAGES * 2 * TILE;
  static constexpr size_t slot_floats = 4 + 2 * NWD * G + NWD * G * D;
  static size_t bytes(int Hq) {
    return tiles + 2 * slot_floats * 4 + (2 * STAGES + 4) * 8 + (2 * STAGES + 4) * 4 + (size_t)Hq * 8 + 1024;
  }
};

// One warp's 16 keys [wk0, wk0 + 16) of a tile whose row 0 is cache index
// key0: S^T = K Q^T, then the running softmax (m, l, O^T rescaled by
// exp(m_old - m_new)) and O^T += V^T P^T; recorded steps store the logits.
__device__ __forceinline__ void warp_tile16(const uint32_t (&qb)[8][2], uint32_t kbase, uint32_t vbase, int wk0,
                                            int lane, int key0, int kend, float scale, float* lg, int64_t lg_hs,
                                            int G, float (&m)[2], float (&l)[2], float (&o)[8][4]) {
  const int gid = lane >> 2, tig = lane & 3;
  float sacc[4] = {0.f, 0.f, 0.f, 0.f};
  {
    const int kk = wk0 + (lane & 7) + 8 * ((lane >> 3) & 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(kbase + swz(kk, 2 * ks + (lane >> 4)), a0, a1, a2, a3);
      mma16816_a4(sacc, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
    }
  }
  float x[4], mx[2];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int key = key0 + wk0 + gid + (c >> 1) * 8;
    x[c] = key < kend ? sacc[c] * scale : -INFINITY;
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    mx[e] = fmaxf(x[e], x[2 + e]);
#pragma unroll
    for (int sh = 4; sh < 32; sh <<= 1) mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], sh));
  }
  float mn[2], alpha[2], p[4], ls[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    mn[e] = fmaxf(m[e], mx[e]);
    alpha[e] = rescale(m[e], mn[e]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) p[c] = mn[c & 1] == -INFINITY ? 0.f : fast_exp2((x[c] - mn[c & 1]) * kLog2e);
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    ls[e] = p[e] + p[2 + e];
#pragma unroll
    for (int sh = 4; sh < 32; sh <<= 1) ls[e] += __shfl_xor_sync(0xffffffffu, ls[e], sh);
    l[e] = l[e] * alpha[e] + ls[e];
    m[e] = mn[e];
  }
#pragma unroll
  for (int md = 0; md < 8; ++md)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[md][c] *= alpha[c & 1];
  if (lg) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * tig + e;
      if (h >= G) continue;
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        const int key = key0 + wk0 + gid + 8 * hi;
        if (key < kend) lg[h * lg_hs + key] = x[2 * hi + e];
      }
    }
  }
  const uint32_t h0 = pack_bf16(p[0], p[1]), h1 = pack_bf16(p[2], p[3]);
  const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h0));
  const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h1));
  const uint32_t l0 = pack_bf16(p[0] - f0.x, p[1] - f0.y), l1 = pack_bf16(p[2] - f1.x, p[3] - f1.y);
  const uint32_t bh0 = movtrans(h0), bh1 = movtrans(h1), bl0 = movtrans(l0), bl1 = movtrans(l1);
  const int kk = wk0 + (lane & 7) + 8 * (lane >> 4);
#pragma unroll
  for (int md = 0; md < 8; ++md) {
    uint32_t a0, a1, a2, a3;
    ldsm_x4_t(vbase + swz(kk, 2 * md + ((lane >> 3) & 1)), a0, a1, a2, a3);
    mma16816_a4(o[md], a0, a1, a2, a3, bh0, bh1);
    mma16816_a4(o[md], a0, a1, a2, a3, bl0, bl1);
  }
}
}  // namespace tcd

template <int G>
__global__ void __launch_bounds__(tcd::DynSmem<G>::THREADS, 2)
    decode_tcd_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                      const AttnArgs a) {
  using namespace tcd;
  using Sm = DynSmem<G>;
  constexpr int NWD = Sm::NWD, CTD = NWD * 32, STAGES = Sm::STAGES, SLOT = (int)Sm::slot_floats;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  unsigned char* tiles = smem;                                        // [STAGES][K tile, V tile]
  float* slots = reinterpret_cast<float*>(smem + Sm::tiles);          // [2][SLOT]
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + 2 * SLOT);
  uint64_t* empty = full + STAGES;
  uint64_t* epi_full = empty + STAGES;  // [2]
  uint64_t* epi_empty = epi_full + 2;   // [2]
  int* tinfo = reinterpret_cast<int*>(epi_empty + 2);  // [STAGES][2]
  int* cring = tinfo + 2 * STAGES;                     // [4] next chunk tickets
  float* fstats = reinterpret_cast<float*>(cring + 4);  // [Hq][2]

  const int c = blockIdx.x, P = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_old + a.append;
  const int total = a.S * a.Hkv * a.nc;
  constexpr int PWD = D + 2;

  if (a.tstamp && tid == 0) atomicMin(&a.tstamp[0], gtimer());
  if (c == 0 && tid == 0 && a.done_self) {  // a stale flag from this slot's previous use must not leak
    *a.done_self = 0;
    __threadfence();
  }
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NWD);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&epi_full[i], NWD);
      mbar_init(&epi_empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto wait_prev = [&]() {
    if (a.done_prev) {
      while (ld_acquire(a.done_prev) == 0) __nanosleep(32);
    } else {
      griddep_wait();
    }
  };

  if (warp == NWD) {
    // ------------------------------------------------------------ producer
    bool waited = false;
    if (!a.prefetch) {
      griddep_wait();
      waited = true;
    }
    const int nce = a.nc - 1, segs = a.S * a.Hkv, early = segs * nce;
    const int DL = a.late > 0 && a.late < segs && nce > 0 ? a.late : 0;
    auto slot_of = [&](int t) {  // ticket -> chunk slot (decode_kernel's order)
      if (t >= total) return t;
      if (DL == 0) return t < early ? (t / nce) * a.nc + (t % nce) : (t - early) * a.nc + nce;
      const int bD = DL * nce;
      const int bEnd = segs * nce + (segs - DL);
      if (t >= bEnd) return (segs - DL + (t - bEnd)) * a.nc + nce;
      int sg, off;
      if (t < bD) {
        sg = t / nce;
        off = t - sg * nce;
      } else {
        sg = DL + (t - bD) / (nce + 1);
        off = (t - bD) - (sg - DL) * (nce + 1);
      }
      return off < nce ? sg * a.nc + off : (sg - DL) * a.nc + nce;
    };
    int u = 0, t1 = 0, t2 = 0;
    if (lane == 0) {
      u = slot_of(atomicAdd(&a.sched[0], 1));
      t1 = atomicAdd(&a.sched[0], 1);
      t2 = atomicAdd(&a.sched[0], 1);
    }
    u = __shfl_sync(0xffffffffu, u, 0);
    int i = 0, kp = 0;
    while (u < total) {
      int u_next = 0;
      if (lane == 0) {
        u_next = slot_of(t1);
        t1 = t2;
        t2 = atomicAdd(&a.sched[0], 1);
        cring[(kp + 1) & 3] = u_next < total ? u_next : -1;  // lets the consumers prefetch q
      }
      u_next = __shfl_sync(0xffffffffu, u_next, 0);
      ++kp;
      const int sigma = u / a.nc, j = u - sigma * a.nc;
      const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
      const int tt0 = j * a.ch, tt1 = min(tt0 + a.ch, a.nt);
      const int seg_row = (int)((((int64_t)s * a.L + a.layer) * a.Hkv + g) * a.cap);
      for (int tt = tt0; tt < tt1; ++tt, ++i) {
        const int ts = tt * TT;
        const int st = i % STAGES;
        if (a.append && a.n_old >= ts && a.n_old < ts + TT) {
          // KvCache.append (the whole warp), then the tile holding the row
          if (!waited) {
            wait_prev();
            waited = true;
          }
          append_row<__nv_bfloat16, D>(a, sigma, n, lane, 32);
          asm volatile("fence.proxy.async.global;\n" ::: "memory");
          __syncwarp();
        }
        if (lane == 0) {
          mbar_wait(&empty[st], ((i / STAGES) & 1) ^ 1);
          tinfo[2 * st] = u;
          tinfo[2 * st + 1] = tt | ((tt == tt1 - 1) ? (1 << 30) : 0);
          unsigned char* ks = tiles + (size_t)(2 * st) * TILE;
          mbar_arrive_expect_tx(&full[st], 2u * TILE);
          const int y = seg_row + ts;
          tma_load_2d(ks, &kmap, 0, y, &full[st]);
          tma_load_2d(ks + REGION, &kmap, 64, y, &full[st]);
          tma_load_2d(ks + TILE, &vmap, 0, y, &full[st]);
          tma_load_2d(ks + TILE + REGION, &vmap, 64, y, &full[st]);
        }
        __syncwarp();
      }
      u = u_next;
    }
    if (lane == 0) {  // end marker
      const int st = i % STAGES;
      mbar_wait(&empty[st], ((i / STAGES) & 1) ^ 1);
      tinfo[2 * st] = -1;
      mbar_arrive(&full[st]);
    }
    return;
  }

  if (warp == NWD + 2) {
    // ------------------------------------------------- window-row fold warp
    const FoldArgs& f = a.fold;
    if (f.n <= 0) return;
    if (!a.prefetch) griddep_wait();
    const int ppc = (f.n + 63) / 64;
    for (int piece = c; piece < a.S * ppc; piece += P) {
      const int s = piece / ppc, col0 = (piece - s * ppc) * 64;
      const float* stt = f.stats + s * f.st_ss;
      for (int h = lane; h < a.Hq; h += 32) {
        fstats[2 * h] = __ldg(stt + 2 * h);
        fstats[2 * h + 1] = __frcp_rn(__ldg(stt + 2 * h + 1));  // staged as 1/L
      }
      __syncwarp();
      fold_columns(f, s, col0, min(col0 + 64, f.n), a.Hq, lane, 32, fstats);
      __syncwarp();
      if (col0 == 0 && lane == 0 && f.wlen) f.wlen[s * f.w_ss] = f.n;
    }
    return;
  }

  if (warp == NWD + 1) {
    // ------------------------------------------------------ epilogue warp
    for (int k = 0;; ++k) {
      const int sl = k & 1;
      mbar_wait(&epi_full[sl], (k >> 1) & 1);
      const float* slot = slots + sl * SLOT;
      const int u = reinterpret_cast<const int*>(slot)[0];
      if (u < 0) break;
      const float* wm = slot + 4;
      const float* wl = wm + NWD * G;
      const float* wo = wl + NWD * G;
      const int sigma = u / a.nc, j = u - sigma * a.nc;
      float* part = a.part + ((int64_t)sigma * a.nc + j) * G * PWD;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float mw = lane < NWD ? wm[lane * G + h] : -INFINITY;
        float M = mw;
#pragma unroll
        for (int off = NWD / 2; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        const float f = lane < NWD ? rescale(mw, M) : 0.f;
        float L = lane < NWD ? f * wl[lane * G + h] : 0.f;
#pragma unroll
        for (int off = NWD / 2; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
        float fw[NWD];
#pragma unroll
        for (int w = 0; w < NWD; ++w) fw[w] = __shfl_sync(0xffffffffu, f, w);
#pragma unroll
        for (int d = lane; d < D; d += 32) {
          float acc = 0.f;
#pragma unroll
          for (int w = 0; w < NWD; ++w) acc = fmaf(fw[w], wo[(w * G + h) * D + d], acc);
          part[h * PWD + d] = acc;
        }
        if (lane == 0) {
          part[h * PWD + D] = M;
          part[h * PWD + D + 1] = L;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&epi_empty[sl]);
      __syncwarp();
      if (lane == 0) red_release_add(&a.counters[sigma], 1);  // the segment's merge counts it
    }
    __threadfence();
    bar_sync_n(2, CTD + 32);
    return;
  }

  // -------------------------------------------------------------- consumers
  if (a.done_prev) {
    if (tid == 0) wait_prev();
    bar_sync_n(1, CTD);
  } else {
    griddep_wait();
  }
  if (tid == 0) griddep_launch();
  const int gid = lane >> 2, tig = lane & 3;
  const bool real = gid < G;
  const int wk0 = warp * 16;
  uint32_t qb[8][2], qn[8][2];
  int qn_sigma = -1, cur = -1;
  auto load_q = [&](uint32_t (&dst)[8][2], int sg) {
    const int s2 = sg / a.Hkv, g2 = sg - s2 * a.Hkv;
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(static_cast<const __nv_bfloat16*>(a.q) + s2 * a.q_ss +
                                                             (int64_t)(g2 * G + (real ? gid : 0)) * D);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      dst[ks][0] = real ? qrow[8 * ks + tig] : 0u;
      dst[ks][1] = real ? qrow[8 * ks + 4 + tig] : 0u;
    }
  };
  float m[2], l[2], o[8][4];
  float* lg = nullptr;
  int k = 0;
  bool fresh = true;
  for (int i = 0;; ++i) {
    const int st = i % STAGES;
    mbar_wait(&full[st], (i / STAGES) & 1);
    const int u = tinfo[2 * st];
    if (u < 0) break;
    const int info = tinfo[2 * st + 1];
    const int tt = info & 0xffff;
    const bool chunk_end = (info >> 30) & 1;
    const int sigma = u / a.nc;
    if (fresh) {
      if (sigma != cur) {
        if (qn_sigma != sigma) load_q(qn, sigma);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          qb[ks][0] = qn[ks][0];
          qb[ks][1] = qn[ks][1];
        }
        cur = sigma;
        const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
        lg = a.logits ? a.logits + s * a.l_ss + (int64_t)(g * G) * a.l_hs : nullptr;
      }
      const int un = a.qpf ? cring[(k + 1) & 3] : -1;
      if (un >= 0 && un / a.nc != sigma) {
        load_q(qn, un / a.nc);
        qn_sigma = un / a.nc;
      }
      m[0] = m[1] = -INFINITY;
      l[0] = l[1] = 0.f;
#pragma unroll
      for (int md = 0; md < 8; ++md) o[md][0] = o[md][1] = o[md][2] = o[md][3] = 0.f;
      fresh = false;
    }
    const uint32_t kbase = smem_u32(tiles + (size_t)(2 * st) * TILE);
    warp_tile16(qb, kbase, kbase + TILE, wk0, lane, tt * TT, n, a.scale, lg, a.l_hs, G, m, l, o);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (!chunk_end) continue;
    // ---- chunk done: hand the warp partials to the epilogue warp
    const int sl = k & 1;
    mbar_wait(&epi_empty[sl], ((k >> 1) & 1) ^ 1);
    float* slot = slots + sl * SLOT;
    float* wm = slot + 4;
    float* wl = wm + NWD * G;
    float* wo = wl + NWD * G;
    warp_stage(o, m, l, lane, G, wo + warp * G * D, wm + warp * G, wl + warp * G);
    if (warp == 0 && lane == 0) reinterpret_cast<int*>(slot)[0] = u;
    __syncwarp();
    if (lane == 0) mbar_arrive(&epi_full[sl]);
    ++k;
    fresh = true;
  }
  {  // end marker for the epilogue warp
    const int sl = k & 1;
    mbar_wait(&epi_empty[sl], ((k >> 1) & 1) ^ 1);
    if (warp == 0 && lane == 0) reinterpret_cast<int*>(slots + sl * SLOT)[0] = -1;
    __syncwarp();
    if (lane == 0) mbar_arrive(&epi_full[sl]);
  }
  bar_sync_n(2, CTD + 32);  // this CTA's epilogue warp has published its partials
  if (a.tstamp && tid == 0) atomicMax(&a.tstamp[1], gtimer());
  if (tid == 0) {
    if (atomicAdd(&a.sched[2], 1) == P - 1) {  // the last CTA out resets the scheduler
      a.sched[0] = 0;
      a.sched[2] = 0;
      if (a.done_prev) *const_cast<int32_t*>(a.done_prev) = 0;
    }
  }
}


// Tensor maps over the K/V stores, encoded once per store (base, rows).
static cudaError_t kv_maps(const AttnArgs& a, const CUtensorMap** km, const CUtensorMap** vm) {
  struct MapCache {
    const void* kb = nullptr;
    const void* vb = nullptr;
    int64_t rows = 0;
    CUtensorMap k, v;
  };
  static thread_local MapCache cache[4];
  static thread_local int next = 0;
  for (auto& e : cache)
    if (e.kb == a.kc_base && e.vb == a.vc_base && e.rows == a.total_rows) {
      *km = &e.k;
      *vm = &e.v;
      return cudaSuccess;
    }
  MapCache* m = &cache[next++ % 4];
  cudaError_t e = make_kv_map(&m->k, a.kc_base, a.total_rows, tcd::TT);
  if (e == cudaSuccess) e = make_kv_map(&m->v, a.vc_base, a.total_rows, tcd::TT);
  if (e != cudaSuccess) {
    m->kb = nullptr;
    return e;
  }
  m->kb = a.kc_base;
  m->vb = a.vc_base;
  m->rows = a.total_rows;
  *km = &m->k;
  *vm = &m->v;
  return cudaSuccess;
}

cudaError_t launch_decode_tcd(int group, int ctas, const AttnArgs& a, cudaStream_t st) {
  if (a.stat) return cudaErrorInvalidValue;
  const CUtensorMap *km = nullptr, *vm = nullptr;
  cudaError_t e = kv_maps(a, &km, &vm);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  static DevOnce attr_set[9];
  auto run = [&](auto kern, int threads, size_t bytes) -> cudaError_t {
    DevOnce& attr = attr_set[group];
    if (!attr.here()) {
      // (two CTAs per SM where the slots are small -- groups 1, 2; one otherwise)
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (r != cudaSuccess) return r;
      attr.here() = true;
    }
    if (bytes > 227 * 1024) return cudaErrorInvalidValue;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = bytes;
    return cudaLaunchKernelEx(&cfg, kern, *km, *vm, a);
  };
  e = cudaErrorInvalidValue;
  if (group == 1) e = run(decode_tcd_kernel<1>, tcd::DynSmem<1>::THREADS, tcd::DynSmem<1>::bytes(a.Hq));
  if (group == 2) e = run(decode_tcd_kernel<2>, tcd::DynSmem<2>::THREADS, tcd::DynSmem<2>::bytes(a.Hq));
  if (group == 4) e = run(decode_tcd_kernel<4>, tcd::DynSmem<4>::THREADS, tcd::DynSmem<4>::bytes(a.Hq));
  if (group == 8) e = run(decode_tcd_kernel<8>, tcd::DynSmem<8>::THREADS, tcd::DynSmem<8>::bytes(a.Hq));
  if (e != cudaSuccess) return e;
  return launch_merge(128, group, a, st);
}

cudaError_t launch_decode_tc(int group, int ctas, const AttnArgs& a, cudaStream_t st) {
  if (a.ch > tcd::MAXT || !a.stat) return cudaErrorInvalidValue;
  // tensor maps depend only on the store (base, rows): encode once per store
  // (host-side encoding costs microseconds per launch on batch-1 steps)
  struct MapCache {
    const void* kb = nullptr;
    const void* vb = nullptr;
    int64_t rows = 0;
    CUtensorMap k, v;
  };
  static thread_local MapCache cache[4];
  static thread_local int next = 0;
  MapCache* m = nullptr;
  for (auto& e : cache)
    if (e.kb == a.kc_base && e.vb == a.vc_base && e.rows == a.total_rows) m = &e;
  cudaError_t e = cudaSuccess;
  if (!m) {
    m = &cache[next++ % 4];
    e = make_kv_map(&m->k, a.kc_base, a.total_rows, tcd::TT);
    if (e == cudaSuccess) e = make_kv_map(&m->v, a.vc_base, a.total_rows, tcd::TT);
    if (e != cudaSuccess) {
      m->kb = nullptr;
      return e;
    }
    m->kb = a.kc_base;
    m->vb = a.vc_base;
    m->rows = a.total_rows;
  }
  const CUtensorMap& kmap = m->k;
  const CUtensorMap& vmap = m->v;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  static DevOnce attr_set[9][5];
  auto run = [&](auto kern, int threads, size_t smem_bytes, DevOnce& attr) -> cudaError_t {
    if (!attr.here()) {
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (r != cudaSuccess) return r;
      attr.here() = true;
    }
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem_bytes;
    return cudaLaunchKernelEx(&cfg, kern, kmap, vmap, a);
  };
  const int mt = a.ch <= 2 && group <= 4 ? 2 : 4;  // (no 2-tile instantiation for groups of 8)
#define SKV_TC_CASE(GG, MM)                                                                                  \
  if (group == GG && mt == MM)                                                                              \
    e = run(decode_tc_kernel<GG, MM>, tcd::SmemT<GG, MM>::THREADS, tcd::SmemT<GG, MM>::bytes(MM == 4 ? 1024 : a.Hq), \
            attr_set[GG][MM]);
  e = cudaErrorInvalidValue;
  SKV_TC_CASE(1, 2)
  SKV_TC_CASE(2, 2)
  SKV_TC_CASE(4, 2)
  SKV_TC_CASE(4, 4)
  SKV_TC_CASE(8, 4)
#undef SKV_TC_CASE
  if (e != cudaSuccess) return e;
  return launch_merge(128, group, a, st);
}

cudaError_t launch_decode_tc_layers(int group, int ctas, const AttnArgs& a, const LayerSteps& ls, cudaStream_t st) {
  if (a.ch > tcd::MAXT || !a.stat || a.nc > 128) return cudaErrorInvalidValue;
  CUtensorMap kmap, vmap;
  cudaError_t e = make_kv_map(&kmap, a.kc_base, a.total_rows, tcd::TT);
  if (e == cudaSuccess) e = make_kv_map(&vmap, a.vc_base, a.total_rows, tcd::TT);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(tcd::THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (group == 4) {
    static DevOnce attr;
    if (!attr.here()) {
      e = cudaFuncSetAttribute(decode_tc_layers_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tcd::Smem<4>::bytes);
      if (e != cudaSuccess) return e;
      attr.here() = true;
    }
    cfg.dynamicSmemBytes = tcd::Smem<4>::bytes;
    return cudaLaunchKernelEx(&cfg, decode_tc_layers_kernel<4>, kmap, vmap, a, ls);
  }
  if (group == 8) {
    static DevOnce attr;
    if (!attr.here()) {
      e = cudaFuncSetAttribute(decode_tc_layers_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tcd::Smem<8>::bytes);
      if (e != cudaSuccess) return e;
      attr.here() = true;
    }
    cfg.dynamicSmemBytes = tcd::Smem<8>::bytes;
    return cudaLaunchKernelEx(&cfg, decode_tc_layers_kernel<8>, kmap, vmap, a, ls);
  }
  return cudaErrorInvalidValue;
}

// Cluster variant: one cluster of a.nc CTAs per segment (a.nc <= 16).
cudaError_t launch_decode_tc_cluster(int group, int mt, const AttnArgs& a, const LayerSteps& ls, cudaStream_t st,
                                     int* max_clusters) {
  CUtensorMap kmap, vmap;
  cudaError_t e = make_kv_map(&kmap, a.kc_base, a.total_rows, tcd::TT);
  if (e == cudaSuccess) e = make_kv_map(&vmap, a.vc_base, a.total_rows, tcd::TT);
  if (e != cudaSuccess) return e;
  const int segs = a.S * a.Hkv;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(segs * a.nc);
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = a.nc;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  static DevOnce attrs_set[2][8];  // per instantiation (G, mt): kern has one type for all of them
  constexpr size_t kMaxSmem = 227 * 1024;
  auto run = [&](auto kern, int threads, size_t need) -> cudaError_t {
    DevOnce& attr = attrs_set[group == 8][mt & 7];
    if (!attr.here()) {
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
      if (r == cudaSuccess) r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (r != cudaSuccess) return r;
      attr.here() = true;
    }
    if (need > kMaxSmem) return cudaErrorInvalidValue;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = std::min(need + 1024, kMaxSmem);  // + alignment slack where it fits (checked in-kernel)
    if (max_clusters) {  // co-residency check only
      cudaLaunchConfig_t q = cfg;
      q.numAttrs = 2;
      return cudaOccupancyMaxActiveClusters(max_clusters, kern, &q);
    }
    return cudaLaunchKernelEx(&cfg, kern, kmap, vmap, a, ls);
  };
#define SKV_CL_CASE(GG, MM)       \
  if (group == GG && mt == MM) \
    return run(decode_tc_cluster_kernel<GG, MM>, ClSmem<GG, MM>::THREADS, ClSmem<GG, MM>::bytes(a.Hq, a.nc));
  SKV_CL_CASE(4, 4)
  SKV_CL_CASE(4, 5)
  SKV_CL_CASE(4, 6)
  SKV_CL_CASE(4, 7)
  SKV_CL_CASE(8, 4)
  SKV_CL_CASE(8, 5)
  SKV_CL_CASE(8, 6)
#undef SKV_CL_CASE
  return cudaErrorInvalidValue;
}

}  // namespace skv
