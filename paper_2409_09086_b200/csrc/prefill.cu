// K4: chunked prefill attention on the 5th-generation tensor cores (sm_100a).
//
// The reference processes the prompt of a round token by token through
// Session.decode_step (engine.py:350-353): token i of a C-token chunk appends
// its k/v and attends to the cached prefix (n0 tokens) plus chunk tokens 0..i.
// A causal chunk attention is the same computation for all C tokens at once;
// the last W query rows additionally produce the window rows
// (AttentionWindow.push, policies.py:107-115) -- their f32 logits and per-row
// (max, sum) are recorded here and folded into head-mean rows afterwards.
//
// One CTA = two 128-query tiles of one head ("ping-pong"): while the softmax
// warpgroup of one tile turns its S tile into P, the tensor core runs the
// other tile's MMAs.  Warp 8 (TMA producer) loads both Q tiles once and
// 128-key K and V tiles into 2- and 3-stage rings, K one tile ahead of V
// (cp.async.bulk.tensor, 128-byte swizzle).  Warps 10-11 convert each landed V tile in place from bf16 to
// fp16 (exact for |v| < 65504; larger values saturate and are counted).
// Warp 9 owns TMEM and issues tcgen05.mma: S_i = Q_i K^T (bf16, M=N=128)
// into a 128-column TMEM tile, O_i += P_i V (fp16, M=N=128) with P read
// straight from TMEM (the .kind::f16 A-from-TMEM form).  fp16 P carries
// 2^-11 relative rounding (bf16 P would carry 2^-8, above the 2e-3 bf16
// tolerance for diffuse rows) at one MMA per 16 keys.  Warps 0-7 take the two
// Q tiles in turn, two threads per query row: warp w reads the 64 S columns
// [64 (w >> 2), +64) of TMEM lanes 32 (w & 3), the halves' row maxima meet in
// shared memory, and each runs the online softmax on its half (exponentials
// on the SFU; exp2_poly2 can take a share on the FMA pipe, SKV_PF_POLY) and
// writes its half of P (fp16) back over the first 64 S columns.  O is
// rescaled lazily: only when a row maximum grows by more than 2^8 (exact --
// O and the row sum share the stale maximum).
//
// Order on the tensor core: S_0(0) S_1(0) | P_0V(0) S_0(1) P_1V(0) S_1(1) |
// ...  S_i(j+1) overwrites the columns P_i(j) V reads; tcgen05.mma from one
// thread executes in issue order, which CUTLASS's SM100 FMHA relies on too.
//
// TMEM columns: S/P of tile 0 [0,128), S/P of tile 1 [128,256), O of tile 0
// [256,384), O of tile 1 [384,512).
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "skv_common.cuh"
#include "skv_internal.h"
#include "skv_fold.cuh"

namespace skv {
namespace pf {

constexpr int BM = 128;                  // queries per Q tile
constexpr int BN = 128;                  // keys per K/V tile
constexpr int HD = 128;                  // head dim
constexpr int QT = 2;                    // Q tiles per CTA
#ifndef KST_V
#define KST_V 2
#endif
#ifndef VST_V
#define VST_V 3
#endif
constexpr int KST = KST_V;                 // K ring depth (S(j+1) runs a step ahead of P(j) V(j))
constexpr int STAGES = VST_V;              // V ring depth
constexpr int REGION = 128 * 64 * 2;     // [128 rows][64 16-bit] swizzled region, 16 KB
constexpr int TILE = 2 * REGION;         // one Q, K or V tile (128 rows x 128 dims), 32 KB
constexpr int SQ = 0;
constexpr int SK = SQ + QT * TILE;
constexpr int SV = SK + KST * TILE;
constexpr int SBAR = SV + STAGES * TILE;
constexpr int SXCH = SBAR + 256;               // [2 halves][128 rows] row-max exchange (softmax)
constexpr int SMEM_BYTES = SXCH + 1024 + 1024;  // barriers, exchange, alignment slack
#ifndef NCONV_V
#define NCONV_V 2
#endif
constexpr int NCONV = NCONV_V;                       // V-conversion warps
constexpr int THREADS = (8 + 2 + NCONV) * 32;
constexpr float kRescaleLog2 = 8.f;            // lazy O rescale threshold (log2 units)
constexpr int kDefaultPoly = 0;                // exp2 pairs (of 8) on the FMA-pipe polynomial (0-4;
                                               // 2 paid off with one thread per row, not with two)

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // SM100 UMMA shared-memory descriptor, 128-byte swizzle (layout type 2), version 1
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: (bf16 x bf16 or fp16 x fp16) -> f32,
// M = 128, N = n; B K-major (K tile of S = Q K^T) or MN-major (V of O += P V).
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn_major, bool f16) {
  return (1u << 4) | (f16 ? 0u : (1u << 7) | (1u << 10)) | (b_mn_major ? (1u << 16) : 0u) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// D[tmem] (+)= A[smem] . B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]  (A: 128 lanes x 16 bf16 packed in 8 columns)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  tc_wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld without the trailing wait (issue several, then tc_wait_ld once)
__device__ __forceinline__ void tmem_ld32_async(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
}

__device__ __forceinline__ void tmem_st32u(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t addr, const float (&v)[32]) {
  uint32_t u[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(v[i]);
  tmem_st32u(addr, u);
}


}  // namespace pf

// Instrumentation (a.prof != null): cycles spent in each wait, per CTA.
#define PF_WAIT(slot, bar, par)                                     \
  do {                                                              \
    if (prof) {                                                     \
      const long long t0_ = clock64();                              \
      mbar_wait(bar, par);                                          \
      pacc##slot += clock64() - t0_;                                \
    } else {                                                        \
      mbar_wait(bar, par);                                          \
    }                                                               \
  } while (0)

namespace pf {
// 2^t for two lanes on the FMA pipe instead of the SFU (MUFU.EX2 issues at
// 16 lanes/clk/SM, the softmax's bound): t = j + f by the 1.5*2^23
// round-to-nearest shifter, f in [-0.5, 0.5], 2^f by a degree-3 minimax
// polynomial (relative error 8.3e-5, below fp16 P's 2^-11 rounding), j added
// into the exponent field.  t is clamped at -125 (the result is then a
// positive denormal: fp16 0, like the SFU path's flush).
__device__ __forceinline__ float2 exp2_poly2(float2 t) {
  t.x = fmaxf(t.x, -125.f);
  t.y = fmaxf(t.y, -125.f);
  const float2 sh = make_float2(12582912.f, 12582912.f), nsh = make_float2(-12582912.f, -12582912.f);
  const float2 m1 = make_float2(-1.f, -1.f);
  const float2 y = __fadd2_rn(t, sh);                  // round(t) in the low mantissa bits
  const float2 f = __ffma2_rn(__fadd2_rn(y, nsh), m1, t);  // t - round(t), exact
  float2 p = __ffma2_rn(f, make_float2(0.055212993f, 0.055212993f), make_float2(0.24271414f, 0.24271414f));
  p = __ffma2_rn(p, f, make_float2(0.69326216f, 0.69326216f));
  p = __ffma2_rn(p, f, make_float2(0.99991959f, 0.99991959f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(y.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(y.y) << 23)));
}

// exp + row-sum + fp16 pack of 64 S columns; POLY of every 8 column pairs
// go through exp2_poly2, the rest through MUFU.EX2.
template <int POLY>
__device__ __forceinline__ void exp_pack64(const uint32_t (&u)[2][32], float2 c12, float2 mo2, float2& psa,
                                           float2& psb, uint32_t (&pk)[32]) {
#pragma unroll
  for (int e = 0; e < 64; e += 2) {
    const float2 x = make_float2(__uint_as_float(u[e >> 5][e & 31]), __uint_as_float(u[e >> 5][(e + 1) & 31]));
    const float2 t = __ffma2_rn(x, c12, mo2);  // (s - m) * scale * log2(e), two lanes
    const int pr = (e >> 1) & 7;
    const bool poly = POLY == 4 ? (pr & 1) == 0 : POLY == 3 ? (pr == 0 || pr == 3 || pr == 5)
                    : POLY == 2 ? (pr == 0 || pr == 4) : POLY == 1 ? pr == 0 : false;
    const float2 pp = poly ? exp2_poly2(t) : make_float2(fast_exp2(t.x), fast_exp2(t.y));
    if ((e >> 1) & 1) psb = __fadd2_rn(psb, pp); else psa = __fadd2_rn(psa, pp);
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(pk[e / 2]) : "f"(pp.y), "f"(pp.x));
  }
}

// S_i = Q_qt K^T from K ring stage kst into TMEM tile i (split mode: both
// TMEM tiles use Q tile 0 against different key tiles)
__device__ __forceinline__ void issue_s_at(uint32_t tmem, uint64_t dq0, uint64_t dk0, uint32_t id_s, int i, int qt,
                                           int kst, uint64_t* s_full) {
  const uint64_t dk = dk0 + (uint64_t)(kst * (TILE >> 4));
  const uint64_t dq = dq0 + (uint64_t)(qt * (TILE >> 4));
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) {
    const uint32_t off = ((ks >> 2) * REGION + (ks & 3) * 32) >> 4;
    mma_ss(tmem + i * 128, dq + off, dk + off, id_s, ks > 0);
  }
  mma_commit(&s_full[i]);
}

// ring position of (TMEM tile i, its step j) in split mode: tile 0's key
// tiles and tile 1's alternate; a last extra tile of tile 1 comes at the end
__device__ __forceinline__ int sp_pos(int i, int j, int nk0) { return j < nk0 ? 2 * j + i : 2 * nk0; }

// S_i(j) = Q_i K_j^T: 8 MMAs (K = 16 each) into TMEM columns [128 i, 128 i + 128)
__device__ __forceinline__ void issue_s(uint32_t tmem, uint64_t dq0, uint64_t dk0, uint32_t id_s, int i, int j,
                                        bool skip, uint64_t* s_full) {
  const uint64_t dk = dk0 + (uint64_t)((j % KST) * (TILE >> 4));
  const uint64_t dq = dq0 + (uint64_t)(i * (TILE >> 4));
  if (!skip) {
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      const uint32_t off = ((ks >> 2) * REGION + (ks & 3) * 32) >> 4;
      mma_ss(tmem + i * 128, dq + off, dk + off, id_s, ks > 0);
    }
  }
  mma_commit(&s_full[i]);
}
}  // namespace pf

// Instrumentation timeline (a.prof and a.timeline): CTA 0's MMA thread logs
// (event, clock) pairs after the per-CTA counters.
#define PF_T(ev)                                                                  \
  do {                                                                            \
    if (tl && tln < 2000) {                                                       \
      tl[2 * tln] = (ev);                                                         \
      tl[2 * tln + 1] = clock64();                                                \
      ++tln;                                                                      \
    }                                                                             \
  } while (0)

// CTA (pair p, head h, stream s): Q tiles t0 = 2p and t0 + 1 (if it exists).
template <int POLY, bool PROF>
__global__ void __launch_bounds__(pf::THREADS, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                   const __grid_constant__ CUtensorMap vmap, const PrefillArgs a) {
  using namespace pf;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align up by offset from the array (keeps the shared state space: LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  if (a.meta_len && blockIdx.x == 0 && threadIdx.x == 0) {  // the chunk's lengths / next positions
    for (int s = 0; s < a.S; ++s) {
      a.meta_len[s * a.meta_ss] = a.meta_n;
      a.meta_next[s * a.meta_ss] += a.C;
    }
  }
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SBAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [KST]
  uint64_t* k_empty = k_full + KST;       // [KST]
  uint64_t* v_full = k_empty + KST;       // [STAGES] TMA landed (bf16)
  uint64_t* v_conv = v_full + STAGES;     // [STAGES] converted to fp16
  uint64_t* v_empty = v_conv + STAGES;    // [STAGES]
  uint64_t* s_full = v_empty + STAGES;    // [QT] S_i(j) in TMEM
  uint64_t* p_full = s_full + QT;         // [QT] P_i(j) written (and O_i rescaled)
  uint64_t* o_final = p_full + QT;        // [QT] last P_i V done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_final + QT);

  // The pairs of one (stream, head) are consecutive CTAs, so its K/V stream
  // is read from DRAM once and served to the other pairs from L2 (a
  // longest-first order over all heads measured the same time with 2.5x the
  // DRAM traffic); within a head the two-tile pairs go from the last (most
  // keys) to the first.  The lone last tiles of an odd tile count (split over
  // both warpgroups: about half a pair's time) come after all pairs and fill
  // the last wave (config 2: 257 -> 237 us per layer).
  const int nqt = (a.C + BM - 1) / BM, npairs = (nqt + 1) / 2, full = nqt / 2;
  int sh, p;
  if (a.order == 1 && npairs > full) {
    // two-tile CTAs first (head-major, L2 reuse within a head), the lone last
    // tiles (about half the work) at the end to fill the last wave
    const int nfull = a.S * a.Hq * full;
    if ((int)blockIdx.x < nfull) {
      sh = blockIdx.x / full;
      p = full - 1 - (int)(blockIdx.x - sh * full);
    } else {
      sh = blockIdx.x - nfull;
      p = full;
    }
  } else {
    sh = blockIdx.x / npairs;
    const int rank = blockIdx.x - sh * npairs;
    p = rank < full ? full - 1 - rank : full;
  }
  const int h = sh % a.Hq, s = sh / a.Hq;
  const int g = h / a.G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = a.C, n0 = a.n0;
  int nkv0, nkv1;
  {
    const int t = 2 * p;
    nkv0 = (n0 + min((t + 1) * BM, C) + BN - 1) / BN;
    nkv1 = t + 1 < nqt ? (n0 + min((t + 2) * BM, C) + BN - 1) / BN : 0;
  }
  (void)npairs;
  // Split mode (a lone Q tile with enough keys): the second softmax
  // warpgroup and TMEM half take the upper half of the key tiles for the same
  // queries, and the two partial (O, m, l) are merged in the epilogue -- two
  // softmax chains in flight instead of one.  Every row must see a key of the
  // upper half's first tile (no all-masked first step).
  const int q0t = 2 * p * BM;
  const bool sp = a.split && nkv1 == 0 && nkv0 >= 2 && (nkv0 / 2) * BN < n0 + q0t + 1;
  const int hsp = sp ? nkv0 / 2 : 0;
  if (sp) {
    nkv1 = nkv0 - hsp;
    nkv0 = hsp;
  }
  const int nkv_max = max(nkv0, nkv1);
  const int npos = sp ? nkv0 + nkv1 : nkv_max;  // K/V ring positions
  const int seg_row = (int)(((int64_t)s * a.L + a.layer) * a.Hkv + g) * a.cap;

  if (tid == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_conv[i], NCONV);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < QT; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);  // every softmax warp (both column halves)
      mbar_init(&o_final[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  unsigned long long* prof = nullptr;
  unsigned long long t_start = 0;
  // register accumulators, stored once at exit
  unsigned long long pacc0 = 0, pacc1 = 0, pacc2 = 0, pacc3 = 0, pacc4 = 0;
  if (PROF && a.prof && lane == 0 && (warp == 9 || warp == 0 || warp == 4)) {
    const int cta = blockIdx.x;
    prof = a.prof + (size_t)cta * 16 + (warp == 9 ? 0 : warp == 0 ? 6 : 11);
    t_start = clock64();
  }

  if (warp >= 8) {
    // (setmaxnreg 208/80 for the softmax / other warpgroups measured no gain)
    if (warp == 8) {
      // ----------------------------------------------------------- producer
      if (lane == 0) {
        const int ntq = (nkv1 > 0 && !sp) ? 2 : 1;
        mbar_arrive_expect_tx(q_full, ntq * TILE);
        for (int i = 0; i < ntq; ++i) {
          const int row = s * C + (2 * p + i) * BM;
          tma_load_3d(smem + SQ + i * TILE, &qmap, 0, h, row, q_full);
          tma_load_3d(smem + SQ + i * TILE + REGION, &qmap, 64, h, row, q_full);
        }
        // K runs one tile ahead of V (S(j+1) is issued before P(j) V(j));
        // position r holds key tile r, or in split mode the alternating halves
        for (int j = 0; j <= npos; ++j) {
          if (j < npos) {
            const int st = j % KST;
            const int kt = !sp ? j : j < 2 * nkv0 ? ((j & 1) ? hsp + (j >> 1) : (j >> 1)) : hsp + nkv0;
            const int y = seg_row + kt * BN;
            mbar_wait(&k_empty[st], ((j / KST) & 1) ^ 1);
            mbar_arrive_expect_tx(&k_full[st], TILE);
            tma_load_2d(smem + SK + st * TILE, &kmap, 0, y, &k_full[st]);
            tma_load_2d(smem + SK + st * TILE + REGION, &kmap, 64, y, &k_full[st]);
          }
          if (j > 0) {
            const int jv = j - 1, st = jv % STAGES;
            const int kt = !sp ? jv : jv < 2 * nkv0 ? ((jv & 1) ? hsp + (jv >> 1) : (jv >> 1)) : hsp + nkv0;
            const int y = seg_row + kt * BN;
            mbar_wait(&v_empty[st], ((jv / STAGES) & 1) ^ 1);
            mbar_arrive_expect_tx(&v_full[st], TILE);
            tma_load_2d(smem + SV + st * TILE, &vmap, 0, y, &v_full[st]);
            tma_load_2d(smem + SV + st * TILE + REGION, &vmap, 64, y, &v_full[st]);
          }
        }
      }
    } else if (warp == 9) {
      // --------------------------------------------------------- MMA issuer
      if (lane == 0) {
        // Descriptors are built once; per MMA only a compile-time offset (in
        // 16-byte units) is added to the start-address field.
        const uint32_t id_s = idesc(BN, false, false), id_o = idesc(HD, true, true);
        const uint64_t dq0 = smem_desc(smem_u32(smem + SQ), 16, 1024);
        const uint64_t dk0 = smem_desc(smem_u32(smem + SK), 16, 1024);
        const uint64_t dv0 = smem_desc(smem_u32(smem + SV), REGION, 1024);
        unsigned long long* tl = (PROF && a.prof && a.timeline && blockIdx.x == 0) ? a.prof + 16 * gridDim.x : nullptr;
        int tln = 0;
        mbar_wait(q_full, 0);
        PF_T(1);
        if (sp) {
          // split mode: each TMEM tile walks its own key half through the
          // shared rings (positions alternate), Q tile 0 for both
#pragma unroll
          for (int i = 0; i < QT; ++i) {
            const int r = sp_pos(i, 0, nkv0);
            mbar_wait(&k_full[r % KST], (r / KST) & 1);
            tc_fence_after();
            issue_s_at(tmem, dq0, dk0, id_s, i, 0, r % KST, s_full);
            mma_commit(&k_empty[r % KST]);
          }
          for (int j = 0; j < nkv_max; ++j) {
#pragma unroll
            for (int i = 0; i < QT; ++i) {
              const int nk = i ? nkv1 : nkv0;
              if (j >= nk) continue;
              const int r = sp_pos(i, j, nkv0), vst = r % STAGES;
              mbar_wait(&v_conv[vst], (r / STAGES) & 1);
              mbar_wait(&p_full[i], j & 1);
              tc_fence_after();
              const uint64_t dv = dv0 + (uint64_t)(vst * (TILE >> 4));
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk)
                mma_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, dv + (uint64_t)((kk * 16 * 128) >> 4), id_o,
                       (j > 0 || kk > 0));
              if (j == nk - 1) mma_commit(&o_final[i]);
              mma_commit(&v_empty[vst]);
              if (j + 1 < nk) {
                const int r2 = sp_pos(i, j + 1, nkv0);
                mbar_wait(&k_full[r2 % KST], (r2 / KST) & 1);
                tc_fence_after();
                issue_s_at(tmem, dq0, dk0, id_s, i, 0, r2 % KST, s_full);
                mma_commit(&k_empty[r2 % KST]);
              }
            }
          }
        } else {
        PF_WAIT(0, &k_full[0], 0);
        PF_T(2);
        tc_fence_after();
        const bool skip_s = a.dbg == 2 || a.dbg == 3;
        issue_s(tmem, dq0, dk0, id_s, 0, 0, skip_s, s_full);
        if (nkv1 > 0) issue_s(tmem, dq0, dk0, id_s, 1, 0, skip_s, s_full);
        mma_commit(&k_empty[0]);
        for (int j = 0; j < nkv_max; ++j) {
          const int st = j % STAGES;
          const bool next = j + 1 < nkv_max;
          PF_T(10);
          PF_WAIT(2, &v_conv[st], (j / STAGES) & 1);
          PF_T(11);
          tc_fence_after();
          const uint64_t dv = dv0 + (uint64_t)(st * (TILE >> 4));
#pragma unroll
          for (int i = 0; i < QT; ++i) {
            const int nk = i ? nkv1 : nkv0;
            if (j >= nk) continue;
            PF_T(20 + i);
            PF_WAIT(3, &p_full[i], j & 1);
            PF_T(30 + i);
            tc_fence_after();
            const long long tp0 = prof ? clock64() : 0;
            if (a.dbg != 2 && a.dbg != 4) {
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk)  // 16 keys of 128-byte rows per step
                mma_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, dv + (uint64_t)((kk * 16 * 128) >> 4), id_o,
                       (j > 0 || kk > 0));
            }
            if (j == nk - 1) mma_commit(&o_final[i]);
            if (prof) pacc1 += clock64() - tp0;
            if (j + 1 < nk) {
              if (i == 0 || nkv0 <= j + 1) {  // first S of tile j+1: its K must have landed
                PF_T(40);
                PF_WAIT(0, &k_full[(j + 1) % KST], ((j + 1) / KST) & 1);
                PF_T(41);
                tc_fence_after();
              }
              const long long tq0 = prof ? clock64() : 0;
              issue_s(tmem, dq0, dk0, id_s, i, j + 1, skip_s, s_full);
              if (prof) pacc4 += clock64() - tq0;
            }
          }
          PF_T(50);
          mma_commit(&v_empty[st]);
          if (next) mma_commit(&k_empty[(j + 1) % KST]);
        }
        }  // !sp
      }
    } else {
      // ------------------------------------------ V conversion bf16 -> fp16
      // in place, same swizzled positions; warp w handles 16-byte chunks
      // w-10, w-10+NCONV, ... of the 32 KB tile
      const int cw = warp - 10;
      uint32_t vmax = 0;  // max |bf16 bits| seen, two halves
      for (int j = 0; j < npos; ++j) {
        const int st = j % STAGES;
        mbar_wait(&v_full[st], (j / STAGES) & 1);
        uint4* base = reinterpret_cast<uint4*>(smem + SV + st * TILE);
#pragma unroll 4
        for (int c = cw * 32 + lane; c < ((a.dbg == 5 || a.dbg == 6) ? 0 : TILE / 16); c += NCONV * 32) {
          uint4 x = base[c];
          uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            vmax = __vmaxu2(vmax, w[e] & 0x7fff7fffu);
            const float lo = __uint_as_float(w[e] << 16), hi = __uint_as_float(w[e] & 0xffff0000u);
            uint32_t hv;
            asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(hv) : "f"(hi), "f"(lo));
            w[e] = hv;
          }
          base[c] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_async_smem();  // generic-proxy stores -> tensor-core (async proxy) reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&v_conv[st]);
      }
      // |v| >= 65536 (bf16 0x4780) does not fit fp16: it was saturated
      const bool sat = (vmax & 0xffffu) >= 0x4780u || (vmax >> 16) >= 0x4780u;
      if (a.ovf && __any_sync(0xffffffffu, sat) && lane == 0) atomicAdd(a.ovf, 1);
    }
  } else {

    // ------------------- softmax: the 8 warps take both Q tiles in turn.
    // Warp w covers TMEM lanes 32 (w & 3) (rows) and S columns
    // [64 c, 64 c + 64), c = w >> 2: both warps of a lane quadrant form the
    // row maximum over all 128 columns (identical, no exchange) and each
    // exponentiates its half -- half the per-step latency of one thread per
    // row, so a tile's softmax fits in the other tile's MMAs.
    const int c = warp >> 2;
    const int r = tid & 127;  // row of the tile: 32 (warp & 3) + lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float c1 = a.scale * kLog2e;
    float m[QT], l[QT];
    int qi[QT], limit[QT], tml[QT], kt0[QT], nk[QT], wrow[QT];
    bool valid[QT], rec[QT], any_rec[QT], lg_aligned[QT];
    float* lgrow[QT];
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      m[i] = -INFINITY;  // running (possibly stale) max of the raw q.k
      l[i] = 0.f;        // this half's share of the row sum
      nk[i] = i ? nkv1 : nkv0;
      const int q0 = sp ? q0t : (2 * p + i) * BM;
      kt0[i] = (sp && i) ? hsp : 0;  // first key tile of TMEM tile i
      qi[i] = q0 + r;                 // query index in the chunk
      valid[i] = qi[i] < C;
      limit[i] = valid[i] ? n0 + qi[i] + 1 : n0 + 1;  // keys [0, limit) are visible
      tml[i] = n0 + q0 + 1;                           // smallest limit of the tile's rows
      wrow[i] = qi[i] - (C - a.W);                    // window row index (>= 0: recorded)
      rec[i] = valid[i] && a.lg && wrow[i] >= 0;
      // row-major [S][W][Hq][lg_cap] (ABI), or column-quad-major (engine):
      // quad t/4 of recorded row wrow at ((s*Hq + h)*(lg_cap/4) + t/4)*4W + 4*wrow
      lgrow[i] = !rec[i] ? nullptr
               : a.lg_t ? a.lg + (int64_t)(s * a.Hq + h) * (a.lg_cap / 4) * (4 * a.W) + 4 * wrow[i]
                        : a.lg + ((int64_t)(s * a.W + wrow[i]) * a.Hq + h) * a.lg_cap;
      any_rec[i] = __any_sync(0xffffffffu, rec[i]);
      lg_aligned[i] = (reinterpret_cast<uintptr_t>(lgrow[i]) & 15) == 0;
    }
    const int pair_bar = 1 + (warp & 3);  // the two warps of this lane quadrant
    float* xmax = reinterpret_cast<float*>(smem + SXCH);
    for (int j = 0; j < nkv_max; ++j) {
#pragma unroll
      for (int i = 0; i < QT; ++i) {
        if (j >= nk[i]) continue;
        PF_WAIT(0, &s_full[i], j & 1);  // also implies P_i(j-1) V is complete
        tc_fence_after();
        if (a.dbg == 1 || a.dbg == 6) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[i]);
          continue;
        }
        const uint32_t s_base = tmem + lane_off + i * 128;
        const uint32_t o_base = tmem + lane_off + 256 + i * 128 + 64 * c;
        const int tbase = (kt0[i] + j) * BN;
        // causal mask needed for some row of the tile (warp-uniform: the last
        // one or two tiles only)
        const bool diag = tbase + BN > tml[i];
        // this warp's 64 columns; the row max meets the partner half's in
        // shared memory (two pair barriers: the buffer is reused every step)
        uint32_t own[2][32];
        tmem_ld32_async(s_base + 64 * c, own[0]);
        tmem_ld32_async(s_base + 64 * c + 32, own[1]);
        tc_wait_ld();
        const int cb = 64 * c;  // this warp's first column
#define PF_U(e) own[(e) >> 5][(e) & 31]
        if (diag) {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (tbase + cb + e >= limit[i]) PF_U(e) = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {m[i], -INFINITY, -INFINITY, -INFINITY};  // four 3-input max chains
#pragma unroll
        for (int e = 0; e < 64; e += 8) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mx4[k] = fmaxf(mx4[k], fmaxf(__uint_as_float(PF_U(e + 2 * k)), __uint_as_float(PF_U(e + 2 * k + 1))));
        }
        const float mh = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));  // max(m, half max)
        xmax[c * 128 + r] = mh;
        // both halves have their S (loaded) and their max before either
        // writes P over S columns [0, 64) or reads the other max
        asm volatile("bar.sync %0, 64;\n" ::"r"(pair_bar) : "memory");
        const float mn = fmaxf(mh, xmax[(c ^ 1) * 128 + r]);  // max(m, row max)
        asm volatile("bar.sync %0, 64;\n" ::"r"(pair_bar) : "memory");  // buffer free again
        const bool grow = (mn - m[i]) * c1 > kRescaleLog2;  // true on the first tile (m = -inf)
        const bool rescale = j > 0 && __any_sync(0xffffffffu, grow);
        const float alpha = grow ? exp2f((m[i] - mn) * c1) : 1.f;
        if (grow) m[i] = mn;
        const float mo = m[i] * c1;
        const float2 c12 = make_float2(c1, c1), mo2 = make_float2(-mo, -mo);
        if (any_rec[i] && lgrow[i] && a.dbg != 7) {  // the last W rows: raw f32 logits for the window fold
          if (a.lg_t) {
            // one 512-byte run per column quad across the warp's recorded rows;
            // raw q.k (the fold applies the scale: the same f32 product), so the
            // stores read the live S registers and no temporaries serialise them
            float* dst = lgrow[i] + (int64_t)((tbase + cb) >> 2) * (4 * a.W);
#pragma unroll
            for (int e = 0; e < 64; e += 4)
              *reinterpret_cast<float4*>(dst + (int64_t)(e >> 2) * (4 * a.W)) =
                  make_float4(__uint_as_float(own[e >> 5][e & 31]), __uint_as_float(own[e >> 5][(e + 1) & 31]),
                              __uint_as_float(own[e >> 5][(e + 2) & 31]), __uint_as_float(own[e >> 5][(e + 3) & 31]));
          } else {
#pragma unroll
            for (int e = 0; e < 64; e += 4) {
              const int t = tbase + cb + e;
              const float x0 = __uint_as_float(own[e >> 5][e & 31]) * a.scale;
              const float x1 = __uint_as_float(own[e >> 5][(e + 1) & 31]) * a.scale;
              const float x2 = __uint_as_float(own[e >> 5][(e + 2) & 31]) * a.scale;
              const float x3 = __uint_as_float(own[e >> 5][(e + 3) & 31]) * a.scale;
              if (t + 3 < limit[i] && lg_aligned[i]) {
                *reinterpret_cast<float4*>(lgrow[i] + t) = make_float4(x0, x1, x2, x3);
              } else {
                if (t < limit[i]) lgrow[i][t] = x0;
                if (t + 1 < limit[i]) lgrow[i][t + 1] = x1;
                if (t + 2 < limit[i]) lgrow[i][t + 2] = x2;
                if (t + 3 < limit[i]) lgrow[i][t + 3] = x3;
              }
            }
          }
        }
        float2 psa = make_float2(0.f, 0.f), psb = make_float2(0.f, 0.f);
        {
          uint32_t pk[32];
          // recorded rows (window statistics) stay on the SFU path
          if (POLY > 0 && !any_rec[i])
            exp_pack64<POLY>(own, c12, mo2, psa, psb, pk);
          else
            exp_pack64<0>(own, c12, mo2, psa, psb, pk);
          tmem_st32u(s_base + c * 32, pk);  // fp16 P of columns [64 c, 64 c + 64)
        }
        const float2 ps = __fadd2_rn(psa, psb);
        if (grow && j > 0) l[i] *= alpha;
        l[i] += ps.x + ps.y;
        if (rescale) {  // this warp's half of the O row
#pragma unroll
          for (int c4 = 0; c4 < 2; ++c4) {
            float o32[32];
            tmem_ld32(o_base + c4 * 32, o32);
#pragma unroll
            for (int e = 0; e < 32; ++e) o32[e] *= alpha;
            tmem_st32(o_base + c4 * 32, o32);
          }
          if (prof) pacc2 += 1;
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i]);
#undef PF_U
      }
    }
    // ---- epilogue: the two halves' row sums meet in shared memory (the K
    // ring is idle once both tiles' last P V completed)
#pragma unroll
    for (int i = 0; i < QT; ++i)
      if (nk[i] > 0) PF_WAIT(3, &o_final[i], 0);
    tc_fence_after();
    float* xl = reinterpret_cast<float*>(smem + SK);  // [tile][half][128 rows]
#pragma unroll
    for (int i = 0; i < QT; ++i) xl[(2 * i + c) * 128 + r] = l[i];
    asm volatile("bar.sync 5, 256;\n" ::: "memory");
    float L[QT];
#pragma unroll
    for (int i = 0; i < QT; ++i) L[i] = xl[(2 * i) * 128 + r] + xl[(2 * i + 1) * 128 + r];
    if (sp) {
      // split: both TMEM tiles hold the same rows over the two key halves
      const float M = fmaxf(m[0], m[1]);
      const float f0 = exp2f((m[0] - M) * c1), f1 = exp2f((m[1] - M) * c1);
      const float Lt = L[0] * f0 + L[1] * f1;
      const float inv = 1.f / Lt;
      const uint32_t ob = tmem + lane_off + 256 + 64 * c;
      float* orow = a.out + ((int64_t)(s * C + (valid[0] ? qi[0] : 0)) * a.Hq + h) * HD + 64 * c;
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        float o0[32], o1[32];
        tmem_ld32(ob + c2 * 32, o0);
        tmem_ld32(ob + 128 + c2 * 32, o1);
        if (valid[0]) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(orow + c2 * 32 + e) =
                make_float4((o0[e] * f0 + o1[e] * f1) * inv, (o0[e + 1] * f0 + o1[e + 1] * f1) * inv,
                            (o0[e + 2] * f0 + o1[e + 2] * f1) * inv, (o0[e + 3] * f0 + o1[e + 3] * f1) * inv);
        }
      }
      if (c == 0 && rec[0] && a.st) {
        a.st[((int64_t)(s * a.W + wrow[0]) * a.Hq + h) * 2] = M * a.scale;
        a.st[((int64_t)(s * a.W + wrow[0]) * a.Hq + h) * 2 + 1] = Lt;
      }
    } else {
#pragma unroll
      for (int i = 0; i < QT; ++i) {
        if (nk[i] == 0) continue;
        const uint32_t ob = tmem + lane_off + 256 + i * 128 + 64 * c;
        float* orow = a.out + ((int64_t)(s * C + (valid[i] ? qi[i] : 0)) * a.Hq + h) * HD + 64 * c;
        const float inv = 1.f / L[i];
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          float o32[32];
          tmem_ld32(ob + c2 * 32, o32);  // warp-uniform (.sync.aligned)
          if (valid[i]) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(orow + c2 * 32 + e) =
                  make_float4(o32[e] * inv, o32[e + 1] * inv, o32[e + 2] * inv, o32[e + 3] * inv);
          }
        }
        if (c == 0 && rec[i] && a.st) {
          a.st[((int64_t)(s * a.W + wrow[i]) * a.Hq + h) * 2] = m[i] * a.scale;
          a.st[((int64_t)(s * a.W + wrow[i]) * a.Hq + h) * 2 + 1] = L[i];
        }
      }
    }
  }
  if (prof) {
    prof[4] = clock64() - t_start;
    prof[0] = pacc0;
    prof[1] += pacc1;
    prof[2] += pacc2;
    prof[3] = pacc3;
    if (warp == 9) prof[5] = pacc4;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- host side
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}
}  // namespace

cudaError_t make_kv_map(CUtensorMap* map, const void* base, int64_t rows, int box_rows) {
  EncodeFn enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)pf::HD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pf::HD * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static unsigned long long* g_prof = nullptr;
void set_prefill_profile(unsigned long long* p) { g_prof = p; }

cudaError_t launch_prefill(const void* q, int streams, const void* kbase, const void* vbase, int64_t kv_rows,
                           const PrefillArgs& a_in, cudaStream_t st) {
  PrefillArgs a = a_in;
  if (g_prof) a.prof = g_prof;
  {
    static int order = -1;  // SKV_PF_ORDER=0: head-major pairs then each head's lone tile
    if (order < 0) {
      const char* e = getenv("SKV_PF_ORDER");
      order = e ? atoi(e) : 1;
    }
    a.order = order;
  }
  {
    static int split = -1;  // SKV_PF_SPLIT=0 disables the lone-tile key split
    if (split < 0) {
      const char* e = getenv("SKV_PF_SPLIT");
      split = e ? atoi(e) != 0 : 1;
    }
    a.split = split;
  }
#ifdef SKV_INSTRUMENT
  // instrumentation build only (build.sh with SKV_INSTRUMENT=1): these skip
  // MMAs / softmax / V conversion and would corrupt outputs in a product run
  if (const char* d = getenv("SKV_PF_DBG")) a.dbg = atoi(d);
  if (const char* d = getenv("SKV_PF_TL")) a.timeline = atoi(d);
#else
  a.dbg = 0;
  a.timeline = 0;
#endif
  EncodeFn enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap qmap, kmap, vmap;
  {
    cuuint64_t dims[3] = {(cuuint64_t)pf::HD, (cuuint64_t)a.Hq, (cuuint64_t)streams * a.C};
    cuuint64_t strides[2] = {(cuuint64_t)pf::HD * 2, (cuuint64_t)a.Hq * pf::HD * 2};
    cuuint32_t box[3] = {64, 1, 128};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  cudaError_t e = make_kv_map(&kmap, kbase, kv_rows, pf::BN);
  if (e != cudaSuccess) return e;
  e = make_kv_map(&vmap, vbase, kv_rows, pf::BN);
  if (e != cudaSuccess) return e;
  // exp2 split between the SFU and the FMA pipe: POLY of every 8 column
  // pairs on the polynomial (SKV_PF_POLY overrides; 0 = SFU only)
  static int poly = -1;
  if (poly < 0) {
    const char* pe = getenv("SKV_PF_POLY");
    poly = pe ? std::min(4, std::max(0, atoi(pe))) : pf::kDefaultPoly;
  }
  // instrumented build (per-CTA wait counters, timeline) only when profiling
  using Kern = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, PrefillArgs);
  static const Kern kerns[2][5] = {
      {prefill_kernel<0, false>, prefill_kernel<1, false>, prefill_kernel<2, false>, prefill_kernel<3, false>,
       prefill_kernel<4, false>},
      {prefill_kernel<0, true>, prefill_kernel<1, true>, prefill_kernel<2, true>, prefill_kernel<3, true>,
       prefill_kernel<4, true>}};
  const int ki = (a.prof ? 5 : 0) + poly;
  const Kern kern = kerns[a.prof ? 1 : 0][poly];
  static DevOnce attr[10];
  if (!attr[ki].here()) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pf::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr[ki].here() = true;
  }
  const int nqt = (a.C + pf::BM - 1) / pf::BM;
  a.S = streams;
  dim3 grid((nqt + 1) / 2 * a.Hq * streams);
  kern<<<grid, pf::THREADS, pf::SMEM_BYTES, st>>>(qmap, kmap, vmap, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    fprintf(stderr, "prefill launch failed: regs %d, static smem %zu, dyn smem %d (opt-in max %d), max threads %d\n",
            fa.numRegs, fa.sharedSizeBytes, pf::SMEM_BYTES, optin, fa.maxThreadsPerBlock);
  }
  return e;
}

}  // namespace skv

namespace skv {

// Appends a C-token chunk's k/v ([S][C][Hkv][D] rows) to cache slots
// [n0, n0+C) of every (stream, kv-head) segment with token metadata
// (KvCache.append, cache.py:112-134, for C tokens at once).  Grid (C, S);
// thread t copies 16 bytes of one head's row.  The streams' lengths and next
// positions are stored by the prefill kernel that follows (PrefillArgs.meta_*).
__global__ void append_chunk_kernel(const uint4* __restrict__ kin, const uint4* __restrict__ vin, uint4* kc, uint4* vc,
                                    int64_t c_ss, int64_t c_hs, int Hkv, int units, int n0, int C, int64_t* pos,
                                    int8_t* modality, int32_t* round_id, int64_t m_ss, const int64_t* next_pos,
                                    int64_t np_ss, int mod, int rnd, const uint4* __restrict__ kraw_in,
                                    uint4* kraw_c) {
  const int i = blockIdx.x, s = blockIdx.y;
  for (int idx = threadIdx.x; idx < Hkv * units; idx += blockDim.x) {
    const int g = idx / units, u = idx - g * units;
    const int64_t src = ((int64_t)(s * C + i) * Hkv + g) * units + u;
    const int64_t d2 = s * c_ss + g * c_hs + (int64_t)(n0 + i) * units + u;
    kc[d2] = kin[src];
    vc[d2] = vin[src];
    if (kraw_c) kraw_c[d2] = kraw_in[src];  // RoPE: raw keys
  }
  if (threadIdx.x == 0) {
    pos[s * m_ss + n0 + i] = next_pos[s * np_ss] + i;
    modality[s * m_ss + n0 + i] = (int8_t)mod;
    round_id[s * m_ss + n0 + i] = rnd;
  }
}

// Folds the W recorded rows of a chunk into the window ring in one launch:
// grid (column blocks, S, W); row w has n_base + w + 1 columns and goes to
// ring slot (slot0 + w) mod Wring.  fold_vec4 (16-byte loads, four columns
// per thread) when the logit rows are 16-byte aligned, fold_piece otherwise.
template <int MODE>
__global__ void __launch_bounds__(256) fold_rows_kernel(const FoldArgs f, int Hq, int slot0, int Wring, int n_base,
                                                        int64_t lg_rs, int64_t st_rs, int64_t slot_stride, int vec) {
  __shared__ float stt[2 * 256];
  const int w = blockIdx.z, s = blockIdx.y;
  const int slot = (slot0 + w) % Wring;
  const int n = n_base + w + 1;
  const float* sg = f.stats + w * st_rs + s * f.st_ss;
  for (int x = threadIdx.x; x < 2 * Hq; x += blockDim.x) stt[x] = (x & 1) ? __frcp_rn(sg[x]) : sg[x];  // (M, 1/L)
  __syncthreads();
  if (vec) {
    const int j0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (j0 < n)
      fold_vec4<MODE>(f.logits + w * lg_rs + s * f.l_ss, f.l_hs, stt, f.rows + slot * slot_stride + s * f.r_ss, j0,
                      n, Hq, (float)(f.agg_div ? f.agg_div : Hq), f.accum);
  } else {
    FoldArgs g = f;
    g.logits = f.logits + w * lg_rs;
    g.stats = f.stats + w * st_rs;
    g.rows = f.rows + slot * slot_stride;
    g.wlen = nullptr;
    g.n = n;
    fold_piece(g, s, blockIdx.x, gridDim.x, Hq, threadIdx.x, blockDim.x);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && f.wlen) f.wlen[slot + s * f.w_ss] = n;
}

// Fold from the column-quad-major record layout (PrefillArgs::lg_t): lane =
// recorded row w (coalesced 16-byte logit loads across the warp), warp = one
// column quad; the CTA's [32 rows][32 columns] results go through shared
// memory so each window row is written in contiguous 128-byte runs.  Same
// per-column arithmetic as fold_vec4 (sequential heads, fold_prob).
template <int MODE>
__global__ void __launch_bounds__(256) fold_rows_t_kernel(const FoldArgs f, int Hq, int W, int64_t ncol4, int slot0,
                                                          int Wring, int n_base, int64_t slot_stride, float scale) {
  extern __shared__ float fsm[];
  float* stt = fsm;                 // [32][2 Hq]
  float* tile = fsm + 64 * Hq;      // [32][33]
  const int s = blockIdx.y, wg = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = wg * 32 + lane;
  const bool wv = w < W;
  // stage (M, 1/L) of the 32 rows: eight loads in flight per thread
  for (int x0 = tid; x0 < 64 * Hq; x0 += 8 * 256) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int x = x0 + i * 256, wl = x / (2 * Hq), k = x - wl * 2 * Hq;
      v[i] = (x < 64 * Hq && wg * 32 + wl < W) ? f.stats[((int64_t)s * W + wg * 32 + wl) * 2 * Hq + k] : 1.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int x = x0 + i * 256;
      if (x < 64 * Hq) stt[x] = (x & 1) ? __frcp_rn(v[i]) : v[i];  // (M, 1/L)
    }
  }
  __syncthreads();
  const float* sw = stt + lane * 2 * Hq;
  const float agg = (float)(f.agg_div ? f.agg_div : Hq);
  const int64_t hstride = ncol4 * 4 * W;  // floats between heads
  const int64_t t4 = (int64_t)blockIdx.x * 8 + warp;
  float acc[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) acc[e] = MODE == 1 ? -INFINITY : 0.f;
  if (wv && t4 < ncol4) {
    const float* src = f.logits + (int64_t)s * Hq * hstride + t4 * 4 * W + 4 * w;
    // rolling prefetch: the loads of heads h+8..h+15 are in flight while
    // head h's columns are folded (sequential head order is kept)
    constexpr int HB = 8;
    float4 x[HB];
#pragma unroll
    for (int b = 0; b < HB; ++b)
      if (b < Hq) x[b] = __ldcs(reinterpret_cast<const float4*>(src + (int64_t)b * hstride));
    for (int h0 = 0; h0 < Hq; h0 += HB) {
#pragma unroll
      for (int b = 0; b < HB; ++b) {
        const int h = h0 + b;
        if (h < Hq) {
          const float M = sw[2 * h], rL = sw[2 * h + 1];
          const float v[4] = {__fmul_rn(x[b].x, scale), __fmul_rn(x[b].y, scale), __fmul_rn(x[b].z, scale),
                              __fmul_rn(x[b].w, scale)};  // logit = f32(q.k * scale)
          if (h + HB < Hq) x[b] = __ldcs(reinterpret_cast<const float4*>(src + (int64_t)(h + HB) * hstride));
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float p = fold_prob(v[e], M, rL);
            acc[e] = MODE == 1 ? fmaxf(acc[e], p) : __fadd_rn(acc[e], p);
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) tile[lane * 33 + warp * 4 + e] = MODE == 1 ? acc[e] : __fdiv_rn(acc[e], agg);
  __syncthreads();
  for (int wl = warp; wl < 32; wl += 8) {
    const int ww = wg * 32 + wl;
    if (ww >= W) break;
    const int n = n_base + ww + 1;
    const int slot = (slot0 + ww) % Wring;
    float* row = f.rows + (int64_t)slot * slot_stride + (int64_t)s * f.r_ss;
    const int j = blockIdx.x * 32 + lane;
    if (j < n) {
      const float v = tile[wl * 33 + lane];
      row[j] = (f.accum && j < n - 1) ? __fadd_rn(row[j], v) : v;
    }
    if (blockIdx.x == 0 && lane == 0 && f.wlen) f.wlen[slot + s * f.w_ss] = n;
  }
}

// Bulk-staged variant (the default): a CTA owns 16 column quads (64 columns)
// of 32 recorded rows and walks the heads; a producer warp copies each
// head's slab (one 8 KB cp.async.bulk when W = 32, else 512 bytes per quad)
// into an 8-deep shared-memory ring, so each SM keeps ~128 KB of logits in
// flight without holding registers.  Lane = recorded row, warp = two quads; same per-column
// arithmetic as fold_rows_t_kernel (sequential heads, fold_prob).
namespace fb {
#ifndef SKV_FB_Q4
#define SKV_FB_Q4 16
#endif
#ifndef SKV_FB_NST
#define SKV_FB_NST 8
#endif
constexpr int Q4 = SKV_FB_Q4;    // column quads per CTA
constexpr int NST = SKV_FB_NST;  // ring depth (heads in flight)
constexpr int SLAB = Q4 * 32 * 16;  // one head's bytes: [quad][row][4 floats]
}  // namespace fb

template <int MODE>
__global__ void __launch_bounds__(288) fold_rows_tb_kernel(const FoldArgs f, int Hq, int W, int64_t ncol4, int slot0,
                                                           int Wring, int n_base, int64_t slot_stride, float scale) {
  using namespace fb;
  extern __shared__ __align__(128) unsigned char fbs[];
  float* ring = reinterpret_cast<float*>(fbs);                       // [NST][Q4][32][4]
  uint64_t* full = reinterpret_cast<uint64_t*>(fbs + NST * SLAB);    // [NST]
  uint64_t* empty = full + NST;                                      // [NST]
  float* stt = reinterpret_cast<float*>(empty + NST);                // [32][2 Hq]
  float* tile = stt + 64 * Hq;                                       // [32][Q4*4 + 1]
  const int s = blockIdx.y, wg = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = min(32, W - wg * 32);
  const int64_t q0 = (int64_t)blockIdx.x * Q4;
  const int nq = (int)min((int64_t)Q4, ncol4 - q0);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);  // one arrive per consumer warp
    }
    mbar_fence_init();
  }
  // stage (M, 1/L) of the 32 rows: eight loads in flight per thread
  for (int x0 = tid; x0 < 64 * Hq && tid < 256; x0 += 8 * 256) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int x = x0 + i * 256, wl = x / (2 * Hq), k = x - wl * 2 * Hq;
      v[i] = (x < 64 * Hq && wl < rows) ? f.stats[((int64_t)s * W + wg * 32 + wl) * 2 * Hq + k] : 1.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int x = x0 + i * 256;
      if (x < 64 * Hq) stt[x] = (x & 1) ? __frcp_rn(v[i]) : v[i];  // (M, 1/L)
    }
  }
  __syncthreads();
  const int64_t hstride = ncol4 * 4 * W;  // floats between heads
  const float* base = f.logits + (int64_t)s * Hq * hstride + q0 * 4 * W + 4 * wg * 32;
  const uint32_t rb = (uint32_t)rows * 16;  // bytes of one quad's rows
  // producer: warp 0 lane 0 keeps NST heads in flight (refills as warps free slots)
  auto issue = [&](int h) {
    const int st = h % NST;
    float* dst = ring + st * (SLAB / 4);
    mbar_arrive_expect_tx(&full[st], rb * nq);
    if (rows == W && W == 32) {  // the quads' rows are contiguous: one copy
      bulk_g2s(dst, base + (int64_t)h * hstride, rb * nq, &full[st]);
    } else {
      for (int q = 0; q < nq; ++q) bulk_g2s(dst + q * 32 * 4, base + (int64_t)h * hstride + q * 4 * W, rb, &full[st]);
    }
  };
  if (warp == 8) {
    // producer warp: keeps NST heads in flight, refilling a slot once all
    // eight consumer warps have read it
    if (lane == 0) {
      for (int h = 0; h < Hq; ++h) {
        if (h >= NST) mbar_wait(&empty[h % NST], ((h / NST) - 1) & 1);
        issue(h);
      }
    }
    return;
  }
  const float* sw = stt + lane * 2 * Hq;
  const float agg = (float)(f.agg_div ? f.agg_div : Hq);
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = MODE == 1 ? -INFINITY : 0.f;
  const int qa = warp * 2;  // this warp's quads qa, qa + 1
  for (int h = 0; h < Hq; ++h) {
    const int st = h % NST;
    mbar_wait(&full[st], (h / NST) & 1);
    const float* slab = ring + st * (SLAB / 4);
    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
    if (lane < rows) {
      if (qa < nq) x0 = *reinterpret_cast<const float4*>(slab + (qa * 32 + lane) * 4);
      if (qa + 1 < nq) x1 = *reinterpret_cast<const float4*>(slab + ((qa + 1) * 32 + lane) * 4);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    const float M = sw[2 * h], rL = sw[2 * h + 1];
    const float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float p = fold_prob(__fmul_rn(v[e], scale), M, rL);  // logit = f32(q.k * scale)
      acc[e] = MODE == 1 ? fmaxf(acc[e], p) : __fadd_rn(acc[e], p);
    }
  }
  constexpr int TW = Q4 * 4 + 1;
#pragma unroll
  for (int e = 0; e < 8; ++e) tile[lane * TW + qa * 4 + e] = MODE == 1 ? acc[e] : __fdiv_rn(acc[e], agg);
  asm volatile("bar.sync 1, 256;\n" ::: "memory");  // the 8 consumer warps (the producer has left)
  for (int wl = warp; wl < rows; wl += 8) {
    const int ww = wg * 32 + wl;
    const int n = n_base + ww + 1;
    const int slot = (slot0 + ww) % Wring;
    float* row = f.rows + (int64_t)slot * slot_stride + (int64_t)s * f.r_ss;
#pragma unroll
    for (int c = lane; c < Q4 * 4; c += 32) {
      const int64_t j = q0 * 4 + c;
      if (j < n) {
        const float val = tile[wl * TW + c];
        row[j] = (f.accum && j < n - 1) ? __fadd_rn(row[j], val) : val;
      }
    }
    if (blockIdx.x == 0 && lane == 0 && f.wlen) f.wlen[slot + s * f.w_ss] = n;
  }
}

cudaError_t launch_fold_rows_t(int streams, int rows, const FoldArgs& f, int Hq, int slot0, int Wring, int n_base,
                               int64_t lg_cap, int64_t slot_stride, float scale, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (Hq > 256 || f.mode == 2 || lg_cap % 128) return cudaErrorInvalidValue;
  const int nmax = n_base + rows;
  const size_t smem = (size_t)(64 * Hq + 32 * 33) * sizeof(float);
  static DevOnce attr;
  if (!attr.here()) {
    cudaFuncSetAttribute(fold_rows_t_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    cudaFuncSetAttribute(fold_rows_t_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    attr.here() = true;
  }
  static int bulk = -1;  // SKV_FOLD_BULK=0: the register-prefetch variant
  if (bulk < 0) {
    const char* e = getenv("SKV_FOLD_BULK");
    bulk = e ? atoi(e) != 0 : 1;
  }
  if (bulk) {
    const size_t bsmem = (size_t)fb::NST * fb::SLAB + 2 * fb::NST * sizeof(uint64_t) +
                         (size_t)(64 * Hq + 32 * (fb::Q4 * 4 + 1)) * sizeof(float);
    static DevOnce battr;
    if (!battr.here()) {
      cudaFuncSetAttribute(fold_rows_tb_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(fold_rows_tb_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      battr.here() = true;
    }
    const int64_t ncol4 = lg_cap / 4;
    const int64_t need4 = ((int64_t)nmax + 3) / 4;  // quads any row needs
    dim3 bgrid((unsigned)((std::min(need4, ncol4) + fb::Q4 - 1) / fb::Q4), streams, (rows + 31) / 32);
    if (f.mode == 1)
      fold_rows_tb_kernel<1><<<bgrid, 288, bsmem, st>>>(f, Hq, rows, ncol4, slot0, Wring, n_base, slot_stride, scale);
    else
      fold_rows_tb_kernel<0><<<bgrid, 288, bsmem, st>>>(f, Hq, rows, ncol4, slot0, Wring, n_base, slot_stride, scale);
    return cudaGetLastError();
  }
  dim3 grid((nmax + 31) / 32, streams, (rows + 31) / 32);
  if (f.mode == 1)
    fold_rows_t_kernel<1><<<grid, 256, smem, st>>>(f, Hq, rows, lg_cap / 4, slot0, Wring, n_base, slot_stride, scale);
  else
    fold_rows_t_kernel<0><<<grid, 256, smem, st>>>(f, Hq, rows, lg_cap / 4, slot0, Wring, n_base, slot_stride, scale);
  return cudaGetLastError();
}

cudaError_t launch_fold_rows(int streams, int rows, const FoldArgs& f, int Hq, int slot0, int Wring, int n_base,
                             int64_t lg_rs, int64_t st_rs, int64_t slot_stride, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (Hq > 256 || f.mode == 2) return cudaErrorInvalidValue;
  const int nmax = n_base + rows;
  const bool vec = (f.l_hs % 4 == 0) && (lg_rs % 4 == 0) && (f.l_ss % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(f.logits) & 15) == 0;
  const int blocks = vec ? (nmax + 1023) / 1024 : std::max(1, std::min(32, (nmax + 255) / 256));
  dim3 grid(blocks, streams, rows);
  if (f.mode == 1)
    fold_rows_kernel<1><<<grid, 256, 0, st>>>(f, Hq, slot0, Wring, n_base, lg_rs, st_rs, slot_stride, vec);
  else
    fold_rows_kernel<0><<<grid, 256, 0, st>>>(f, Hq, slot0, Wring, n_base, lg_rs, st_rs, slot_stride, vec);
  return cudaGetLastError();
}

cudaError_t launch_append_chunk(const void* kin, const void* vin, void* kc, void* vc, int64_t c_ss_units,
                                int64_t c_hs_units, int S, int Hkv, int units, int n0, int C, int64_t* pos,
                                int8_t* modality, int32_t* round_id, int64_t m_ss, int64_t* next_pos, int32_t* len,
                                int64_t ss, int mod, int rnd, cudaStream_t st, const void* kraw_in, void* kraw_c) {
  (void)len;  // (stored by the prefill kernel after this one)
  dim3 grid(C, S);
  const int threads = std::min(1024, ((Hkv * units + 31) / 32) * 32);
  append_chunk_kernel<<<grid, threads, 0, st>>>(static_cast<const uint4*>(kin), static_cast<const uint4*>(vin),
                                                static_cast<uint4*>(kc), static_cast<uint4*>(vc), c_ss_units,
                                                c_hs_units, Hkv, units, n0, C, pos, modality, round_id, m_ss, next_pos,
                                                ss, mod, rnd, static_cast<const uint4*>(kraw_in),
                                                static_cast<uint4*>(kraw_c));
  return cudaGetLastError();
}

}  // namespace skv
