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
// One CTA = 128 queries x one head.  Warp 4 (TMA producer) loads the Q tile
// once and 128-key K/V tiles into a 2-stage ring with cp.async.bulk.tensor
// (128-byte swizzle); warp 5 owns TMEM and issues tcgen05.mma
// (M=128, N=128, K=16, bf16 -> f32): S = Q K^T into one of two TMEM S buffers,
// O += P V into a TMEM O accumulator.  Warps 0-3 (one query row per thread)
// read S with tcgen05.ld, run the online softmax, write P (bf16, swizzled
// K-major) to shared memory for the P.V MMA, and rescale O in TMEM when a
// row maximum grows.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

#include "skv_common.cuh"
#include "skv_internal.h"
#include "skv_fold.cuh"

namespace skv {
namespace pf {

constexpr int BM = 128;  // queries per CTA
constexpr int BN = 128;  // keys per tile
constexpr int HD = 128;  // head dim
constexpr int REGION = 128 * 64 * 2;                // [128 rows][64 bf16] swizzled region, 16 KB
constexpr int TILE_BYTES = 2 * REGION;              // 128 rows x 128 dims
constexpr int SQ = 0;
constexpr int SK = SQ + TILE_BYTES;                 // 2 stages
constexpr int SV = SK + 2 * TILE_BYTES;             // 2 stages
constexpr int SP = SV + 2 * TILE_BYTES;             // P, bf16 high part
constexpr int SP_LO = SP + TILE_BYTES;              // P - bf16(P), bf16 low part
constexpr int SBAR = SP_LO + TILE_BYTES;            // barriers after the tiles
constexpr int SMEM_BYTES = SBAR + 128 + 3 * 512 + 1008;  // barriers, row-max exchange, alignment slack

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

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M=128, N=128
// a_f16: A operand in fp16 (P), B in bf16 (V).
__host__ __device__ constexpr uint32_t idesc(bool b_mn_major, bool a_f16 = false) {
  return (1u << 4) | (a_f16 ? 0u : (1u << 7)) | (1u << 10) | (b_mn_major ? (1u << 16) : 0u) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// P enters the P.V MMA as two bf16 terms, hi = bf16(p) and lo = bf16(p - hi)
// (mixed fp16 x bf16 operands are not a tcgen05 kind::f16 combination): a
// single bf16 P costs ~2^-9 relative output error, above the 2e-3 bf16
// tolerance for rows dominated by one key; hi + lo keeps ~2^-16.
constexpr bool kPHalf = false;

__device__ __forceinline__ uint32_t pack_p(float lo, float hi) {
  if (kPHalf) {
    const uint32_t l = __half_as_ushort(__float2half_rn(lo));
    const uint32_t h = __half_as_ushort(__float2half_rn(hi));
    return l | (h << 16);
  }
  const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return l | (h << 16);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc)
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

__device__ __forceinline__ void tmem_st32(uint32_t addr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(addr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
      "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
      "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
      "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
      "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return l | (h << 16);
}

}  // namespace pf

// One CTA: 128 queries [q0, q0+128) of stream s, query head h (kv head h/G).
__global__ void __maxnreg__(168)  // 10 warps: <= 3 per SM sub-partition x 168 regs fit its 16K registers
    prefill_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                   const __grid_constant__ CUtensorMap vmap, const PrefillArgs a) {
  using namespace pf;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SBAR);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* p_ready = bars + 7;
  uint64_t* o_full = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int q0 = blockIdx.x * BM, h = blockIdx.y, s = blockIdx.z;
  const int g = h / a.G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = a.C, n0 = a.n0;
  const int q_hi = min(q0 + BM, C);                    // exclusive
  const int ntiles = (n0 + q_hi + BN - 1) / BN;        // key tiles touched by the causal rows
  const int seg_row = (int)(((int64_t)s * a.L + a.layer) * a.Hkv + g) * a.cap;

  if (tid == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
    }
    mbar_init(p_ready, 8);
    mbar_init(o_full, 1);
    mbar_fence_init();
  }
  if (warp == 9) {  // TMEM: S0 [0,128), S1 [128,256), O [256,384)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------- producer
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE_BYTES);
      tma_load_3d(smem + SQ, &qmap, 0, h, s * C + q0, q_full);
      tma_load_3d(smem + SQ + REGION, &qmap, 64, h, s * C + q0, q_full);
      for (int j = 0; j < ntiles; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * TILE_BYTES);
        const int y = seg_row + j * BN;
        tma_load_2d(smem + SK + st * TILE_BYTES, &kmap, 0, y, &kv_full[st]);
        tma_load_2d(smem + SK + st * TILE_BYTES + REGION, &kmap, 64, y, &kv_full[st]);
        tma_load_2d(smem + SV + st * TILE_BYTES, &vmap, 0, y, &kv_full[st]);
        tma_load_2d(smem + SV + st * TILE_BYTES + REGION, &vmap, 64, y, &kv_full[st]);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t id_s = idesc(false), id_o = idesc(true, kPHalf);
      const uint32_t sq = smem_u32(smem + SQ), sp = smem_u32(smem + SP), sp_lo = smem_u32(smem + SP_LO);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + SK + st * TILE_BYTES);
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint32_t off = (ks >> 2) * REGION + (ks & 3) * 32;
          mma_bf16(tmem + st * 128, smem_desc(sq + off, 16, 1024), smem_desc(sk + off, 16, 1024), id_s, ks > 0);
        }
        mma_commit(&s_full[st]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < ntiles; ++j) {
        if (j + 1 < ntiles) issue_s(j + 1);
        mbar_wait(p_ready, j & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + SV + (j & 1) * TILE_BYTES);
#pragma unroll
        for (int ks = 0; ks < 2 * (BN / 16); ++ks) {  // P_hi . V, then P_lo . V
          const int kk = ks & (BN / 16 - 1);
          const uint32_t pa = (ks < BN / 16 ? sp : sp_lo) + (kk >> 2) * REGION + (kk & 3) * 32;
          const uint32_t vb = sv + kk * 16 * 128;  // 16 keys of 128-byte rows
          mma_bf16(tmem + 256, smem_desc(pa, 16, 1024), smem_desc(vb, REGION, 1024), id_o, (j > 0 || ks > 0));
        }
        mma_commit(o_full);
        mma_commit(&kv_empty[j & 1]);
      }
    }
  } else {
    // -------------------------- softmax: 8 warps, two threads per query row
    // thread t owns row t & 127 (its TMEM lane) and key/output columns
    // [64*hf, 64*hf + 64), hf = t >> 7; the pair exchanges its row maximum
    // through shared memory once per tile and its row sum once at the end.
    const int r = tid & 127, hf = tid >> 7;
    const int qi = q0 + r;                 // query index in the chunk
    const bool valid = qi < C;
    const int limit = valid ? n0 + qi + 1 : 1;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + hf * 64;
    const int wrow = qi - (C - a.W);      // window row index (>= 0: recorded)
    const bool rec = valid && a.lg && wrow >= 0;
    float* lgrow = rec ? a.lg + ((int64_t)(s * a.W + wrow) * a.Hq + h) * a.lg_cap : nullptr;
    const bool lg_aligned = (reinterpret_cast<uintptr_t>(lgrow) & 15) == 0;
    unsigned* xch = reinterpret_cast<unsigned*>(bars + 16);  // [3][128] row maxima (orderable keys)
    float m = -INFINITY, l = 0.f;
    unsigned char* prow_base = smem + SP + hf * REGION + r * 128;
    for (int j = 0; j < ntiles; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float sv[64];
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        float t32[32];
        tmem_ld32(lane_base + st * 128 + c2 * 32, t32);
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c2 * 32 + i] = t32[i];
      }
      const int tbase = j * BN + hf * 64;
      float pm = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        sv[i] = tbase + i < limit ? sv[i] * a.scale : -INFINITY;
        pm = fmaxf(pm, sv[i]);
      }
      // pair maximum through a 3-buffer ring of atomicMax keys: buffer (j+2)%3 is
      // reset here and first used again after the next barrier
      if (j == 0) {
        if (hf == 0) {
          xch[r] = 0u;
          xch[128 + r] = 0u;
        }
        asm volatile("bar.sync 3, 256;\n" ::: "memory");
      }
      atomicMax(&xch[(j % 3) * 128 + r], orderable(pm));
      if (hf == 0) xch[((j + 2) % 3) * 128 + r] = 0u;
      asm volatile("bar.sync 3, 256;\n" ::: "memory");
      const unsigned key = xch[(j % 3) * 128 + r];
      const float tmax = __uint_as_float((key & 0x80000000u) ? (key & 0x7fffffffu) : ~key);
      if (lgrow) {
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const int t = tbase + i;
          if (t + 3 < limit && lg_aligned) {
            *reinterpret_cast<float4*>(lgrow + t) = make_float4(sv[i], sv[i + 1], sv[i + 2], sv[i + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (t + e < limit) lgrow[t + e] = sv[i + e];
          }
        }
      }
      const float mn = fmaxf(m, tmax);
      const float alpha = m == -INFINITY ? 0.f : exp2f((m - mn) * kLog2e);
      // P.V of the previous tile must be done before P is overwritten (and O rescaled)
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, mn > m)) {  // rescale this thread's O columns (warp-uniform tcgen05)
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            float o32[32];
            tmem_ld32(lane_base + 256 + c2 * 32, o32);
#pragma unroll
            for (int i = 0; i < 32; ++i) o32[i] *= alpha;
            tmem_st32(lane_base + 256 + c2 * 32, o32);
          }
          tc_wait_st();
        }
      }
      float psum = 0.f;
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) {
        float p8[8], lo8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          p8[e] = exp2f((sv[kc * 8 + e] - mn) * kLog2e);
          psum += p8[e];
          lo8[e] = p8[e] - __bfloat162float(__float2bfloat16_rn(p8[e]));
        }
        const uint4 hi = make_uint4(pack_p(p8[0], p8[1]), pack_p(p8[2], p8[3]), pack_p(p8[4], p8[5]),
                                    pack_p(p8[6], p8[7]));
        const uint4 lo = make_uint4(pack_p(lo8[0], lo8[1]), pack_p(lo8[2], lo8[3]), pack_p(lo8[4], lo8[5]),
                                    pack_p(lo8[6], lo8[7]));
        const int off = (kc ^ (r & 7)) << 4;
        *reinterpret_cast<uint4*>(prow_base + off) = hi;
        *reinterpret_cast<uint4*>(prow_base + (SP_LO - SP) + off) = lo;
      }
      l = l * alpha + psum;
      m = mn;
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
    }
    // epilogue: O / (l_self + l_partner) (two-term sum: the same in either order)
    float* lx = reinterpret_cast<float*>(xch);
    asm volatile("bar.sync 3, 256;\n" ::: "memory");  // everyone is done with the max ring
    lx[hf * 128 + r] = l;
    asm volatile("bar.sync 3, 256;\n" ::: "memory");
    const float lt = l + lx[(hf ^ 1) * 128 + r];
    mbar_wait(o_full, (ntiles - 1) & 1);
    tc_fence_after();
    float* orow = a.out + ((int64_t)(s * C + (valid ? qi : 0)) * a.Hq + h) * HD + hf * 64;
    const float inv = 1.f / lt;
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      float o32[32];
      tmem_ld32(lane_base + 256 + c2 * 32, o32);  // warp-uniform (.sync.aligned)
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(orow + c2 * 32 + i) =
              make_float4(o32[i] * inv, o32[i + 1] * inv, o32[i + 2] * inv, o32[i + 3] * inv);
      }
    }
    if (rec && a.st && hf == 0) {
      a.st[((int64_t)(s * a.W + wrow) * a.Hq + h) * 2] = m;
      a.st[((int64_t)(s * a.W + wrow) * a.Hq + h) * 2 + 1] = lt;
    }
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

cudaError_t make_kv_map(CUtensorMap* map, const void* base, int64_t rows) {
  EncodeFn enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)pf::HD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pf::HD * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_prefill(const void* q, int streams, const void* kbase, const void* vbase, int64_t kv_rows,
                           const PrefillArgs& a, cudaStream_t st) {
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
  cudaError_t e = make_kv_map(&kmap, kbase, kv_rows);
  if (e != cudaSuccess) return e;
  e = make_kv_map(&vmap, vbase, kv_rows);
  if (e != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pf::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((a.C + pf::BM - 1) / pf::BM, a.Hq, streams);
  prefill_kernel<<<grid, 320, pf::SMEM_BYTES, st>>>(qmap, kmap, vmap, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, prefill_kernel);
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
// thread t copies 16 bytes of one head's row.
__global__ void append_chunk_kernel(const uint4* __restrict__ kin, const uint4* __restrict__ vin, uint4* kc, uint4* vc,
                                    int64_t c_ss, int64_t c_hs, int Hkv, int units, int n0, int C, int64_t* pos,
                                    int8_t* modality, int32_t* round_id, int64_t m_ss, const int64_t* next_pos,
                                    int64_t np_ss, int mod, int rnd) {
  const int i = blockIdx.x, s = blockIdx.y;
  for (int idx = threadIdx.x; idx < Hkv * units; idx += blockDim.x) {
    const int g = idx / units, u = idx - g * units;
    const int64_t src = ((int64_t)(s * C + i) * Hkv + g) * units + u;
    const int64_t d2 = s * c_ss + g * c_hs + (int64_t)(n0 + i) * units + u;
    kc[d2] = kin[src];
    vc[d2] = vin[src];
  }
  if (threadIdx.x == 0) {
    pos[s * m_ss + n0 + i] = next_pos[s * np_ss] + i;
    modality[s * m_ss + n0 + i] = (int8_t)mod;
    round_id[s * m_ss + n0 + i] = rnd;
  }
}

// Folds the W recorded rows of a chunk into the window ring in one launch:
// grid (pieces, S, W); row w has n_base + w + 1 columns and goes to ring slot
// (slot0 + w) mod Wring.
__global__ void fold_rows_kernel(const FoldArgs f, int Hq, int slot0, int Wring, int n_base, int64_t lg_rs,
                                 int64_t st_rs, int64_t slot_stride) {
  const int w = blockIdx.z, s = blockIdx.y;
  const int slot = (slot0 + w) % Wring;
  FoldArgs g = f;
  g.logits = f.logits + w * lg_rs;
  g.stats = f.stats + w * st_rs;
  g.rows = f.rows + slot * slot_stride;
  g.wlen = f.wlen ? f.wlen + slot : nullptr;
  g.n = n_base + w + 1;
  fold_piece(g, s, blockIdx.x, gridDim.x, Hq, threadIdx.x, blockDim.x);
}

cudaError_t launch_fold_rows(int streams, int rows, const FoldArgs& f, int Hq, int slot0, int Wring, int n_base,
                             int64_t lg_rs, int64_t st_rs, int64_t slot_stride, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int pieces = std::max(1, std::min(32, (n_base + rows + 255) / 256));
  dim3 grid(pieces, streams, rows);
  fold_rows_kernel<<<grid, 256, 0, st>>>(f, Hq, slot0, Wring, n_base, lg_rs, st_rs, slot_stride);
  return cudaGetLastError();
}

// After the chunk: lengths and the next original position of every stream.
__global__ void chunk_meta_kernel(int32_t* len, int64_t* next_pos, int64_t ss, int n, int C, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < S) {
    len[s * ss] = n;
    next_pos[s * ss] += C;
  }
}

cudaError_t launch_append_chunk(const void* kin, const void* vin, void* kc, void* vc, int64_t c_ss_units,
                                int64_t c_hs_units, int S, int Hkv, int units, int n0, int C, int64_t* pos,
                                int8_t* modality, int32_t* round_id, int64_t m_ss, int64_t* next_pos, int32_t* len,
                                int64_t ss, int mod, int rnd, cudaStream_t st) {
  dim3 grid(C, S);
  const int threads = std::min(1024, ((Hkv * units + 31) / 32) * 32);
  append_chunk_kernel<<<grid, threads, 0, st>>>(static_cast<const uint4*>(kin), static_cast<const uint4*>(vin),
                                                static_cast<uint4*>(kc), static_cast<uint4*>(vc), c_ss_units,
                                                c_hs_units, Hkv, units, n0, C, pos, modality, round_id, m_ss, next_pos,
                                                ss, mod, rnd);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  chunk_meta_kernel<<<(S + 127) / 128, 128, 0, st>>>(len, next_pos, ss, n0 + C, C, S);
  return cudaGetLastError();
}

}  // namespace skv
