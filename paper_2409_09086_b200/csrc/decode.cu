// K1: split-KV flash-decode for one layer of S independent streams (sm_100a).
//
// Replaces, per (stream, layer) and decode step, the body of
// Session.decode_step (reference engine.py:264-273):
//   KvCache.append (cache.py:112-134)   -> the new k/v row is bulk-copied from the
//                                          input straight into the last tile and
//                                          written to the cache slot n_old;
//   Session._attend (engine.py:235-246) -> split-KV online softmax, packed FFMA2
//                                          dot products, reduce-scattered
//                                          warp-shuffle reductions, P.V in fp32;
//   aggregate_heads + AttentionWindow.push (policies.py:259-263, 107-115)
//                                       -> each tile records its logits; the
//                                          head-aggregated row is materialised
//                                          ("folded") by the NEXT launch of the
//                                          layer once the per-head (max, sum)
//                                          of this step exist.
//
// Persistent grid (CTAs/SM x SMs).  A chunk is a run of 64-token tiles of one
// (stream, kv-head) segment: large batches take 4-tile chunk tickets from a
// global counter (three in flight), small batches run a static schedule of
// one 2..8-tile chunk per CTA.  The producer warp streams each K and V tile
// into a 3-4 stage shared-memory ring with 1-D bulk async copies (TMA engine,
// mbarrier completion).  8 consumer warps (16 for GQA groups of 4+: two per
// row slice, each with half the group's heads) compute; a chunk's warp
// partials are merged by the epilogue warp (dynamic schedule, overlapped with
// the next chunk) or by all consumer threads (static), published and counted
// per segment.  merge_kernel (next in the stream, PDL) merges a segment's
// chunk partials in chunk order as soon as they are all counted and writes the
// output and per-head (max, sum).  A fold warp materialises the previous
// recorded step's window row meanwhile.  Under programmatic dependent launch
// the producer of layer l+1 streams cached K/V while layer l drains; anything
// that depends on the previous launch waits on griddepcontrol.wait.
#include "skv_common.cuh"
#include "skv_internal.h"
#include "skv_fold.cuh"
#include "skv_append.cuh"

namespace skv {

template <typename T, int D>
struct Geo {
  static constexpr int ELT = sizeof(T);
  static constexpr int RB = D * ELT;      // bytes per cached row
  static constexpr int LPR = RB / 16;     // lanes per row (16 B each)
  static constexpr int EPL = 16 / ELT;    // elements per lane
  static constexpr int RPW = 32 / LPR;    // rows per warp load
  static constexpr int NW = 8;            // consumer warps
  static constexpr int TT = 8 * NW;       // tokens per tile (8 rows per warp)
  static constexpr int RPWARP = TT / NW;  // rows per warp per tile
  static constexpr int ITERS = RPWARP / RPW;
  static constexpr int TILE = TT * RB;    // bytes per K (or V) tile
  static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "row geometry");
  static_assert(ITERS >= 1, "tile geometry");
};

// Consumer warps: NW row-warps x HS head groups.  GQA groups of 4+ heads are
// split over two warps per row slice (HS = 2: each warp carries half the
// group's q / accumulators), which doubles the warps per SM on the
// latency-bound small-batch path at the cost of reading each K/V row twice
// from shared memory.
template <int G>
struct Cw {
  static constexpr int HS = G >= 4 ? 2 : 1;  // head groups
  static constexpr int GH = G / HS;          // heads per consumer warp
  static constexpr int NCW = 8 * HS;         // consumer warps
  static constexpr int CT = NCW * 32;        // consumer threads
  static constexpr int THREADS = CT + 3 * 32;  // + producer, epilogue, fold warps
};

template <int CT>
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(CT) : "memory"); }
template <int CT>
__device__ __forceinline__ void handoff_sync() { asm volatile("bar.sync 2, %0;\n" ::"n"(CT + 32) : "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Publication of a chunk partial: a gpu-scope release add after a warp/CTA
// barrier orders every participating thread's partial stores before the
// count (release is cumulative), without a membar.gl per thread.
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ float rescale(float m, float M) {
  return m == -INFINITY ? 0.f : exp2f((m - M) * kLog2e);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}


template <typename T, int D, int G>
struct Smem {
  using Gm = Geo<T, D>;
  static constexpr int NW = Gm::NW;
  // ring depth: 4 stages (128 KB for bf16 D=128) where one CTA per SM is
  // resident anyway, so a static 4-tile chunk is prefetched whole under PDL
  // epilogue slot: header (4 ints) + wm[NW][G] + wl[NW][G] + wo[NW][G][D]
  static constexpr size_t slot_floats = 4 + 2 * NW * G + NW * G * D;
  static constexpr size_t slots = 2 * slot_floats * sizeof(float);
  static constexpr size_t pbuf = (size_t)NW * G * Gm::RPWARP * sizeof(float);
  // ring depth: as many K+V stages as fit next to the slots and 8 KB of fold
  // stats (f32 at D = 128 is 64 KB per stage: 2 stages)
  static constexpr int WANT = G >= 4 ? 4 : 3;
  static constexpr int SCAP = (int)((232448 - slots - pbuf - 8192 - 512) / (2 * Gm::TILE));
  static constexpr int STAGES = WANT < SCAP ? WANT : SCAP;
  static_assert(STAGES >= 2, "decode ring needs two stages");
  static constexpr size_t tiles = (size_t)STAGES * 2 * Gm::TILE;
  static constexpr size_t bars = (2 * STAGES + 4) * sizeof(uint64_t);
  static constexpr size_t tinfo = (2 * STAGES + 4) * sizeof(int);
  static constexpr size_t fixed = tiles + bars + tinfo + slots + pbuf;
  static size_t bytes(int Hq) { return fixed + 2 * (size_t)Hq * sizeof(float) + 16; }
};

template <typename T, int D, int G>
__global__ void __launch_bounds__(Cw<G>::THREADS, (G >= 4 ? 1 : 2)) decode_kernel(const AttnArgs a) {
  using Gm = Geo<T, D>;
  using Sm = Smem<T, D, G>;
  constexpr int GH = Cw<G>::GH, NCW = Cw<G>::NCW, kCT = Cw<G>::CT;
  constexpr int TT = Gm::TT, RB = Gm::RB, LPR = Gm::LPR, EPL = Gm::EPL, RPW = Gm::RPW;
  constexpr int NW = Gm::NW, ITERS = Gm::ITERS, STAGES = Sm::STAGES, TILE = Gm::TILE;
  constexpr int PW = D + 2;  // floats per head in a partial
  constexpr int SLOT = (int)Sm::slot_floats;

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* tiles = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Sm::tiles);
  uint64_t* empty = full + STAGES;
  uint64_t* epi_full = empty + STAGES;  // [2]
  uint64_t* epi_empty = epi_full + 2;   // [2]
  int* tinfo = reinterpret_cast<int*>(epi_empty + 2);               // [STAGES][2]
  int* cring = tinfo + 2 * STAGES;                                  // [4] next chunk tickets
  float* slots = reinterpret_cast<float*>(tinfo + 2 * STAGES + 4);  // [2][SLOT]
  float* pbuf_all = slots + 2 * SLOT;                               // [NW][G][RPWARP]
  float* fstats = pbuf_all + NW * G * Gm::RPWARP;                   // [Hq][2]

  const int c = blockIdx.x, P = gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n_old + a.append;
  const int total = a.S * a.Hkv * a.nc;

  if (a.gate) {  // speculative step: the gate grid ahead has completed and decided
    griddep_wait();
    if (*reinterpret_cast<const volatile int32_t*>(a.gate) != 1) return;
  }
  if (a.tstamp && tid == 0) atomicMin(&a.tstamp[0], globaltimer());
  if (a.ctat && tid == 0) a.ctat[8 * c] = globaltimer();
  if (c == 0 && tid == 0 && a.done_self) {  // a stale flag from this slot's previous use must not leak
    *a.done_self = 0;
    __threadfence();
  }
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&epi_full[i], NCW);
      mbar_init(&epi_empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  // Everything that depends on the previous launch (the preceding layer's
  // merge: q, in a real model, and the shared scratch) waits here.
  auto wait_prev = [&]() {
    if (a.done_prev) {  // the preceding merge kernel publishes its completion flag
      while (ld_acquire(a.done_prev) == 0) __nanosleep(32);
    } else {
      griddep_wait();
    }
  };

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      bool waited = false;
      if (!a.prefetch) {
        griddep_wait();
        waited = true;
      }
      int i = 0, taken = 0, kp = 0;
      // dynamic: three tickets in flight, so the atomic's latency is hidden
      // even for 1-tile chunks; static (few chunks): chunk blockIdx.x only
      int u = a.stat ? c : atomicAdd(&a.sched[0], 1);
      int t1 = a.stat ? total : atomicAdd(&a.sched[0], 1);
      int t2 = a.stat ? total : atomicAdd(&a.sched[0], 1);
      // Dynamic tickets hand out every segment's chunks but its last first,
      // then the last chunks (the short remainder chunk, and the one holding
      // the appended token, which waits for the previous launch): the launch
      // ends on the smallest work and no producer stalls on the release early.
      // With a.late = DL > 0, segment sigma's last chunk is handed out right
      // after segment sigma + DL's other chunks instead (DL segments ~ one
      // ticket per CTA later: past the release), so most segments complete --
      // and merge -- while later segments still stream, not all at the end.
      const int nce = a.nc - 1, segs = a.S * a.Hkv, early = segs * nce;
      const int DL = a.late > 0 && a.late < segs && nce > 0 ? a.late : 0;
      auto slot_of = [&](int t) {  // ticket -> chunk slot sigma * nc + j
        if (a.stat || t >= total) return t;
        if (DL == 0) return t < early ? (t / nce) * a.nc + (t % nce) : (t - early) * a.nc + nce;
        // blocks: sigma's nce early chunks, then (sigma >= DL) the last chunk of sigma - DL
        const int bD = DL * nce;                         // start of block DL
        const int bEnd = segs * nce + (segs - DL);       // after the last block
        if (t >= bEnd) return (segs - DL + (t - bEnd)) * a.nc + nce;  // remaining last chunks
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
      u = slot_of(u);
      while (u < total) {
        ++taken;
        const int u_next = slot_of(t1);
        t1 = t2;
        t2 = a.stat ? total : atomicAdd(&a.sched[0], 1);
        // published with this chunk's first tile: lets the consumers prefetch q
        cring[(kp + 1) & 3] = u_next < total ? u_next : -1;
        ++kp;
        const int sigma = u / a.nc, j = u - sigma * a.nc;
        const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
        const int tt0 = j * a.ch, tt1 = min(tt0 + a.ch, a.nt);
        const int64_t base = s * a.c_ss + (int64_t)g * a.c_hs;
        for (int tt = tt0; tt < tt1; ++tt, ++i) {
          const int ts = tt * TT;
          const int rows = min(TT, n - ts);
          const int rc = max(0, min(rows, a.n_old - ts));
          const int st = i % STAGES;
          mbar_wait(&empty[st], ((i / STAGES) & 1) ^ 1);
          tinfo[2 * st] = u;
          tinfo[2 * st + 1] = tt | ((tt == tt1 - 1) ? (1 << 30) : 0);
          unsigned char* ks = tiles + (2 * st) * TILE;
          unsigned char* vs = ks + TILE;
          mbar_arrive_expect_tx(&full[st], 2u * rows * RB);
          if (rc > 0) {
            bulk_g2s(ks, static_cast<const T*>(a.kc) + base + (int64_t)ts * D, rc * RB, &full[st]);
            bulk_g2s(vs, static_cast<const T*>(a.vc) + base + (int64_t)ts * D, rc * RB, &full[st]);
          }
          if (rc < rows) {  // the appended token: straight from the step input
            if (!waited) {
              wait_prev();
              waited = true;
            }
            const int64_t in = s * a.in_ss + (int64_t)g * D;
            bulk_g2s(ks + rc * RB, static_cast<const T*>(a.kin) + in, RB, &full[st]);
            bulk_g2s(vs + rc * RB, static_cast<const T*>(a.vin) + in, RB, &full[st]);
          }
        }
        u = u_next;
      }
      const int st = i % STAGES;  // end marker
      mbar_wait(&empty[st], ((i / STAGES) & 1) ^ 1);
      tinfo[2 * st] = -1;
      mbar_arrive(&full[st]);
      if (a.ctat) {
        a.ctat[8 * c + 6] = globaltimer();
        a.ctat[8 * c + 7] = taken;
      }
    }
    return;
  }

  if (warp == NCW + 2) {
    // ------------------------------------------------- window-row fold warp
    // Materialises the previous recorded step's window row (64-column pieces
    // c, c+P, ...) while the other warps stream K/V.
    const FoldArgs& f = a.fold;
    if (f.n <= 0) return;
    if (!a.prefetch) griddep_wait();  // same layer back to back: wait for its logits
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

  if (warp == NCW + 1) {
    // ------------------------------------------------------ epilogue warp
    if (!a.prefetch) griddep_wait();  // same layer back to back: the cache slot and metadata
    for (int k = 0;; ++k) {
      const int sl = k & 1;
      const uint32_t ph = (k >> 1) & 1;
      mbar_wait(&epi_full[sl], ph);
      const float* slot = slots + sl * SLOT;
      const int u = reinterpret_cast<const int*>(slot)[0];
      if (u < 0) break;
      const float* wm = slot + 4;
      const float* wl = wm + NW * G;
      const float* wo = wl + NW * G;
      const int sigma = u / a.nc, j = u - sigma * a.nc;
      // the segment's last chunk appends the new row first: its stores are in
      // flight while the partials merge, and precede the chunk's publication
      if (!a.stat && a.append && j == a.nc - 1) append_row<T, D>(a, sigma, n, lane, 32);
      // merge the consumer warps' partials of this chunk (static schedule:
      // the consumers already did)
      float* part = a.part + ((int64_t)sigma * a.nc + j) * G * PW;
#pragma unroll
      for (int h = 0; h < (a.stat ? 0 : G); ++h) {
        // lane w < NW holds warp w's (m, l); rescale factors computed once per head
        const float mw = lane < NW ? wm[lane * G + h] : -INFINITY;
        float M = mw;
#pragma unroll
        for (int off = NW / 2; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        const float f = lane < NW ? rescale(mw, M) : 0.f;
        float L = lane < NW ? f * wl[lane * G + h] : 0.f;
#pragma unroll
        for (int off = NW / 2; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
        float fw[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) fw[w] = __shfl_sync(0xffffffffu, f, w);
#pragma unroll
        for (int d = lane; d < D; d += 32) {
          float acc = 0.f;
#pragma unroll
          for (int w = 0; w < NW; ++w) acc = fmaf(fw[w], wo[(w * G + h) * D + d], acc);
          part[h * PW + d] = acc;
        }
        if (lane == 0) {
          part[h * PW + D] = M;
          part[h * PW + D + 1] = L;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&epi_empty[sl]);  // slot consumed
      if (!a.stat) {
        __syncwarp();
        // publish the chunk partial: the segment's merge CTA starts once all
        // nc chunks of the segment are counted
        if (lane == 0) red_release_add(&a.counters[sigma], 1);
      }
    }
    __threadfence();  // every chunk partial of this CTA visible GPU-wide
    handoff_sync<kCT>();
    return;
  }

  // -------------------------------------------------------------- consumers
  // q (the previous layer's output in a real model) crosses launches
  if (a.done_prev) {
    if (tid == 0) wait_prev();
    consumers_sync<kCT>();
  } else {
    griddep_wait();
  }
  // Let this launch's merge kernel be scheduled only once this CTA is
  // released: merges (and the decode launches they release early) then run at
  // most one launch ahead, which bounds the per-launch counter ring (a tiny
  // grid would otherwise let a whole captured graph's launches go resident).
  if (tid == 0) griddep_launch();
  if (a.ctat && tid == 0) a.ctat[8 * c + 1] = globaltimer();
  // Lane layout: LPR lanes read one cached row (16 B each); a warp reads RPW
  // rows per shared-memory load and ITERS loads per tile.  Partial dot products
  // of the ITERS rows are reduce-scattered across the LPR lanes (log2(LPR)
  // shuffles for ITERS rows instead of ITERS*log2(LPR)); afterwards each lane
  // owns the logit of row `ridx*RPW + rsub`, replicated REP times.
  constexpr int REP = LPR / ITERS;
  constexpr int E2 = EPL / 2;
  const int rsub = lane / LPR, c16 = lane % LPR;
  int ridx = 0;
#pragma unroll
  for (int cnt = ITERS, off = LPR / 2; cnt > 1; cnt >>= 1, off >>= 1)
    if (c16 & off) ridx += cnt / 2;
  const bool owner = (c16 & (REP - 1)) == 0;
  // row-warp rw takes rows [rw*RPWARP, ...) of each tile; head group hg the
  // group's heads [h0, h0 + GH)
  const int rw = warp % NW, hg = warp / NW, h0 = hg * GH;
  float* pbuf = pbuf_all + warp * GH * Gm::RPWARP;  // [GH][RPW][ITERS]
  float2 q2[GH][E2];
  float2 o2[GH][E2];
  float m_run[GH], l_run[GH];
  float* lg = nullptr;
  int cur = -1;
  int k = 0;  // chunks handed to the epilogue warp
  bool fresh = true;
  constexpr bool kPrefetchQ = G <= 2;  // register budget
  float qn[GH][EPL];  // prefetched q of the next chunk's segment
  int qn_sigma = -1;
  unsigned long long t_epi_wait = 0;
  for (int i = 0;; ++i) {
    const int st = i % STAGES;
    mbar_wait(&full[st], (i / STAGES) & 1);
    const int u = tinfo[2 * st];
    if (u < 0) break;
    const int info = tinfo[2 * st + 1];
    const int tt = info & 0xffff;
    const bool chunk_end = (info >> 30) & 1;
    const int sigma = u / a.nc;
    const int ts = tt * TT;
    const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
    if (fresh) {
      if (sigma != cur) {
        if (qn_sigma != sigma) {  // not prefetched (first chunk)
#pragma unroll
          for (int h = 0; h < GH; ++h)
            Vec16<T>::load(qn[h], static_cast<const T*>(a.q) + s * a.q_ss + (int64_t)(g * G + h0 + h) * D + c16 * EPL);
        }
#pragma unroll
        for (int h = 0; h < GH; ++h)
#pragma unroll
          for (int e = 0; e < E2; ++e) q2[h][e] = make_float2(qn[h][2 * e], qn[h][2 * e + 1]);
        cur = sigma;
        lg = a.logits ? a.logits + s * a.l_ss + (int64_t)(g * G + h0) * a.l_hs : nullptr;
      }
      // prefetch the next chunk's q (its ticket was published with this tile)
      const int un = (kPrefetchQ && a.qpf) ? cring[(k + 1) & 3] : -1;
      if (un >= 0 && un / a.nc != sigma) {
        const int sn = un / a.nc;
        const int s2 = sn / a.Hkv, g2 = sn - s2 * a.Hkv;
#pragma unroll
        for (int h = 0; h < GH; ++h)
          Vec16<T>::load(qn[h], static_cast<const T*>(a.q) + s2 * a.q_ss + (int64_t)(g2 * G + h0 + h) * D + c16 * EPL);
        qn_sigma = sn;
      }
#pragma unroll
      for (int h = 0; h < GH; ++h) {
#pragma unroll
        for (int e = 0; e < E2; ++e) o2[h][e] = make_float2(0.f, 0.f);
        m_run[h] = -INFINITY;
        l_run[h] = 0.f;
      }
      fresh = false;
    }
    const int rows = min(TT, n - ts);
    const unsigned char* ks = tiles + (2 * st) * TILE;
    const unsigned char* vs = ks + TILE;

    // ---- q . k for ITERS rows, packed FMA
    float d[ITERS][GH];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int row = rw * Gm::RPWARP + it * RPW + rsub;
      float2 kf[E2];
      Vec16<T>::load2(kf, ks + row * RB + c16 * 16);
#pragma unroll
      for (int h = 0; h < GH; ++h) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < E2; ++e) acc = __ffma2_rn(q2[h][e], kf[e], acc);
        d[it][h] = acc.x + acc.y;
      }
    }
    // ---- reduce-scatter across the LPR lanes of a row
#pragma unroll
    for (int cnt = ITERS, off = LPR / 2; cnt > 1; cnt >>= 1, off >>= 1) {
      const bool up = (c16 & off) != 0;
#pragma unroll
      for (int jj = 0; jj < cnt / 2; ++jj) {
#pragma unroll
        for (int h = 0; h < GH; ++h) {
          const float send = up ? d[jj][h] : d[jj + cnt / 2][h];
          const float keep = up ? d[jj + cnt / 2][h] : d[jj][h];
          d[jj][h] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
    }
#pragma unroll
    for (int off = REP / 2; off > 0; off >>= 1)
#pragma unroll
      for (int h = 0; h < GH; ++h) d[0][h] += __shfl_xor_sync(0xffffffffu, d[0][h], off);

    const int myrow = rw * Gm::RPWARP + ridx * RPW + rsub;
    const bool valid = myrow < rows;
    float sc[GH];
#pragma unroll
    for (int h = 0; h < GH; ++h) sc[h] = valid ? d[0][h] * a.scale : -INFINITY;
    if (lg && owner && valid) {
#pragma unroll
      for (int h = 0; h < GH; ++h) lg[h * a.l_hs + ts + myrow] = sc[h];
    }
    // ---- online softmax: one row per lane
#pragma unroll
    for (int h = 0; h < GH; ++h) {
      float mt = sc[h];
#pragma unroll
      for (int off = 16; off >= REP; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
      const float mn = fmaxf(m_run[h], mt);
      const float alpha = rescale(m_run[h], mn);
      const float pv = mn == -INFINITY ? 0.f : fast_exp2((sc[h] - mn) * kLog2e);
      l_run[h] = l_run[h] * alpha + (owner ? pv : 0.f);
      const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
      for (int e = 0; e < E2; ++e) o2[h][e] = __fmul2_rn(o2[h][e], a2);
      m_run[h] = mn;
      if (owner) pbuf[(h * RPW + rsub) * ITERS + ridx] = pv;
    }
    __syncwarp();
    // ---- P . V
    float pr[GH][ITERS];
#pragma unroll
    for (int h = 0; h < GH; ++h)
#pragma unroll
      for (int it = 0; it < ITERS; ++it) pr[h][it] = pbuf[(h * RPW + rsub) * ITERS + it];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int row = rw * Gm::RPWARP + it * RPW + rsub;
      if (row < rows) {
        float2 vf[E2];
        Vec16<T>::load2(vf, vs + row * RB + c16 * 16);
#pragma unroll
        for (int h = 0; h < GH; ++h) {
          const float2 p2 = make_float2(pr[h][it], pr[h][it]);
#pragma unroll
          for (int e = 0; e < E2; ++e) o2[h][e] = __ffma2_rn(p2, vf[e], o2[h][e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (!chunk_end) continue;

    // ---- chunk done: hand the warp partials to the epilogue warp
    const int sl = k & 1;
    unsigned long long tw0 = 0;
    if (a.ctat && tid == 0) tw0 = globaltimer();
    mbar_wait(&epi_empty[sl], ((k >> 1) & 1) ^ 1);
    if (a.ctat && tid == 0) t_epi_wait += globaltimer() - tw0;
    float* slot = slots + sl * SLOT;
    float* wm = slot + 4;
    float* wl = wm + NW * G;
    float* wo = wl + NW * G;
#pragma unroll
    for (int h = 0; h < GH; ++h) {
      float l = l_run[h];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
      float o[EPL];
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        o[2 * e] = o2[h][e].x;
        o[2 * e + 1] = o2[h][e].y;
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
#pragma unroll
        for (int off = LPR; off < 32; off <<= 1) o[e] += __shfl_xor_sync(0xffffffffu, o[e], off);
      }
      if (rsub == 0) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) wo[(rw * G + h0 + h) * D + c16 * EPL + e] = o[e];
      }
      if (lane == 0) {
        wm[rw * G + h0 + h] = m_run[h];
        wl[rw * G + h0 + h] = l;
      }
    }
    if (warp == 0 && lane == 0) reinterpret_cast<int*>(slot)[0] = u;
    if (a.stat) {
      // Static schedule (one chunk per CTA, latency-bound small batches): all
      // consumer threads merge the warp partials instead of the single
      // epilogue warp (same arithmetic order), then publish the chunk.
      consumers_sync<kCT>();
      const int j = u - sigma * a.nc;
      // the segment's last chunk stores the appended row (before publishing)
      if (a.append && j == a.nc - 1) append_row<T, D>(a, sigma, n, tid, kCT);
      float* part = a.part + ((int64_t)sigma * a.nc + j) * G * PW;
      for (int idx = tid; idx < G * D; idx += kCT) {
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
        if (d == 0) {  // the epilogue warp's xor-tree order over the NW warps
          float x[NW];
#pragma unroll
          for (int w = 0; w < NW; ++w) x[w] = f[w] * wl[w * G + h];
#pragma unroll
          for (int off = NW / 2; off > 0; off >>= 1)
#pragma unroll
            for (int w = 0; w < off; ++w) x[w] = x[w] + x[w + off];
          part[h * PW + D] = M;
          part[h * PW + D + 1] = x[0];
        }
      }
      consumers_sync<kCT>();
      if (tid == 0) red_release_add(&a.counters[sigma], 1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&epi_full[sl]);
    ++k;
    fresh = true;
  }
  if (a.ctat && tid == 0) {
    a.ctat[8 * c + 3] = globaltimer();
    a.ctat[8 * c + 4] = k;
    a.ctat[8 * c + 5] = t_epi_wait;
  }
  // end marker for the epilogue warp
  {
    const int sl = k & 1;
    mbar_wait(&epi_empty[sl], ((k >> 1) & 1) ^ 1);
    if (warp == 0 && lane == 0) reinterpret_cast<int*>(slots + sl * SLOT)[0] = -1;
    __syncwarp();
    if (lane == 0) mbar_arrive(&epi_full[sl]);
  }

  handoff_sync<kCT>();  // this CTA's epilogue warp has published its partials
  if (a.tstamp && tid == 0) atomicMax(&a.tstamp[1], globaltimer());
  if (a.ctat && tid == 0) a.ctat[8 * c + 2] = globaltimer();
  if (tid == 0) {
    // the last CTA out resets the ticket counter and the (already observed)
    // flag of the previous merge
    if (atomicAdd(&a.sched[2], 1) == P - 1) {
      a.sched[0] = 0;
      a.sched[2] = 0;
      if (a.done_prev) *const_cast<int32_t*>(a.done_prev) = 0;
    }
  }
}

// Segment merge (one CTA per (stream, kv-head) segment, one thread per output
// element): combines the nc chunk partials in chunk order (deterministic),
// writes the attention output and the per-head (max, sum).  Launched right
// after the decode kernel with programmatic dependent launch: its CTAs are
// small, become resident while the decode kernel still runs, and let the next
// layer's decode CTAs launch and prefetch as soon as decode CTAs retire.
// Warp h computes head h's chunk weights and row sum; then thread (h, d)
// accumulates its output element over the chunks with all partial loads of a
// 16-chunk batch in flight (the previous 128-thread version staged every
// partial through shared memory first, serialising the L2 round trips).
template <int D, int G>
__global__ void __launch_bounds__(G * D) merge_kernel(const AttnArgs a) {
  constexpr int PW = D + 2;
  extern __shared__ __align__(16) float msm[];  // [G][nc] weights, [G] sums
  griddep_launch();
  // speculative step: every decode CTA passed its griddepcontrol.wait on the
  // gate grid before this grid could start, so the decision is final here
  if (a.gate && *reinterpret_cast<const volatile int32_t*>(a.gate) != 1) return;
  const int sigma = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nc = a.nc;
  // wait until every chunk partial of this segment is published (decode CTAs
  // are all resident before any merge CTA exists, so the spin completes);
  // segments finish in ticket order, so most merges overlap the streaming of
  // later segments
  if (tid == 0) {
    while (ld_acquire(&a.counters[sigma]) < nc) {
    }
    a.counters[sigma] = 0;  // next launch: incremented only after this grid completes
    if (a.mstamp && sigma == 0) a.mstamp[1] = globaltimer();
  }
  __syncthreads();
  const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
  const float* seg = a.part + (int64_t)sigma * nc * G * PW;
  float* fac = msm;
  // One L2 round trip: every thread issues its output element's partial loads
  // (first kPre chunks) and warp h its head's (m, l) loads together.
  constexpr int kPre = 32;
  const int h = tid / D, d = tid - h * D;
  const float* pp = seg + h * PW + d;
  float x[kPre];
#pragma unroll
  for (int u = 0; u < kPre; ++u) x[u] = u < nc ? __ldcg(pp + u * G * PW) : 0.f;
  if (warp < G) {
    const int hh = warp;
    float mj[4], lj[4];  // nc <= 128 chunks per segment on this path (asserted by the host)
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
      if (a.stats) {
        a.stats[s * a.st_ss + (g * G + hh) * 2] = M;
        a.stats[s * a.st_ss + (g * G + hh) * 2 + 1] = L;
      }
    }
  }
  __syncthreads();
  {
    const float* wf = fac + h * nc;
    float acc = 0.f;
#pragma unroll
    for (int u = 0; u < kPre; ++u)
      if (u < nc) acc = fmaf(wf[u], x[u], acc);
    for (int jj = kPre; jj < nc; ++jj) acc = fmaf(wf[jj], __ldcg(pp + jj * G * PW), acc);
    a.out[s * a.o_ss + (int64_t)(g * G) * D + tid] = acc / fac[G * nc + h];
  }
  // Flag mode only: the last merge CTA publishes completion.  Otherwise the
  // next launch's griddepcontrol.wait on this grid's completion is the
  // release, and the fence + atomic chain (about three L2 round trips) is
  // left off the critical path.
  if (!a.done_self && !a.mstamp) return;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&a.sched[3], 1) == (int)gridDim.x - 1) {
      a.sched[3] = 0;
      __threadfence();
      if (a.done_self) asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(a.done_self), "r"(1) : "memory");
      if (a.mstamp) a.mstamp[2] = globaltimer();
    }
  }
}

__global__ void fold_kernel(const FoldArgs f, int Hq) {
  fold_piece(f, blockIdx.y, blockIdx.x, gridDim.x, Hq, threadIdx.x, blockDim.x);
}

template <int D, int G>
static cudaError_t launch_merge_t(const AttnArgs& a, cudaStream_t st);

template <typename T, int D, int G>
static cudaError_t launch_decode_t(int ctas, const AttnArgs& a, cudaStream_t st) {
  using Sm = Smem<T, D, G>;
  static DevOnce attr;
  if (!attr.here()) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Sm::bytes(1024));
    if (e != cudaSuccess) return e;
    attr.here() = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(Cw<G>::THREADS);
  cfg.dynamicSmemBytes = Sm::bytes(a.Hq);
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, decode_kernel<T, D, G>, a);
  if (e != cudaSuccess) return e;
  return launch_merge_t<D, G>(a, st);
}

template <int D, int G>
static cudaError_t launch_merge_t(const AttnArgs& a, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  // segment merge, also with programmatic dependent launch
  const size_t msmem = (size_t)G * (a.nc + 1) * sizeof(float);
  static DevOnce mattr;
  if (!mattr.here()) {
    e = cudaFuncSetAttribute(merge_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    mattr.here() = true;
  }
  if (msmem > 64 * 1024) return cudaErrorInvalidValue;
  cfg.gridDim = dim3(a.S * a.Hkv);
  cfg.blockDim = dim3(G * D);
  cfg.dynamicSmemBytes = msmem;
  return cudaLaunchKernelEx(&cfg, merge_kernel<D, G>, a);
}

template <typename T, int D, int G>
static int occupancy_t() {
  using Sm = Smem<T, D, G>;
  static int occ_dev[kMaxDevices] = {};
  int& occ = occ_dev[device_slot()];
  if (!occ) {
    cudaFuncSetAttribute(decode_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sm::bytes(1024));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decode_kernel<T, D, G>, Cw<G>::THREADS, Sm::bytes(64)) !=
            cudaSuccess ||
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

int decode_tile_tokens() { return Geo<float, 64>::TT; }

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

// Gate of a speculative host step (launch_spec_gate).  The outputs of the
// step ahead (device staging) go to the host's mapped buffer first, then the
// completion word: the grids ahead happen-before this one and fence.sc.sys is
// cumulative, so a host that reads `done` reads the outputs.  After the
// decision, a GO copies the step's q/k/v from mapped host memory into device
// staging with every thread's loads in flight at once (one PCIe round trip;
// the decode kernels then read L2, not PCIe).
__global__ void __launch_bounds__(256) spec_gate_kernel(SpecGate g) {
  const int tid = threadIdx.x;
  __shared__ int sd;
  // launched early (programmatic dependent launch under the step ahead's
  // merge): its outputs are complete and visible after this wait
  griddep_wait();
  if (g.signal_tick > 0) {
    for (int i = tid; i < g.out_vec; i += blockDim.x) g.out_dst[i] = __ldcg(g.out_src + i);
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
      if (g.dbg) g.dbg[8 * (g.signal_tick & 63) + 2] = globaltimer();
      g.hostw[1] = g.signal_tick;
      __threadfence_system();
    }
  }
  if (g.tick <= 0) return;  // signal only: the end of a speculation chain
  // the gated decode grid may become resident now (its griddepcontrol.wait
  // still waits for this grid to finish)
  griddep_launch();
  if (tid == 0) {
    const unsigned long long t0 = globaltimer();
    if (g.dbg) {
      g.dbg[8 * (g.tick & 63) + 0] = t0;
      g.dbg[8 * (g.tick & 63) + 4] = ~0ull;
      g.dbg[8 * (g.tick & 63) + 5] = 0;
    }
    int d = 0;
    for (;;) {
      if (*reinterpret_cast<volatile int32_t*>(g.broken) == g.gen) { d = 2; break; }
      const int b = g.hostw[0];
      if (b == g.tick) { d = 1; break; }
      if (b < 0 && -b <= g.tick) { d = 2; break; }
      if ((long long)(globaltimer() - t0) > g.timeout_ns) { d = 3; break; }
    }
    *reinterpret_cast<volatile int32_t*>(g.gate) = d;
    if (g.dbg) g.dbg[8 * (g.tick & 63) + 1] = globaltimer();
    if (d == 3) {
      *reinterpret_cast<volatile int32_t*>(g.broken) = g.gen;
      __threadfence_system();
      g.hostw[2] = g.tick;
    }
    sd = d;
  }
  __syncthreads();
  if (sd == 1) {  // every load in flight before the first store: one PCIe round trip
    constexpr int U = 8;
    for (int i0 = 0; i0 < g.in_vec; i0 += U * 256) {
      int4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * 256 + tid;
        if (i < g.in_vec) r[u] = __ldcv(g.in_src + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * 256 + tid;
        if (i < g.in_vec) g.in_dst[i] = r[u];
      }
    }
  }
  if (g.dbg) {
    __syncthreads();
    if (tid == 0) g.dbg[8 * (g.tick & 63) + 3] = globaltimer();
  }
}

cudaError_t launch_spec_gate(const SpecGate& g, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.stream = st;
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, spec_gate_kernel, g);
}

// One row per stream, four columns per thread (fold_vec4).
template <int MODE>
__global__ void __launch_bounds__(256) fold_vec_kernel(const FoldArgs f, int Hq) {
  __shared__ float stt[2 * 256];
  const int s = blockIdx.y;
  const float* sg = f.stats + s * f.st_ss;
  for (int x = threadIdx.x; x < 2 * Hq; x += blockDim.x) stt[x] = (x & 1) ? __frcp_rn(sg[x]) : sg[x];  // (M, 1/L)
  __syncthreads();
  const int j0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (j0 < f.n)
    fold_vec4<MODE>(f.logits + s * f.l_ss, f.l_hs, stt, f.rows + s * f.r_ss, j0, f.n, Hq,
                    (float)(f.agg_div ? f.agg_div : Hq), f.accum);
  if (blockIdx.x == 0 && threadIdx.x == 0 && f.wlen) f.wlen[s * f.w_ss] = f.n;
}

cudaError_t launch_merge(int head_dim, int group, const AttnArgs& a, cudaStream_t st) {
  if (head_dim != 128) return cudaErrorInvalidValue;
  switch (group) {
    case 1: return launch_merge_t<128, 1>(a, st);
    case 2: return launch_merge_t<128, 2>(a, st);
    case 4: return launch_merge_t<128, 4>(a, st);
    case 8: return launch_merge_t<128, 8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fold(int streams, int pieces, const FoldArgs& f, int Hq, cudaStream_t st) {
  if (f.n <= 0) return cudaSuccess;
  const bool vec = f.mode != 2 && Hq <= 256 && f.l_hs % 4 == 0 && f.l_ss % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(f.logits) & 15) == 0;
  if (vec) {
    dim3 grid((f.n + 1023) / 1024, streams);
    if (f.mode == 1)
      fold_vec_kernel<1><<<grid, 256, 0, st>>>(f, Hq);
    else
      fold_vec_kernel<0><<<grid, 256, 0, st>>>(f, Hq);
    return cudaGetLastError();
  }
  dim3 grid(pieces, streams);
  fold_kernel<<<grid, 128, 0, st>>>(f, Hq);
  return cudaGetLastError();
}

}  // namespace skv
