// C ABI + native runtime for the streamkv B200 hot path (see include/streamkv_b200.h).
//
// The context owns every device buffer (allocated once in skv_create; nothing is
// allocated on the hot path) and a host mirror of the per-layer state that is
// uniform across the lock-stepped streams: cached length n, window ring
// head/count, the logit double-buffer parity and the pending (not yet folded)
// window row.  Kernels read everything per-stream from device memory, so a
// recorded CUDA graph of a state-invariant sequence (one eviction period) can be
// replayed indefinitely.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/streamkv_b200.h"
#include "skv_internal.h"

using namespace skv;

// decode tiles (decode_tile_tokens() tokens) per scheduling chunk (SKV_CHUNK_TILES overrides, for tuning)
static int chunk_tiles(int G) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_CHUNK_TILES");
    env = e ? std::max(1, atoi(e)) : 0;
  }
  // 4 tiles (256 tokens) per dynamic chunk: fewer partials and hand-offs per
  // segment than 2 (config 1: 82% -> 86% of the HBM peak; config 4: 87% ->
  // 93%) while the end-of-launch tail stays under one chunk (8+ loses it)
  (void)G;
  return env ? env : 4;
}
static bool chunk_tiles_forced() { return getenv("SKV_CHUNK_TILES") != nullptr; }
constexpr int kStaticMaxTiles = 8;  // largest static chunk (tiles of 64 tokens)
constexpr int kMaxChunks = 128;     // chunks per segment the merge kernel combines
static int q_prefetch() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_QPREFETCH");
    env = e ? atoi(e) : 0;
  }
  return env;
}
static int use_flags() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_FLAGS");
    env = e ? atoi(e) : 0;
  }
  return env;
}
static int use_tc_decode() {  // SKV_TC_DECODE=0 keeps GQA small batches on the CUDA-core kernel
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_TC_DECODE");
    env = e ? atoi(e) : 1;
  }
  return env;
}
// Segments between a segment's early chunks and its last chunk in the dynamic
// ticket order (SKV_LAST_DELAY: -1 automatic = one ticket per CTA later, 0 = all
// last chunks at the end of the launch, > 0 explicit).
static int last_delay_env() {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SKV_LAST_DELAY");
    env = e ? atoi(e) : -1;
  }
  return env;
}
static int use_tc_wide() {  // SKV_TC_WIDE=1: throughput launches on the tensor-core chunk kernel
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_TC_WIDE");
    env = e ? atoi(e) : 0;
  }
  return env;
}
static int use_tcd() {  // SKV_TCD=0: dynamic-schedule launches on the CUDA-core decode kernel
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_TCD");
    env = e ? atoi(e) : 1;
  }
  return env;
}
static int ctas_per_sm_override() {
  const char* e = getenv("SKV_CTAS_PER_SM");
  return e ? std::max(1, atoi(e)) : 0;
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return SKV_ECUDA;
}

#define SKV_CK(call)                                      \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

struct skv_ctx {
  skv_config cfg;
  int S, L, Hq, Hkv, D, G, cap, W, B, elt;
  int Hq_total;  // query heads across all head shards (row mean divisor)
  float scale;
  int max_ctas;    // persistent decode grid bound (CTAs/SM x SMs)
  int last_layer = -1;  // layer of the last decode launch on the ctx (-1: other work since)
  bool layers_chain = false;  // the last launch was an all-layer persistent decode step
  int32_t* lay_cnt = nullptr;  // persistent decode: [S*Hkv] segment chunk counters, [L] layers done, [1] exits
  unsigned long long* lay_tl = nullptr;  // instrumentation: persistent decode timeline (skv_layers_timeline)
  std::map<int, int> cluster_fit;  // (G, chunk tiles, cluster size) -> co-resident clusters
  int launch_seq = 0;   // decode launches (selects the scheduler slot)
  const char* last_kernel = "";  // the last decode launch's kernel (skv_last_decode_kernel)
  int32_t* sched = nullptr;  // [64][4] per-launch ticket / barrier / exit counters
  int32_t* done = nullptr;   // [64] per-launch completion flags
  size_t part_floats = 0;    // one parity half of the double-buffered partials
  // device state
  void* k = nullptr;
  void* v = nullptr;
  int64_t* pos = nullptr;
  int8_t* modality = nullptr;
  int32_t* round_id = nullptr;
  int32_t* len = nullptr;
  int64_t* next_pos = nullptr;
  float* rows = nullptr;
  int32_t* wlen = nullptr;
  int32_t* newlen = nullptr;
  float* logits[2] = {nullptr, nullptr};
  float* stats[2] = {nullptr, nullptr};
  float* part = nullptr;
  int32_t* counters = nullptr;
  float* acc = nullptr;  // heavy-hitter accumulators [S][L][cap] (SKV_POLICY_HEAVY_HITTER)
  // RoPE engines: raw key store (cache.keys()), f64 inverse frequencies, the
  // cache-relative cos/sin table [cap][D/2], rotated q / new-k scratch
  void* kraw = nullptr;
  double* inv_freq = nullptr;
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  void* qr = nullptr;
  void* kr = nullptr;
  void* pqr = nullptr;  // prefill: rotated chunk q / k
  void* pkr = nullptr;
  size_t p_tokens = 0;  // S*C capacity of pqr/pkr
  int32_t* kept = nullptr;
  int32_t* first_moved = nullptr;
  // slot map (see select.cu plan_moves): perm [S][L][cap] logical slot ->
  // physical row; moves [S][L][4 cap] planning scratch + (src, dst, index)
  // triplets; mcount [S][L] rows moved by the last eviction.  Off (dense
  // stable compaction) for cache-relative RoPE, whose moved keys change
  // position anyway.
  bool slotmap = false;
  int32_t* perm = nullptr;
  int32_t* moves = nullptr;
  int32_t* mcount = nullptr;
  float* scores = nullptr;
  int64_t* pos_in = nullptr;  // staging for explicit positions
  // sticky device error word: bit 0 = a chunked prefill saw |v| >= 65504 (its
  // fp16 P.V saturated); reported (and cleared) by skv_sync and every call
  // that returns host data
  int32_t* err_word = nullptr;       // device view of err_host (mapped pinned host memory)
  volatile int32_t* err_host = nullptr;  // read after a synchronisation without a copy
  float* plogits = nullptr;   // prefill: [S][Hq][plg_cap/4][W][4] logits of the recorded rows
  int64_t plg_cap() const { return (cap + 127) / 128 * 128; }
  float* pstats = nullptr;    // prefill: [S][W][Hq][2]
  unsigned long long* tbuf = nullptr;  // timing ring [8192][2]
  unsigned long long* cbuf = nullptr;  // per-CTA timing [64][max_ctas][3]
  int tcount = 0;
  bool timing = false;
  int64_t device_bytes = 0;
  // host mirror (uniform over streams)
  std::vector<int> n, whead, wcount, parity, pend_n, pend_slot, pend_par, round_value;
  // per-(stream, layer) lengths / window rows set by skv_state_inject while a
  // layer's streams disagree (ragged[layer]); the kernels run every stream of
  // a layer in lock step, so a ragged layer refuses work until it is uniform
  std::vector<int> sn, sm;
  std::vector<char> ragged;
  int64_t launches = 0;
  // graphs: host-mirror snapshots at capture begin / end (a replay moves the
  // mirror from `gbegin` to `gend`; it is refused unless the mirror is at `gbegin`)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  struct Mirror {
    std::vector<int> n, whead, wcount, parity, pend_n, pend_slot, pend_par;
    bool operator==(const Mirror& o) const {
      return n == o.n && whead == o.whead && wcount == o.wcount && parity == o.parity && pend_n == o.pend_n &&
             pend_slot == o.pend_slot && pend_par == o.pend_par;
    }
  } gbegin, gend;
  Mirror snap() const { return Mirror{n, whead, wcount, parity, pend_n, pend_slot, pend_par}; }
  void restore(const Mirror& m) {
    n = m.n;
    whead = m.whead;
    wcount = m.wcount;
    parity = m.parity;
    pend_n = m.pend_n;
    pend_slot = m.pend_slot;
    pend_par = m.pend_par;
  }
  // host-buffer pipeline
  cudaStream_t hs[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> ev_in, ev_out;
  cudaEvent_t ev_done = nullptr;
  cudaEvent_t ev_entry = nullptr;  // caller's stream at entry of skv_decode_step_host
  void* stage_q = nullptr;
  void* stage_k = nullptr;
  void* stage_v = nullptr;
  float* stage_out = nullptr;
  std::vector<void*> allocs;
  // host-buffer steps captured as graphs, per engine state (host_step_graph)
  struct HostGraph {
    Mirror pre, post;
    int record = 0, last_layer = -1, post_last_layer = -1, launches = 0;
    bool chain = false, post_chain = false;
    cudaGraph_t graph = nullptr;  // kept: exec updates name its nodes
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t nq = nullptr, nk = nullptr, nv = nullptr, nout = nullptr;
    float* zc_out = nullptr;  // outputs stored straight into this mapped host buffer (no copy node)
  };
  std::vector<HostGraph> hgraphs;
  // speculative host steps (skv_host_speculate): the next token's gate +
  // decode + merge are launched on `st` before the host has its q/k/v; the
  // gate waits for the host's doorbell, so a token costs a PCIe round trip
  // instead of launches plus a stream synchronisation
  struct Spec {
    int on = 0;
    long long timeout_ns = 0;
    volatile int32_t* hostw = nullptr;  // mapped pinned: [0] bell, [1] done, [2] expired
    int32_t* gate = nullptr;            // device [64] decisions, one per step
    int32_t* broken = nullptr;          // device: generation whose chain expired
    char* io = nullptr;                 // mapped pinned: two (q | k | v | out) sets, by tick parity
    char* dio = nullptr;                // device staging: one (q | k | v | out) set
    size_t set_bytes = 0, k_off = 0, v_off = 0, o_off = 0;
    cudaStream_t st = nullptr;
    int tick = 0, gen = 0;
    // the pending (launched, not yet rung) step
    bool pending = false;
    int p_tick = 0, p_record = 0;
    Mirror p_mirror;  // host state before the pending step (restored on cancel)
    int p_launch_seq = 0, p_last_layer = -1, p_tcount = 0;
    int64_t p_launches = 0;
    const char* p_last_kernel = "";
    bool p_chain = false;
    unsigned long long* dbg = nullptr;  // probe (SKV_SPEC_PROF): gate start / go / signalled [64][4]
    int64_t hits = 0, misses = 0;  // steps served from a pending launch / cancelled or expired
  } spec;

  template <typename P>
  cudaError_t alloc(P** p, size_t bytes) {
    void* raw = nullptr;
    cudaError_t e = cudaMalloc(&raw, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) return e;
    allocs.push_back(raw);
    device_bytes += (int64_t)bytes;
    *p = static_cast<P*>(raw);
    return cudaMemset(raw, 0, std::max<size_t>(bytes, 16));
  }

  size_t sl_count() const { return (size_t)S * L; }
  int64_t kv_layer_stride() const { return (int64_t)Hkv * cap * D; }  // elements
  int64_t kv_stream_stride() const { return (int64_t)L * kv_layer_stride(); }

};

namespace skv {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace skv

// A layer whose streams were injected with different lengths / window rows
// cannot run: every kernel takes one length per layer (lock-stepped streams).
static int ragged_fail(const skv_ctx* x, int layer) {
  int s1 = 1;
  while (s1 < x->S && x->sn[(size_t)s1 * x->L + layer] == x->sn[layer] &&
         x->sm[(size_t)s1 * x->L + layer] == x->sm[layer])
    ++s1;
  char buf[256];
  snprintf(buf, sizeof buf,
           "layer %d: streams hold different states (stream 0: n=%d, %d window rows; stream %d: n=%d, %d rows); "
           "the engine runs the streams of a layer in lock step -- inject every stream with the same n and rows",
           layer, x->sn[layer], x->sm[layer], s1, s1 < x->S ? x->sn[(size_t)s1 * x->L + layer] : -1,
           s1 < x->S ? x->sm[(size_t)s1 * x->L + layer] : -1);
  return fail(SKV_ESTATE, buf);
}

// Sticky device errors (skv_ctx::err_word), read with a synchronisation.
static int check_sticky(skv_ctx* x) {
  const int32_t w = *x->err_host;
  if (w == 0) return SKV_OK;
  *x->err_host = 0;
  if (w & (1 << 30))  // (the low bits count prefill V overflows)
    return fail(SKV_ECUDA, "dynamic shared memory base not 1024-byte aligned: a kernel skipped its work");
  return fail(SKV_EINVAL,
              "value overflow: a chunked prefill read |v| >= 65504, which its fp16 P.V cannot represent "
              "(outputs of that chunk are saturated)");
}

extern "C" {

static int spec_cancel(skv_ctx* x);
// every entry point but skv_decode_step_host first retires a pending
// speculative step (its host state would otherwise show through)
#define SPEC_CANCEL(x)                                          \
  do {                                                          \
    const int _src = spec_cancel(const_cast<skv_ctx*>(x));      \
    if (_src) return _src;                                      \
  } while (0)

const char* skv_last_error(void) { return g_err.c_str(); }
int skv_version(void) { return 1; }

int skv_create(const skv_config* cfg, skv_ctx** out) {
  if (!cfg || !out) return fail(SKV_EINVAL, "null argument");
  const skv_config& c = *cfg;
  if (c.streams < 1 || c.layers < 1 || c.heads_q < 1 || c.heads_kv < 1 || c.head_dim < 1)
    return fail(SKV_EINVAL, "layers, heads and head_dim must be positive");
  if (c.head_dim != 64 && c.head_dim != 128) return fail(SKV_EINVAL, "head_dim must be 64 or 128");
  if (c.heads_q % c.heads_kv) return fail(SKV_EINVAL, "heads_q must be a multiple of heads_kv");
  const int G = c.heads_q / c.heads_kv;
  if (G != 1 && G != 2 && G != 4 && G != 8) return fail(SKV_EINVAL, "heads_q/heads_kv must be 1, 2, 4 or 8");
  if (c.dtype != SKV_DTYPE_F32 && c.dtype != SKV_DTYPE_BF16) return fail(SKV_EINVAL, "dtype must be f32 or bf16");
  if (c.recent_len < 1) return fail(SKV_EINVAL, "recent_len must be >= 1");
  if (c.relevant_budget < 0) return fail(SKV_EINVAL, "relevant_budget must be >= 0");
  if (!(c.bias >= 0.f)) return fail(SKV_EINVAL, "bias must be >= 0");
  if (c.window < 1 || c.window > 1024) return fail(SKV_EINVAL, "window capacity must be in [1, 1024]");
  if (c.head_agg != SKV_AGG_MEAN && c.head_agg != SKV_AGG_MAX) return fail(SKV_EINVAL, "unknown head_agg");
  if (c.heads_q_total < 0 || (c.heads_q_total > 0 && c.heads_q_total < c.heads_q))
    return fail(SKV_EINVAL, "heads_q_total must be 0 or >= heads_q");
  // a head shard's max over its own heads cannot be combined by the score sum
  // of the sharded eviction (the reference max runs over all heads,
  // policies.py:263-264)
  if (c.head_agg == SKV_AGG_MAX && c.heads_q_total > c.heads_q)
    return fail(SKV_EINVAL, "head_agg='max' cannot be head-sharded (heads_q_total > heads_q)");
  if (c.capacity < c.recent_len + c.relevant_budget + 1)
    return fail(SKV_EINVAL, "capacity must exceed recent_len + relevant_budget");
  if (c.policy < SKV_POLICY_INF_MLLM || c.policy > SKV_POLICY_NONE) return fail(SKV_EINVAL, "unknown policy");
  if (c.rope_mode < SKV_ROPE_NONE || c.rope_mode > SKV_ROPE_ORIGINAL) return fail(SKV_EINVAL, "unknown rope mode");
  if (c.rope_mode != SKV_ROPE_NONE && !(c.rope_base > 0.f)) return fail(SKV_EINVAL, "rope_base must be > 0");
  // sink_recent_decide: require budget > sink_count >= 0 (policies.py:218-219)
  if (c.policy == SKV_POLICY_SINK_RECENT && !(c.recent_len + c.relevant_budget > c.sink_count && c.sink_count >= 0))
    return fail(SKV_EINVAL, "require budget > sink_count >= 0");

  skv_ctx* x = new skv_ctx();
  x->cfg = c;
  x->S = c.streams;
  x->L = c.layers;
  x->Hq = c.heads_q;
  x->Hq_total = c.heads_q_total > 0 ? c.heads_q_total : c.heads_q;
  x->Hkv = c.heads_kv;
  x->D = c.head_dim;
  x->G = G;
  x->cap = (c.capacity + 31) / 32 * 32;
  x->W = c.window;
  x->B = c.recent_len + c.relevant_budget;
  x->elt = c.dtype == SKV_DTYPE_BF16 ? 2 : 4;
  x->scale = (float)(1.0 / std::sqrt((double)c.head_dim));
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int occ = decode_ctas_per_sm(c.dtype, c.head_dim, G);
    const int ovr = ctas_per_sm_override();
    x->max_ctas = sms * (ovr ? std::min(ovr, occ) : occ);
  }

  const size_t SL = x->sl_count();
  const size_t kv_bytes = SL * (size_t)x->kv_layer_stride() * x->elt;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) {
    if (e == cudaSuccess && r != cudaSuccess) e = r;
  };
  chk(x->alloc(&x->k, kv_bytes));
  chk(x->alloc(&x->v, kv_bytes));
  chk(x->alloc(&x->pos, SL * x->cap * sizeof(int64_t)));
  chk(x->alloc(&x->modality, SL * x->cap));
  chk(x->alloc(&x->round_id, SL * x->cap * sizeof(int32_t)));
  chk(x->alloc(&x->len, SL * sizeof(int32_t)));
  chk(x->alloc(&x->next_pos, SL * sizeof(int64_t)));
  chk(x->alloc(&x->rows, SL * x->W * (size_t)x->cap * sizeof(float)));
  chk(x->alloc(&x->wlen, SL * x->W * sizeof(int32_t)));
  chk(x->alloc(&x->newlen, SL * x->W * sizeof(int32_t)));
  for (int p = 0; p < 2; ++p) {
    chk(x->alloc(&x->logits[p], SL * x->Hq * (size_t)x->cap * sizeof(float)));
    chk(x->alloc(&x->stats[p], SL * x->Hq * 2 * sizeof(float)));
  }
  const int tiles_cap = (x->cap + decode_tile_tokens() - 1) / decode_tile_tokens();
  // chunk partials: at most ceil(tiles / 2) chunks per segment (2-tile static chunks)
  const int min_ch = std::min(2, chunk_tiles(x->G));
  x->part_floats = (size_t)x->S * x->Hkv * ((tiles_cap + min_ch - 1) / min_ch) * x->G * (x->D + 2);
  chk(x->alloc(&x->part, 2 * x->part_floats * sizeof(float)));
  chk(x->alloc(&x->done, 64 * sizeof(int32_t)));
  chk(x->alloc(&x->sched, 64 * 4 * sizeof(int32_t)));
  // [4][S*Hkv]: per-launch slot (seq % 4) -- the merge of launch N+1 may be
  // resident (PDL) before launch N's merge has reset its counters
  chk(x->alloc(&x->counters, (size_t)4 * x->S * x->Hkv * sizeof(int32_t)));
  // all-layer decode counters ([S*Hkv] segments, [L] layer_done, exit), here so
  // that no allocation happens inside a caller's stream capture
  chk(x->alloc(&x->lay_cnt, ((size_t)x->S * x->Hkv + x->L + 1) * sizeof(int32_t)));
  chk(x->alloc(&x->kept, SL * x->B * sizeof(int32_t)));
  chk(x->alloc(&x->first_moved, SL * sizeof(int32_t)));
  chk(x->alloc(&x->scores, SL * x->cap * sizeof(float)));
  chk(x->alloc(&x->pos_in, x->S * sizeof(int64_t)));
  {
    void* h = nullptr;
    chk(cudaHostAlloc(&h, sizeof(int32_t), cudaHostAllocMapped));
    if (h) {
      x->err_host = static_cast<volatile int32_t*>(h);
      *x->err_host = 0;
      chk(cudaHostGetDevicePointer(reinterpret_cast<void**>(&x->err_word), h, 0));
    }
  }
  x->slotmap = c.rope_mode != SKV_ROPE_CACHE_RELATIVE && x->cap <= kMaxMapRows;
  if (x->slotmap) {
    chk(x->alloc(&x->perm, SL * x->cap * sizeof(int32_t)));
    chk(x->alloc(&x->moves, SL * 4 * (size_t)x->cap * sizeof(int32_t)));
    chk(x->alloc(&x->mcount, SL * sizeof(int32_t)));
    if (e == cudaSuccess) chk(launch_iota(x->perm, (int64_t)SL * x->cap, x->cap, nullptr));
    if (e == cudaSuccess) chk(cudaDeviceSynchronize());
  }
  // heavy-hitter accumulators (engine.py:274): one column per cached token
  if (c.policy == SKV_POLICY_HEAVY_HITTER) chk(x->alloc(&x->acc, SL * (size_t)x->cap * sizeof(float)));
  if (c.rope_mode != SKV_ROPE_NONE) {
    const int half = x->D / 2;
    chk(x->alloc(&x->kraw, kv_bytes));
    chk(x->alloc(&x->inv_freq, half * sizeof(double)));
    chk(x->alloc(&x->rope_cos, (size_t)x->cap * half * sizeof(float)));
    chk(x->alloc(&x->rope_sin, (size_t)x->cap * half * sizeof(float)));
    chk(x->alloc(&x->qr, (size_t)x->S * x->Hq * x->D * x->elt));
    chk(x->alloc(&x->kr, (size_t)x->S * x->Hkv * x->D * x->elt));
    if (e == cudaSuccess) {
      // inv_freq = base ** (-2 i / D) and the f32 cos/sin of pos * inv_freq,
      // both in f64 like engine.py:176-178, 200-207; cache-relative positions
      // are slot indices, so the table covers every position that mode uses
      std::vector<double> inv(half);
      for (int i = 0; i < half; ++i) inv[i] = std::pow((double)c.rope_base, -2.0 * i / x->D);
      std::vector<float> tc((size_t)x->cap * half), ts((size_t)x->cap * half);
      for (int p = 0; p < x->cap; ++p)
        for (int i = 0; i < half; ++i) {
          const double ang = (double)p * inv[i];
          tc[(size_t)p * half + i] = (float)std::cos(ang);
          ts[(size_t)p * half + i] = (float)std::sin(ang);
        }
      chk(cudaMemcpy(x->inv_freq, inv.data(), half * sizeof(double), cudaMemcpyHostToDevice));
      chk(cudaMemcpy(x->rope_cos, tc.data(), tc.size() * sizeof(float), cudaMemcpyHostToDevice));
      chk(cudaMemcpy(x->rope_sin, ts.data(), ts.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
  }
  if (e != cudaSuccess) {
    skv_destroy(x);
    return e == cudaErrorMemoryAllocation ? fail(SKV_ENOMEM, "device allocation failed")
                                          : cuda_fail(e, "skv_create");
  }
  x->n.assign(x->L, 0);
  x->whead.assign(x->L, 0);
  x->wcount.assign(x->L, 0);
  x->parity.assign(x->L, 0);
  x->pend_n.assign(x->L, 0);
  x->pend_slot.assign(x->L, 0);
  x->pend_par.assign(x->L, 0);
  x->round_value.assign(x->L, 0);
  x->sn.assign(SL, 0);
  x->sm.assign(SL, 0);
  x->ragged.assign(x->L, 0);
  *out = x;
  return SKV_OK;
}

int skv_destroy(skv_ctx* x) {
  if (!x) return SKV_OK;
  spec_cancel(x);
  cudaDeviceSynchronize();
  if (x->spec.st) cudaStreamDestroy(x->spec.st);
  if (x->spec.hostw) cudaFreeHost(const_cast<int32_t*>(x->spec.hostw));
  if (x->spec.io) cudaFreeHost(x->spec.io);
  for (auto& e : x->hgraphs) {
    cudaGraphExecDestroy(e.exec);
    cudaGraphDestroy(e.graph);
  }
  if (x->exec) cudaGraphExecDestroy(x->exec);
  if (x->graph) cudaGraphDestroy(x->graph);
  for (auto ev : x->ev_in) cudaEventDestroy(ev);
  for (auto ev : x->ev_out) cudaEventDestroy(ev);
  if (x->ev_done) cudaEventDestroy(x->ev_done);
  if (x->ev_entry) cudaEventDestroy(x->ev_entry);
  for (auto s : x->hs)
    if (s) cudaStreamDestroy(s);
  for (void* p : x->allocs) cudaFree(p);
  if (x->err_host) cudaFreeHost(const_cast<int32_t*>(x->err_host));
  delete x;
  return SKV_OK;
}

int64_t skv_device_bytes(const skv_ctx* x) { return x ? x->device_bytes : 0; }
int64_t skv_kernel_launches(const skv_ctx* x) {
  if (!x) return 0;
  spec_cancel(const_cast<skv_ctx*>(x));
  return x->launches;
}

int skv_timing(skv_ctx* x, int enable) {
  SPEC_CANCEL(x);
  if (!x) return fail(SKV_EINVAL, "null argument");
  if (enable) {
    if (!x->tbuf) {
      cudaError_t e = x->alloc(&x->tbuf, 8192 * 2 * sizeof(unsigned long long));
      if (e != cudaSuccess) return cuda_fail(e, "timing buffer");
    }
    std::vector<unsigned long long> init(8192 * 2);
    for (int i = 0; i < 8192; ++i) {
      init[2 * i] = ~0ull;
      init[2 * i + 1] = 0;
    }
    SKV_CK(cudaMemcpy(x->tbuf, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    if (enable == 1 || enable == 3) x->tcount = 0;  // 2: clear values, keep slots (graph replays)
    if (enable == 3 && !x->cbuf) {
      cudaError_t e = x->alloc(&x->cbuf, (size_t)64 * (x->max_ctas + 1) * 8 * sizeof(unsigned long long));
      if (e != cudaSuccess) return cuda_fail(e, "timing buffer");
    }
  }
  x->timing = enable != 0;
  return SKV_OK;
}

const char* skv_last_decode_kernel(const skv_ctx* x) {
  if (!x) return "";
  spec_cancel(const_cast<skv_ctx*>(x));
  return x->last_kernel;
}

int skv_layers_timeline(skv_ctx* x, uint64_t* buf_dev) {
  SPEC_CANCEL(x);
  if (!x) return fail(SKV_EINVAL, "null argument");
  x->lay_tl = reinterpret_cast<unsigned long long*>(buf_dev);
  return SKV_OK;
}

int skv_timing_cta(skv_ctx* x, int slot, uint64_t* out) {
  SPEC_CANCEL(x);
  if (!x || !out || !x->cbuf || slot < 0 || slot >= 64) return fail(SKV_EINVAL, "no per-CTA timing");
  SKV_CK(cudaDeviceSynchronize());
  SKV_CK(cudaMemcpy(out, x->cbuf + (size_t)slot * (x->max_ctas + 1) * 8, (size_t)(x->max_ctas + 1) * 8 * sizeof(uint64_t),
                    cudaMemcpyDeviceToHost));
  return x->max_ctas;
}

int skv_timing_read(skv_ctx* x, uint64_t* out, int max_pairs) {
  SPEC_CANCEL(x);
  if (!x || !out) return fail(SKV_EINVAL, "null argument");
  if (!x->tbuf) return 0;
  const int n = std::min(std::min(x->tcount, 8192), max_pairs);
  SKV_CK(cudaDeviceSynchronize());
  SKV_CK(cudaMemcpy(out, x->tbuf, (size_t)n * 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return n;
}

// ------------------------------------------------------------------ decode --

static RopeArgs rope_base_args(skv_ctx* x) {
  RopeArgs r{};
  r.Hq = x->Hq;
  r.Hkv = x->Hkv;
  r.D = x->D;
  r.mode = x->cfg.rope_mode;
  r.inv_freq = x->inv_freq;
  r.tcos = x->rope_cos;
  r.tsin = x->rope_sin;
  r.tab_rows = x->cfg.rope_mode == SKV_ROPE_CACHE_RELATIVE ? x->cap : 0;
  return r;
}

// Rotated keys of rows [r0 or first[b], r1) from the raw store: every
// (stream, layer) block of layers [l0, l1).
static int rope_rows(skv_ctx* x, int l0, int l1, int r0, int r1, const int32_t* first, cudaStream_t st) {
  RopeRowsArgs rr{};
  rr.ra = rope_base_args(x);
  rr.D = x->D;
  rr.r0 = r0;
  rr.r1 = r1;
  rr.hs = (int64_t)x->cap * x->D;
  const bool all = l0 == 0 && l1 == x->L;
  for (int l = l0; l < (all ? l0 + 1 : l1); ++l) {
    const int64_t off = (int64_t)l * x->kv_layer_stride() * x->elt;
    rr.raw = static_cast<char*>(x->kraw) + off;
    rr.rot = static_cast<char*>(x->k) + off;
    rr.bs = all ? x->kv_layer_stride() : x->kv_stream_stride();
    rr.first = first ? first + (all ? 0 : (int64_t)l * x->S) : nullptr;
    if (x->cfg.rope_mode == SKV_ROPE_ORIGINAL) {
      rr.pos = x->pos + (int64_t)l * x->cap;
      rr.pos_bs = all ? x->cap : (int64_t)x->L * x->cap;
      if (all) rr.pos = x->pos;
    }
    cudaError_t e = launch_rope_rows(x->cfg.dtype, x->Hkv, all ? x->S * x->L : x->S, rr, st);
    if (e != cudaSuccess) return cuda_fail(e, "rope kernel launch");
    x->launches++;
  }
  return SKV_OK;
}

// Where the folded (head-aggregated) row of a recorded step goes: the window
// ring slot (Inf-MLLM), or added into the heavy-hitter accumulator.
static void fold_target(skv_ctx* x, int layer, int slot, FoldArgs& f) {
  if (x->cfg.policy == SKV_POLICY_HEAVY_HITTER) {
    f.rows = x->acc + (int64_t)layer * x->cap;
    f.r_ss = (int64_t)x->L * x->cap;
    f.wlen = nullptr;
    f.accum = 1;
  } else {
    f.rows = x->rows + ((int64_t)layer * x->W + slot) * x->cap;
    f.r_ss = (int64_t)x->L * x->W * x->cap;
    f.wlen = x->wlen + (int64_t)layer * x->W + slot;
    f.w_ss = (int64_t)x->L * x->W;
  }
}

static int last_delay(const skv_ctx* x, int ctas, int nc);

// A decode launch's schedule and arguments for one layer (no kernel of the
// attention itself is launched here; RoPE rotation of q / new k is).
struct DecodePlan {
  AttnArgs a;
  int record, n, nt, ch, nc, ctas, par;
  bool stat, tc, tcd;
};

static int prepare_layer(skv_ctx* x, int layer, const void* q, const void* k, const void* v, const int64_t* pos_dev,
                         float* out, int record, cudaStream_t st, DecodePlan& plan) {
  // Rows feed only the Inf-MLLM window and the heavy-hitter accumulator; the
  // heavy hitter needs every step's row (engine.py:274)
  if (x->cfg.policy == SKV_POLICY_HEAVY_HITTER) record = 1;
  else if (x->cfg.policy != SKV_POLICY_INF_MLLM) record = 0;
  if (x->ragged[layer]) return ragged_fail(x, layer);
  const int n_old = x->n[layer];
  if (n_old + 1 > x->cap)
    return fail(SKV_ESTATE, "cache capacity exceeded: evict before appending more tokens");
  // schedule first: nothing is launched (and no host state moves) unless the
  // whole step can be issued
  const int n = n_old + 1;
  const int nt = (n + decode_tile_tokens() - 1) / decode_tile_tokens();
  // Few segments (batch-1 GQA, small configs): a static schedule with chunks
  // just large enough that every chunk gets its own CTA; its tiles are
  // prefetched under PDL and no CTA idles while another streams a backlog.
  // Otherwise chunk_tiles() tiles per chunk handed out dynamically.  Either
  // way a segment has at most kMaxChunks chunks (the segment merge's limit):
  // long caches get longer chunks.
  const int segs = x->S * x->Hkv;
  int ch = 2;  // static chunks start small (latency-bound: as many CTAs as fit)
  while (ch < kStaticMaxTiles &&
         ((int64_t)segs * ((nt + ch - 1) / ch) > x->max_ctas || (nt + ch - 1) / ch > kMaxChunks))
    ++ch;
  const bool stat = (int64_t)segs * ((nt + ch - 1) / ch) <= x->max_ctas && (nt + ch - 1) / ch <= kMaxChunks &&
                    !chunk_tiles_forced();
  if (!stat) ch = std::max(chunk_tiles(x->G), (nt + kMaxChunks - 1) / kMaxChunks);
  // Throughput launches on the tensor cores (SKV_TC_WIDE): one 2-tile chunk per
  // CTA, three CTAs per SM, as many waves as chunks -- mma.sync does a tile's
  // dot products and P.V in a fraction of the CUDA-core instructions, so the
  // launch stays HBM-bound when the SM clock drops (power cap)
  const bool wide = !stat && use_tc_wide() && x->cfg.dtype == SKV_DTYPE_BF16 && x->D == 128 &&
                    (x->G == 1 || x->G == 2 || x->G == 4) && (nt + 1) / 2 <= kMaxChunks && !chunk_tiles_forced();
  if (wide) ch = 2;
  const int nc = (nt + ch - 1) / ch;
  const int ctas = wide ? segs * nc : std::min(segs * nc, x->max_ctas);
  const void* kraw_in = nullptr;
  if (x->cfg.rope_mode != SKV_ROPE_NONE) {
    // rotate q and the new k at the token's position (engine.py:265-268)
    RopeArgs ra = rope_base_args(x);
    ra.pos0 = n_old;  // cache-relative: the new token's slot
    ra.pos_in = pos_dev;
    ra.next_pos = x->next_pos + layer;
    ra.np_ss = x->L;
    ra.q = q;
    ra.qr = x->qr;
    ra.q_ss = (int64_t)x->Hq * x->D;
    ra.k = k;
    ra.kr = x->kr;
    ra.k_ss = (int64_t)x->Hkv * x->D;
    cudaError_t e = launch_rope_tokens(x->cfg.dtype, 1, x->S, ra, st);
    if (e != cudaSuccess) return cuda_fail(e, "rope kernel launch");
    x->launches++;
    x->last_layer = -1;
    x->layers_chain = false;
    kraw_in = k;
    q = x->qr;
    k = x->kr;
  }
  const int64_t SLstride = (int64_t)x->L;  // stream stride in (stream, layer) units

  AttnArgs a{};
  a.err = x->err_word;
  a.Hq = x->Hq;
  a.Hkv = x->Hkv;
  a.n_old = n_old;
  a.append = 1;
  a.nt = nt;
  a.ch = ch;
  a.qpf = q_prefetch();
  a.late = last_delay(x, ctas, nc);
  a.nc = nc;
  a.S = x->S;
  a.stat = stat || wide;
  const int seq = x->launch_seq++;
  a.sched = x->sched + 4 * (seq % 64);
  a.prefetch = x->last_layer >= 0 && x->last_layer != layer;
  a.done_self = use_flags() ? x->done + (seq % 64) : nullptr;
  a.done_prev = (a.prefetch && use_flags()) ? x->done + ((seq + 63) % 64) : nullptr;
  a.dctas = ctas;
  a.scale = x->scale;
  const int64_t kv_off = (int64_t)layer * x->kv_layer_stride() * x->elt;
  a.kc = static_cast<char*>(x->k) + kv_off;
  a.vc = static_cast<char*>(x->v) + kv_off;
  a.c_ss = x->kv_stream_stride();
  a.c_hs = (int64_t)x->cap * x->D;
  a.q = q;
  a.q_ss = (int64_t)x->Hq * x->D;
  a.kin = k;
  a.vin = v;
  a.in_ss = (int64_t)x->Hkv * x->D;
  if (kraw_in) {
    a.kraw = kraw_in;
    a.kc_raw = static_cast<char*>(x->kraw) + kv_off;
  }
  a.out = out;
  a.o_ss = (int64_t)x->Hq * x->D;
  const int par = x->parity[layer];
  const int64_t lg_sl = (int64_t)x->Hq * x->cap;
  if (record) {
    a.logits = x->logits[par] + (int64_t)layer * lg_sl;
    a.l_ss = SLstride * lg_sl;
    a.l_hs = x->cap;
  }
  a.stats = x->stats[par] + (int64_t)layer * x->Hq * 2;
  a.st_ss = SLstride * x->Hq * 2;
  a.part = x->part + (size_t)(seq & 1) * x->part_floats;
  a.counters = x->counters + (size_t)(seq % 4) * x->S * x->Hkv;
  a.pos = x->pos + (int64_t)layer * x->cap;
  a.modality = x->modality + (int64_t)layer * x->cap;
  a.round_id = x->round_id + (int64_t)layer * x->cap;
  a.m_ss = SLstride * x->cap;
  a.len = x->len + layer;
  a.len_ss = SLstride;
  a.next_pos = x->next_pos + layer;
  a.pos_in = pos_dev;
  a.round_value = x->round_value[layer];
  if (x->timing) {
    if (x->cbuf) {
      a.ctat = x->cbuf + (size_t)(x->tcount % 64) * (x->max_ctas + 1) * 8;
      a.mstamp = a.ctat + (size_t)x->max_ctas * 8;  // extra row: [0, first merge start, last merge end]
    }
    a.tstamp = x->tbuf + 2 * (x->tcount++ % 8192);
  }
  // fold of the pending row (previous recorded step) into its ring slot
  if (x->pend_n[layer] > 0) {
    const int pp = x->pend_par[layer];
    FoldArgs& f = a.fold;
    f.logits = x->logits[pp] + (int64_t)layer * lg_sl;
    f.l_ss = SLstride * lg_sl;
    f.l_hs = x->cap;
    f.stats = x->stats[pp] + (int64_t)layer * x->Hq * 2;
    f.st_ss = SLstride * x->Hq * 2;
    fold_target(x, layer, x->pend_slot[layer], f);
    f.n = x->pend_n[layer];
    f.mode = x->cfg.head_agg == SKV_AGG_MAX ? 1 : 0;
    f.agg_div = x->Hq_total;
  }
  plan.a = a;
  plan.record = record;
  plan.n = n;
  plan.nt = nt;
  plan.ch = ch;
  plan.nc = nc;
  plan.ctas = ctas;
  plan.par = par;
  plan.stat = stat || wide;
  plan.tc = wide || (stat && x->G >= 4 && x->cfg.dtype == SKV_DTYPE_BF16 && x->D == 128 && ch <= 4 && use_tc_decode());
  // dynamic schedule on the tensor cores (decode_tcd_kernel)
  plan.tcd = !plan.tc && !stat && use_tcd() && x->cfg.dtype == SKV_DTYPE_BF16 && x->D == 128 &&
             (x->G == 1 || x->G == 2 || x->G == 4 || x->G == 8);
  if (plan.tc || plan.tcd) {
    plan.a.L = x->L;
    plan.a.layer = layer;
    plan.a.cap = x->cap;
    plan.a.kc_base = x->k;
    plan.a.vc_base = x->v;
    plan.a.total_rows = (int64_t)x->S * x->L * x->Hkv * x->cap;
  }
  return SKV_OK;
}

// Host mirror after a decode of `layer` (uniform over the streams).
static int last_delay(const skv_ctx* x, int ctas, int nc) {
  const int env = last_delay_env();
  if (env >= 0) return env;
  return nc > 1 ? (ctas + nc - 2) / (nc - 1) : 0;  // ~one ticket per CTA
}

static void commit_layer(skv_ctx* x, int layer, const DecodePlan& p) {
  x->pend_n[layer] = 0;
  if (p.record) {
    x->pend_n[layer] = p.n;
    x->pend_slot[layer] = x->whead[layer];
    x->pend_par[layer] = p.par;
    if (x->cfg.policy == SKV_POLICY_INF_MLLM) {  // the heavy hitter accumulates instead of pushing
      x->whead[layer] = (x->whead[layer] + 1) % x->W;
      x->wcount[layer] = std::min(x->wcount[layer] + 1, x->W);
    }
    x->parity[layer] = p.par ^ 1;
  }
  x->n[layer] = p.n;
}

static int decode_layer_impl(skv_ctx* x, int layer, const void* q, const void* k, const void* v,
                             const int64_t* pos_dev, float* out, int record, cudaStream_t st) {
  DecodePlan p;
  int rc = prepare_layer(x, layer, q, k, v, pos_dev, out, record, st, p);
  if (rc) return rc;
  cudaError_t e = p.tc    ? launch_decode_tc(x->G, p.ctas, p.a, st)
                  : p.tcd ? launch_decode_tcd(x->G, p.ctas, p.a, st)
                          : launch_decode(x->cfg.dtype, x->D, x->G, p.ctas, p.a, st);
  if (e != cudaSuccess) return cuda_fail(e, "decode kernel launch");
  x->launches += 2;  // decode + segment merge
  x->last_kernel = p.tc ? "decode_tc_kernel" : p.tcd ? "decode_tcd_kernel" : "decode_kernel";
  x->last_layer = layer;
  x->layers_chain = false;
  commit_layer(x, layer, p);
  return SKV_OK;
}

static int flush_pending(skv_ctx* x, int layer, cudaStream_t st) {
  if (x->pend_n[layer] <= 0) return SKV_OK;
  const int pp = x->pend_par[layer];
  const int64_t lg_sl = (int64_t)x->Hq * x->cap;
  FoldArgs f{};
  f.logits = x->logits[pp] + (int64_t)layer * lg_sl;
  f.l_ss = (int64_t)x->L * lg_sl;
  f.l_hs = x->cap;
  f.stats = x->stats[pp] + (int64_t)layer * x->Hq * 2;
  f.st_ss = (int64_t)x->L * x->Hq * 2;
  fold_target(x, layer, x->pend_slot[layer], f);
  f.n = x->pend_n[layer];
  f.mode = x->cfg.head_agg == SKV_AGG_MAX ? 1 : 0;
  f.agg_div = x->Hq_total;
  const int pieces = std::max(1, std::min(64, (f.n + 255) / 256));
  cudaError_t e = launch_fold(x->S, pieces, f, x->Hq, st);
  if (e != cudaSuccess) return cuda_fail(e, "fold kernel launch");
  x->launches++;
  x->last_layer = -1;
  x->layers_chain = false;
  x->pend_n[layer] = 0;
  return SKV_OK;
}

int skv_prefill_chunk(skv_ctx* x, int layer, const void* q, const void* k, const void* v, int C, int modality,
                      float* out, void* stream) {
  SPEC_CANCEL(x);
  if (!x || !q || !k || !v || !out) return fail(SKV_EINVAL, "null argument");
  if (layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "layer out of range");
  if (x->cfg.dtype != SKV_DTYPE_BF16 || x->D != 128) return fail(SKV_EINVAL, "chunked prefill needs bf16, head_dim 128");
  if (C < 1) return fail(SKV_EINVAL, "chunk must be non-empty");
  if (x->cfg.policy == SKV_POLICY_HEAVY_HITTER)
    return fail(SKV_EINVAL, "the heavy-hitter policy needs every token's row: feed prompts through decode steps");
  if (x->ragged[layer]) return ragged_fail(x, layer);
  const int n0 = x->n[layer];
  if (n0 + C > x->cap) return fail(SKV_ESTATE, "cache capacity exceeded: evict before appending more tokens");
  cudaStream_t st = as_stream(stream);
  int rc = flush_pending(x, layer, st);  // keep the window rows in push order
  if (rc) return rc;
  if (!x->plogits) {
    cudaError_t e = x->alloc(&x->plogits, (size_t)x->S * x->W * x->Hq * x->plg_cap() * sizeof(float));
    if (e == cudaSuccess) e = x->alloc(&x->pstats, (size_t)x->S * x->W * x->Hq * 2 * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "prefill scratch");
  }
  const int units = x->D * x->elt / 16;
  const int64_t SLs = x->L;
  const int64_t kv_off = (int64_t)layer * x->kv_layer_stride() * x->elt;
  const void* kraw_in = nullptr;
  if (x->cfg.rope_mode != SKV_ROPE_NONE) {
    // rotate the chunk's q and k at positions n0 + i (cache-relative) or the
    // original stream positions
    const size_t need = (size_t)x->S * C;
    if (x->p_tokens < need) {
      SKV_CK(cudaStreamSynchronize(st));
      cudaError_t ea = x->alloc(&x->pqr, need * x->Hq * x->D * x->elt);
      if (ea == cudaSuccess) ea = x->alloc(&x->pkr, need * x->Hkv * x->D * x->elt);
      if (ea != cudaSuccess) return cuda_fail(ea, "rope scratch");
      x->p_tokens = need;
    }
    RopeArgs ra = rope_base_args(x);
    ra.pos0 = n0;
    ra.next_pos = x->next_pos + layer;
    ra.np_ss = x->L;
    ra.q = q;
    ra.qr = x->pqr;
    ra.q_ss = (int64_t)C * x->Hq * x->D;
    ra.k = k;
    ra.kr = x->pkr;
    ra.k_ss = (int64_t)C * x->Hkv * x->D;
    cudaError_t er = launch_rope_tokens(x->cfg.dtype, C, x->S, ra, st);
    if (er != cudaSuccess) return cuda_fail(er, "rope kernel launch");
    x->launches++;
    kraw_in = k;
    q = x->pqr;
    k = x->pkr;
  }
  cudaError_t e = launch_append_chunk(k, v, static_cast<char*>(x->k) + kv_off, static_cast<char*>(x->v) + kv_off,
                                      x->kv_stream_stride() * x->elt / 16, (int64_t)x->cap * units, x->S, x->Hkv,
                                      units, n0, C, x->pos + (int64_t)layer * x->cap,
                                      x->modality + (int64_t)layer * x->cap, x->round_id + (int64_t)layer * x->cap,
                                      SLs * x->cap, x->next_pos + layer, x->len + layer, SLs, modality,
                                      x->round_value[layer], st, kraw_in,
                                      kraw_in ? static_cast<char*>(x->kraw) + kv_off : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "append kernel launch");
  // window rows are recorded for the Inf-MLLM policy only (the index-range
  // baselines need none)
  const int wrec = x->cfg.policy == SKV_POLICY_INF_MLLM ? std::min(x->W, C) : 0;
  PrefillArgs a{};
  a.C = C;
  a.n0 = n0;
  a.W = wrec;
  a.Hq = x->Hq;
  a.Hkv = x->Hkv;
  a.G = x->G;
  a.L = x->L;
  a.layer = layer;
  a.cap = x->cap;
  a.scale = x->scale;
  a.out = out;
  a.lg = wrec ? x->plogits : nullptr;
  a.lg_cap = x->plg_cap();
  a.lg_t = 1;
  a.st = wrec ? x->pstats : nullptr;
  a.ovf = x->err_word;  // |v| >= 65504 saturates the fp16 V: sticky error (skv_sync)
  a.meta_len = x->len + layer;  // the chunk's lengths / next positions (after the append read them)
  a.meta_next = x->next_pos + layer;
  a.meta_ss = SLs;
  a.meta_n = n0 + C;
  e = launch_prefill(q, x->S, x->k, x->v, (int64_t)x->S * x->L * x->Hkv * x->cap, a, st);
  if (e != cudaSuccess) return cuda_fail(e, "prefill kernel launch");
  x->launches += 3;
  // fold the recorded rows (oldest first) into the window ring, one launch
  if (wrec > 0) {
    FoldArgs f{};
    f.logits = x->plogits;
    f.l_ss = (int64_t)wrec * x->Hq * x->cap;
    f.l_hs = x->cap;
    f.stats = x->pstats;
    f.st_ss = (int64_t)wrec * x->Hq * 2;
    f.rows = x->rows + (int64_t)layer * x->W * x->cap;
    f.r_ss = SLs * x->W * x->cap;
    f.wlen = x->wlen + (int64_t)layer * x->W;
    f.w_ss = SLs * x->W;
    f.mode = x->cfg.head_agg == SKV_AGG_MAX ? 1 : 0;
    f.agg_div = x->Hq_total;
    e = launch_fold_rows_t(x->S, wrec, f, x->Hq, x->whead[layer], x->W, n0 + C - wrec, x->plg_cap(), x->cap, x->scale, st);
    if (e != cudaSuccess) return cuda_fail(e, "fold kernel launch");
    x->launches++;
  }
  x->whead[layer] = (x->whead[layer] + wrec) % x->W;
  x->wcount[layer] = std::min(x->wcount[layer] + wrec, x->W);
  x->n[layer] = n0 + C;
  x->last_layer = -1;
  x->layers_chain = false;
  return SKV_OK;
}

int skv_decode_layer(skv_ctx* x, int layer, const void* q, const void* k, const void* v,
                     const int64_t* positions_host, float* out, int record, void* stream) {
  SPEC_CANCEL(x);
  if (!x || !q || !k || !v || !out) return fail(SKV_EINVAL, "null argument");
  if (layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "layer out of range");
  cudaStream_t st = as_stream(stream);
  const int64_t* pos_dev = nullptr;
  if (positions_host) {
    // original positions must strictly increase (cache.py:125-126)
    std::vector<int64_t> prev(x->S);
    if (x->n[layer] > 0) {
      for (int s = 0; s < x->S; ++s) {
        SKV_CK(cudaMemcpyAsync(&prev[s], x->pos + ((int64_t)s * x->L + layer) * x->cap + x->n[layer] - 1,
                               sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      }
      SKV_CK(cudaStreamSynchronize(st));
      for (int s = 0; s < x->S; ++s)
        if (positions_host[s] <= prev[s]) return fail(SKV_EINVAL, "original_position must be strictly increasing");
    }
    SKV_CK(cudaMemcpyAsync(x->pos_in, positions_host, x->S * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    SKV_CK(cudaStreamSynchronize(st));
    pos_dev = x->pos_in;
  }
  return decode_layer_impl(x, layer, q, k, v, pos_dev, out, record, st);
}

// All-layer decode steps of latency-bound GQA engines: 1 (default) one
// persistent launch with a cluster per segment; 0 per-layer launches; 2 the
// persistent launch with a last-arriver global merge (A/B only)
static int use_layers_kernel() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_LAYERS");
    env = e ? atoi(e) : 1;
  }
  return env;
}

// All layers of one token in one persistent launch (decode_tc_layers_kernel)
// when every layer is in the same state and its decode would run on the
// static tensor-core schedule (latency-bound GQA steps, config 3).  Returns
// 1 when launched, 0 to fall back to per-layer launches.
// Whether a decode step of every layer may run as one all-layer launch (the
// cluster fit is decided by decode_step_layers itself).
static bool layers_eligible(const skv_ctx* x) {
  if (x->L < 2 || !use_layers_kernel() || x->cfg.rope_mode != SKV_ROPE_NONE || x->timing) return false;
  for (int l = 0; l < x->L; ++l)
    if (x->ragged[l] || x->n[l] != x->n[0] || x->parity[l] != x->parity[0] || x->pend_n[l] != x->pend_n[0] ||
        x->pend_slot[l] != x->pend_slot[0] || x->pend_par[l] != x->pend_par[0] || x->whead[l] != x->whead[0] ||
        x->wcount[l] != x->wcount[0] || x->round_value[l] != x->round_value[0])
      return false;
  return x->G >= 4 && x->cfg.dtype == SKV_DTYPE_BF16 && x->D == 128 && use_tc_decode();
}

// The all-layer launch's counters (allocated outside any stream capture).
static int ensure_layer_counters(skv_ctx* x) {
  if (x->lay_cnt) return SKV_OK;
  cudaError_t e = x->alloc(&x->lay_cnt, ((size_t)x->S * x->Hkv + x->L + 1) * sizeof(int32_t));
  return e == cudaSuccess ? SKV_OK : cuda_fail(e, "layer counters");
}

static int decode_step_layers(skv_ctx* x, const void* q, const void* k, const void* v, float* out, int record,
                              cudaStream_t st) {
  if (!layers_eligible(x)) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  DecodePlan p;
  int rc = prepare_layer(x, 0, q, k, v, nullptr, out, record, st, p);
  if (rc) return rc;
  const int segs = x->S * x->Hkv;
  // cluster variant (default): one cluster of CS <= 16 CTAs per segment,
  // chunks of mt = 4..7 tiles (4..6 at G = 8); all clusters must be co-resident
  // (the smallest chunk whose cluster of CS <= 16 CTAs per segment fits: a
  // GPC must hold a whole cluster, and not every GPC has 16 free SMs)
  int mt = 0, CS = 0;
  bool cluster = false;

  for (int t = 4; t <= (x->G == 4 ? 7 : 6) && use_layers_kernel() == 1 && !cluster; ++t) {
    const int cs = (p.nt + t - 1) / t;
    if (cs > 16 || segs * cs > sms) continue;
    const int key = (x->G * 8 + t) * 32 + cs;
    auto it = x->cluster_fit.find(key);
    if (it == x->cluster_fit.end()) {
      AttnArgs qa = p.a;
      qa.nc = cs;
      qa.ch = t;
      int maxc = 0;
      cudaError_t e = launch_decode_tc_cluster(x->G, t, qa, LayerSteps{}, st, &maxc);
      if (e != cudaSuccess) {
        cudaGetLastError();
        maxc = 0;
      }
      if (getenv("SKV_DEBUG_CLUSTER"))
        fprintf(stderr, "[skv] cluster fit G=%d mt=%d CS=%d segs=%d: %d co-resident clusters (%s)\n", x->G, t, cs,
                segs, maxc, cudaGetErrorString(e));
      it = x->cluster_fit.emplace(key, maxc).first;
    }
    if (it->second >= segs) {
      cluster = true;
      mt = t;
      CS = cs;
    }
  }
  if (!cluster && (!p.tc || p.ctas != segs * p.nc || p.ctas > sms || use_layers_kernel() != 2))
    return 0;  // per-layer launches
  if (!x->lay_cnt) return fail(SKV_ESTATE, "layer counters not allocated");
  LayerSteps ls{};
  ls.L = x->L;
  ls.q_ls = (int64_t)x->S * x->Hq * x->D;
  ls.in_ls = (int64_t)x->S * x->Hkv * x->D;
  ls.o_ls = (int64_t)x->S * x->Hq * x->D;
  ls.kv_ls = x->kv_layer_stride();
  ls.m_ls = x->cap;
  ls.lg_ls = (int64_t)x->Hq * x->cap;
  ls.st_ls = (int64_t)x->Hq * 2;
  ls.fr_ls = x->cfg.policy == SKV_POLICY_HEAVY_HITTER ? x->cap : (int64_t)x->W * x->cap;
  ls.fw_ls = x->W;
  ls.seg_count = x->lay_cnt;
  ls.layer_done = x->lay_cnt + (size_t)x->S * x->Hkv;
  ls.exit_count = ls.layer_done + x->L;
  ls.prefetch0 = x->layers_chain ? 1 : 0;
  ls.tl = x->lay_tl;
  {
    static const int lp = getenv("SKV_LATE_PREFETCH") ? atoi(getenv("SKV_LATE_PREFETCH")) : 0;
    ls.late_prefetch = lp;
  }
  cudaError_t e;
  if (cluster) {
    AttnArgs ca = p.a;
    ca.nc = CS;
    ca.ch = mt;
    e = launch_decode_tc_cluster(x->G, mt, ca, ls, st);
  } else {
    e = launch_decode_tc_layers(x->G, p.ctas, p.a, ls, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "decode (all layers) kernel launch");
  x->launches += 1;
  x->last_kernel = cluster ? "decode_tc_cluster_kernel" : "decode_tc_layers_kernel";
  x->last_layer = -1;
  x->layers_chain = true;
  for (int l = 0; l < x->L; ++l) commit_layer(x, l, p);
  return 1;
}

int skv_decode_step(skv_ctx* x, const void* q, const void* k, const void* v, float* out, int record, void* stream) {
  SPEC_CANCEL(x);
  if (!x || !q || !k || !v || !out) return fail(SKV_EINVAL, "null argument");
  cudaStream_t st = as_stream(stream);
  if (layers_eligible(x)) {
    const int ec = ensure_layer_counters(x);
    if (ec) return ec;
  }
  {
    const int rc = decode_step_layers(x, q, k, v, out, record, st);
    if (rc < 0) return rc;
    if (rc == 1) return SKV_OK;
  }
  const int64_t qb = (int64_t)x->S * x->Hq * x->D * x->elt;
  const int64_t kb = (int64_t)x->S * x->Hkv * x->D * x->elt;
  const int64_t ob = (int64_t)x->S * x->Hq * x->D;
  for (int l = 0; l < x->L; ++l) {
    int rc = decode_layer_impl(x, l, static_cast<const char*>(q) + l * qb, static_cast<const char*>(k) + l * kb,
                               static_cast<const char*>(v) + l * kb, nullptr, out + l * ob, record, st);
    if (rc) return rc;
  }
  return SKV_OK;
}

// SKV_HOST_ZC=0: host steps always stage through device buffers and copies
static bool use_host_zc() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SKV_HOST_ZC");
    env = e ? atoi(e) : 1;
  }
  return env != 0;
}

// pinned host memory the kernels can address directly (UVA: the device
// address of the mapping is the host address)
static bool mapped_host(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost && at.devicePointer == p;
}

static bool pinned_host(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Host-buffer decode step as one CUDA graph: [H2D q, k, v] -> every layer's
// decode -> [D2H out].  Graphs are cached per engine state (a steady-state
// period revisits the same states), and each call only rebinds the four copy
// nodes to the caller's pinned buffers, so a token costs one graph launch
// instead of ~3 runtime calls per layer.  Returns 1 when launched on s_c,
// 0 when not applicable (pageable buffers, SKV_HOST_GRAPHS=0).
static int host_step_graph(skv_ctx* x, const void* q, const void* k, const void* v, float* out, int record,
                           cudaStream_t s_c, int64_t qb, int64_t kb, int64_t ob) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("SKV_HOST_GRAPHS");
    enabled = e ? atoi(e) : 1;
  }
  if (!enabled || x->timing) return 0;
  // large steps (config 1: 10 MB of copies per token) keep the layer-group
  // pipeline, which overlaps their copies with the decode kernels
  if ((qb + 2 * kb + ob) * (int64_t)x->L > (int64_t)2 << 20) return 0;
  // a few layers issue few launches: the eager path is as fast (config 0:
  // 18.2 K vs 17.0 K tokens/s), the graph pays off for deep models (config 3)
  if (x->L < 4) return 0;
  if (!pinned_host(q) || !pinned_host(k) || !pinned_host(v) || !pinned_host(out)) return 0;
  if (layers_eligible(x)) {
    const int ec = ensure_layer_counters(x);
    if (ec) return ec;
  }
  // The kernels store the outputs through the caller's mapped pinned buffer
  // instead of a device staging buffer and a trailing copy node: the PCIe
  // writes overlap the later layers (config 3: 283.6 -> 268.6 us per token).
  float* zc_out = use_host_zc() && mapped_host(out) ? out : nullptr;
  float* dst = zc_out ? zc_out : x->stage_out;
  const skv_ctx::Mirror pre = x->snap();
  skv_ctx::HostGraph* hg = nullptr;
  for (auto& e : x->hgraphs)
    if (e.record == record && e.last_layer == x->last_layer && e.chain == x->layers_chain && e.pre == pre &&
        e.zc_out == zc_out) {
      hg = &e;
      break;
    }
  const size_t L = x->L;
  if (!hg) {
    if (x->hgraphs.size() >= 1024) {  // bounded cache
      for (auto& e : x->hgraphs) {
        cudaGraphExecDestroy(e.exec);
        cudaGraphDestroy(e.graph);
      }
      x->hgraphs.clear();
    }
    skv_ctx::HostGraph ng;
    ng.pre = pre;
    ng.record = record;
    ng.last_layer = x->last_layer;
    ng.chain = x->layers_chain;
    ng.zc_out = zc_out;
    const int launches0 = (int)x->launches;
    SKV_CK(cudaStreamBeginCapture(s_c, cudaStreamCaptureModeThreadLocal));
    int rc = SKV_OK;
    auto ck = [&](cudaError_t e) {
      if (rc == SKV_OK && e != cudaSuccess) rc = cuda_fail(e, "host step capture");
    };
    ck(cudaMemcpyAsync(x->stage_q, q, qb * L, cudaMemcpyHostToDevice, s_c));
    ck(cudaMemcpyAsync(x->stage_k, k, kb * L, cudaMemcpyHostToDevice, s_c));
    ck(cudaMemcpyAsync(x->stage_v, v, kb * L, cudaMemcpyHostToDevice, s_c));
    if (rc == SKV_OK) {  // every layer in one launch where the engine allows it (latency-bound GQA)
      const int lr = decode_step_layers(x, x->stage_q, x->stage_k, x->stage_v, dst, record, s_c);
      if (lr < 0) rc = lr;
      for (int l = 0; lr == 0 && l < x->L && rc == SKV_OK; ++l)
        rc = decode_layer_impl(x, l, static_cast<char*>(x->stage_q) + l * qb, static_cast<char*>(x->stage_k) + l * kb,
                               static_cast<char*>(x->stage_v) + l * kb, nullptr, dst + l * (ob / sizeof(float)),
                               record, s_c);
    }
    if (!zc_out) ck(cudaMemcpyAsync(out, x->stage_out, ob * L, cudaMemcpyDeviceToHost, s_c));
    cudaGraph_t g = nullptr;
    cudaError_t ee = cudaStreamEndCapture(s_c, &g);
    ng.post = x->snap();
    ng.post_last_layer = x->last_layer;
    ng.post_chain = x->layers_chain;
    ng.launches = (int)x->launches - launches0;
    x->restore(pre);
    x->last_layer = ng.last_layer;
    x->layers_chain = ng.chain;
    x->launches = launches0;
    if (rc != SKV_OK || ee != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return rc != SKV_OK ? rc : cuda_fail(ee, "host step capture");
    }
    // the four copy nodes, recognised by their staging side
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    int found = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nd, &t);
      if (t != cudaGraphNodeTypeMemcpy) continue;
      cudaMemcpy3DParms mp{};
      cudaGraphMemcpyNodeGetParams(nd, &mp);
      const void* dst = mp.dstPtr.ptr;
      const void* src = mp.srcPtr.ptr;
      if (dst == x->stage_q) ng.nq = nd, ++found;
      else if (dst == x->stage_k) ng.nk = nd, ++found;
      else if (dst == x->stage_v) ng.nv = nd, ++found;
      else if (src == x->stage_out) ng.nout = nd, ++found;
    }
    cudaError_t ei = found == (zc_out ? 3 : 4) ? cudaGraphInstantiate(&ng.exec, g, 0) : cudaErrorInvalidValue;
    if (ei != cudaSuccess) {
      cudaGraphDestroy(g);
      cudaGetLastError();
      return 0;
    }
    ng.graph = g;
    x->hgraphs.push_back(ng);
    hg = &x->hgraphs.back();
  } else {
    SKV_CK(cudaGraphExecMemcpyNodeSetParams1D(hg->exec, hg->nq, x->stage_q, q, qb * L, cudaMemcpyHostToDevice));
    SKV_CK(cudaGraphExecMemcpyNodeSetParams1D(hg->exec, hg->nk, x->stage_k, k, kb * L, cudaMemcpyHostToDevice));
    SKV_CK(cudaGraphExecMemcpyNodeSetParams1D(hg->exec, hg->nv, x->stage_v, v, kb * L, cudaMemcpyHostToDevice));
    if (!zc_out)
      SKV_CK(cudaGraphExecMemcpyNodeSetParams1D(hg->exec, hg->nout, out, x->stage_out, ob * L, cudaMemcpyDeviceToHost));
  }
  SKV_CK(cudaGraphLaunch(hg->exec, s_c));
  x->restore(hg->post);
  x->last_layer = hg->post_last_layer;
  x->layers_chain = hg->post_chain;
  x->launches += hg->launches;
  return 1;
}

// ---------------------------------------------------------------------------
// Speculative host steps (skv_host_speculate).  Shallow engines (config 0) at
// batch 1 are bound by the host: two launches and a stream synchronisation
// cost more than the step.  Instead, the next token's launches wait on the
// device behind a one-thread gate kernel polling a doorbell in mapped pinned
// memory; a call copies the caller's q/k/v into the engine's mapped input set,
// rings the bell, launches the token after it (whose gate first reports this
// one's completion), spins on the done word and copies the outputs out.  The
// launches are planned with the host state advanced as if the call had come
// with the same `record` flag; any other call (a different flag, or any other
// entry point) cancels the pending step: its kernels exit before touching any
// state and the host state goes back.  A gate that is not rung within the
// timeout expires the same way, so nothing waits on the host for long.
struct SpecSnap {
  skv_ctx::Mirror m;
  int launch_seq, last_layer, tcount;
  int64_t launches;
  const char* last_kernel;
  bool chain;
};
static SpecSnap spec_snap(const skv_ctx* x) {
  return SpecSnap{x->snap(), x->launch_seq, x->last_layer, x->tcount, x->launches, x->last_kernel, x->layers_chain};
}
static void spec_back(skv_ctx* x, const SpecSnap& s) {
  x->restore(s.m);
  x->launch_seq = s.launch_seq;
  x->last_layer = s.last_layer;
  x->tcount = s.tcount;
  x->launches = s.launches;
  x->last_kernel = s.last_kernel;
  x->layers_chain = s.chain;
}
// host state before the pending step
static void spec_set_before(skv_ctx* x, const SpecSnap& b) {
  auto& p = x->spec;
  p.p_mirror = b.m;
  p.p_launch_seq = b.launch_seq;
  p.p_last_layer = b.last_layer;
  p.p_tcount = b.tcount;
  p.p_launches = b.launches;
  p.p_last_kernel = b.last_kernel;
  p.p_chain = b.chain;
}
static SpecSnap spec_before(const skv_ctx* x) {
  const auto& p = x->spec;
  return SpecSnap{p.p_mirror, p.p_launch_seq, p.p_last_layer, p.p_tcount, p.p_launches, p.p_last_kernel, p.p_chain};
}

// the pending step's kernels are drained (they exit without side effects),
// the bell is cleared for the next chain, the host state goes back
static int spec_drain(skv_ctx* x, int bell) {
  auto& p = x->spec;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  p.hostw[0] = bell;
  p.pending = false;
  p.misses++;
  spec_back(x, spec_before(x));
  SKV_CK(cudaStreamSynchronize(p.st));
  p.hostw[0] = 0;
  p.gen++;
  return SKV_OK;
}

static int spec_cancel(skv_ctx* x) {
  if (!x || !x->spec.pending) return SKV_OK;
  return spec_drain(x, -x->spec.p_tick);
}

static bool spec_room(const skv_ctx* x) {
  for (int l = 0; l < x->L; ++l)
    if (x->ragged[l] || x->n[l] + 1 > x->cap) return false;
  return true;
}

static SpecGate spec_gate_args(skv_ctx* x, int signal_tick, int tick, int32_t* gate) {
  auto& p = x->spec;
  SpecGate g{};
  g.hostw = p.hostw;
  g.gate = gate;
  g.broken = p.broken;
  g.signal_tick = signal_tick;
  g.tick = tick;
  g.gen = p.gen;
  g.timeout_ns = p.timeout_ns;
  g.in_src = reinterpret_cast<const int4*>(p.io + (size_t)(tick & 1) * p.set_bytes);
  g.in_dst = reinterpret_cast<int4*>(p.dio);
  g.in_vec = (int)(p.o_off / 16);
  // (measured: the merge storing the outputs into mapped memory itself is
  // slower -- 7.2 vs 4.7 us from the last decode CTA to the done word)
  g.out_src = reinterpret_cast<const int4*>(p.dio + p.o_off);
  g.out_dst = reinterpret_cast<int4*>(p.io + (size_t)(signal_tick & 1) * p.set_bytes + p.o_off);
  g.out_vec = (int)((p.set_bytes - p.o_off) / 16);
  g.dbg = p.dbg;
  return g;
}

// Gate + every layer of step `tick` on spec.st, planned from the current host
// state (advanced on success).  Returns 1 launched, 0 not eligible (nothing
// left enqueued), < 0 error.
static int spec_launch(skv_ctx* x, int record, int signal_tick) {
  auto& p = x->spec;
  const int64_t qb = (int64_t)x->S * x->Hq * x->D * x->elt;
  const int64_t kb = (int64_t)x->S * x->Hkv * x->D * x->elt;
  const int64_t ob = (int64_t)x->S * x->Hq * x->D;
  const int tick = ++p.tick;
  const SpecSnap before = spec_snap(x);
  int32_t* gate = p.gate + (tick % 64);
  cudaError_t e = launch_spec_gate(spec_gate_args(x, signal_tick, tick, gate), p.st);
  if (e != cudaSuccess) return cuda_fail(e, "speculative gate launch");
  x->launches++;
  char* set = p.dio;
  for (int l = 0; l < x->L; ++l) {
    DecodePlan pl;
    int rc = prepare_layer(x, l, set + l * qb, set + p.k_off + l * kb, set + p.v_off + l * kb, nullptr,
                           reinterpret_cast<float*>(set + p.o_off) + l * ob, record, p.st, pl);
    if (rc == SKV_OK && (pl.tc || pl.tcd)) {  // tensor-core plans are not gated: not eligible
      p.on = 0;
      rc = 1;
    }
    if (rc == SKV_OK) {
      pl.a.gate = gate;
      if (p.dbg) pl.a.tstamp = p.dbg + 8 * (tick & 63) + 4;
      e = launch_decode(x->cfg.dtype, x->D, x->G, pl.ctas, pl.a, p.st);
      if (e != cudaSuccess) rc = cuda_fail(e, "speculative decode launch");
    }
    if (rc != SKV_OK) {  // the launched part is cancelled and drained
      spec_set_before(x, before);
      p.pending = true;
      p.p_tick = tick;
      const int drc = spec_drain(x, -tick);
      p.misses--;
      if (drc) return drc;
      return rc < 0 ? rc : 0;
    }
    x->launches += 2;
    x->last_kernel = "decode_kernel";
    x->last_layer = l;
    x->layers_chain = false;
    commit_layer(x, l, pl);
  }
  spec_set_before(x, before);
  p.pending = true;
  p.p_tick = tick;
  p.p_record = record;
  return 1;
}

// Returns 1 when the step was served (outputs in `out`), 0 when the caller
// should run the regular path, < 0 on error.
static int spec_step(skv_ctx* x, const void* q, const void* k, const void* v, float* out, int record,
                     cudaStream_t caller) {
  auto& p = x->spec;
  const int64_t qb = (int64_t)x->S * x->Hq * x->D * x->elt * x->L;
  const int64_t kb = (int64_t)x->S * x->Hkv * x->D * x->elt * x->L;
  const int64_t ob = (int64_t)x->S * x->Hq * x->D * sizeof(float) * x->L;
  if (p.pending && p.p_record != record) {
    const int rc = spec_cancel(x);
    if (rc) return rc;
  }
  if (!p.pending) {
    if (!spec_room(x)) return 0;
    // the first step of a chain is ordered after the caller's work
    SKV_CK(cudaEventRecord(x->ev_entry, caller));
    SKV_CK(cudaStreamWaitEvent(p.st, x->ev_entry, 0));
    const int rc = spec_launch(x, record, 0);
    if (rc <= 0) return rc;
  }
  static const bool prof = getenv("SKV_SPEC_PROF") != nullptr;  // probe: per-phase host times
  static double acc[4] = {0, 0, 0, 0};
  static int64_t cnt = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto p0 = now();
  const int t = p.p_tick;
  const SpecSnap before_t = spec_before(x);
  char* set = p.io + (size_t)(t & 1) * p.set_bytes;
  std::memcpy(set, q, qb);
  std::memcpy(set + p.k_off, k, kb);
  std::memcpy(set + p.v_off, v, kb);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  p.hostw[0] = t;  // ring: the gate releases step t
  p.pending = false;
  const auto p1 = now();
  // the next step goes in under this one's device time; its gate reports t
  int rc = spec_room(x) ? spec_launch(x, record, t) : 0;
  if (rc < 0) return rc;
  if (rc == 0) {
    cudaError_t e = launch_spec_gate(spec_gate_args(x, t, 0, p.gate + ((t + 1) % 64)), p.st);
    if (e != cudaSuccess) return cuda_fail(e, "speculative gate launch");
    x->launches++;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const auto p2 = t0;
  for (uint32_t spin = 1;; ++spin) {
    if (p.hostw[1] == t) break;
    if ((spin & 4095) == 0) {
      cudaError_t e = cudaStreamQuery(p.st);
      if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_fail(e, "speculative step");
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10))
        return fail(SKV_ECUDA, "speculative step did not complete within 10 s");
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (p.hostw[2] == t) {
    // step t expired before the bell: nothing of it ran; the step after it
    // (if launched) is cancelled by the broken chain
    if (p.pending) {
      const int drc = spec_drain(x, -p.p_tick);
      if (drc) return drc;
    } else {
      SKV_CK(cudaStreamSynchronize(p.st));
      p.hostw[0] = 0;
      p.gen++;
      p.misses++;
    }
    spec_back(x, before_t);
    return 0;
  }
  std::memcpy(out, set + p.o_off, ob);
  p.hits++;
  if (prof) {
    const auto p3 = now();
    acc[0] += std::chrono::duration<double, std::micro>(p1 - p0).count();
    acc[1] += std::chrono::duration<double, std::micro>(p2 - p1).count();
    acc[2] += std::chrono::duration<double, std::micro>(p3 - p2).count();
    if (p.dbg && cnt % 2048 == 2047) {  // the last 64 ticks' device timeline (device memory: no PCIe skew)
      std::vector<unsigned long long> h(64 * 8);
      cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
      double d[5] = {0, 0, 0, 0, 0};
      int m = 0;
      for (int i = 0; i < 64; ++i) {
        const unsigned long long* d0 = h.data() + 8 * i;
        if (!d0[2] || !d0[5] || d0[2] < d0[5] || d0[4] < d0[3]) continue;
        d[0] += (double)(d0[3] - d0[1]) * 1e-3;  // go -> inputs staged
        d[1] += (double)(d0[4] - d0[3]) * 1e-3;  // -> first decode CTA
        d[2] += (double)(d0[5] - d0[4]) * 1e-3;  // decode span
        d[3] += (double)(d0[2] - d0[5]) * 1e-3;  // last decode CTA -> signalled (merge, gate, copy out)
        d[4] += (double)(d0[2] - d0[1]) * 1e-3;
        ++m;
      }
      if (m)
        fprintf(stderr, "device (%d ticks): go->staged %.2f, ->decode start %.2f, decode %.2f, ->signal %.2f, go->signal %.2f us\n",
                m, d[0] / m, d[1] / m, d[2] / m, d[3] / m, d[4] / m);
    }
    if (++cnt % 2048 == 0)
      fprintf(stderr, "spec step: copy+ring %.2f us, launch next %.2f us, wait+copy out %.2f us; device go->signal %.2f us\n",
              acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt);
  }
  return 1;
}

int skv_host_speculate(skv_ctx* x, int enable, int timeout_us) {
  if (!x) return fail(SKV_EINVAL, "null context");
  SPEC_CANCEL(x);
  auto& p = x->spec;
  if (!enable) {
    p.on = 0;
    return SKV_OK;
  }
  if (timeout_us <= 0) return fail(SKV_EINVAL, "timeout_us must be > 0");
  if (x->L > 2 || x->cfg.rope_mode != SKV_ROPE_NONE)
    return fail(SKV_EINVAL, "speculative host steps serve shallow (<= 2 layers) engines without RoPE");
  if (!p.hostw) {
    void* hw = nullptr;
    SKV_CK(cudaHostAlloc(&hw, 64, cudaHostAllocMapped));
    std::memset(hw, 0, 64);
    p.hostw = static_cast<volatile int32_t*>(hw);
    cudaError_t e = x->alloc(&p.gate, 64 * sizeof(int32_t));
    if (e == cudaSuccess) e = x->alloc(&p.broken, sizeof(int32_t));
    if (e != cudaSuccess) return cuda_fail(e, "speculation state");
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t qb = (size_t)x->S * x->Hq * x->D * x->elt * x->L;
    const size_t kb = (size_t)x->S * x->Hkv * x->D * x->elt * x->L;
    const size_t ob = (size_t)x->S * x->Hq * x->D * sizeof(float) * x->L;
    p.k_off = up(qb);
    p.v_off = p.k_off + up(kb);
    p.o_off = p.v_off + up(kb);
    p.set_bytes = p.o_off + up(ob);
    void* io = nullptr;
    SKV_CK(cudaHostAlloc(&io, 2 * p.set_bytes, cudaHostAllocMapped));
    std::memset(io, 0, 2 * p.set_bytes);
    p.io = static_cast<char*>(io);
    if (cudaError_t e2 = x->alloc(&p.dio, p.set_bytes)) return cuda_fail(e2, "speculation staging");
    SKV_CK(cudaStreamCreateWithFlags(&p.st, cudaStreamNonBlocking));
    p.gen = 1;
    if (getenv("SKV_SPEC_PROF")) {
      if (cudaError_t e3 = x->alloc(&p.dbg, 64 * 8 * sizeof(unsigned long long))) return cuda_fail(e3, "probe");
    }
  }
  p.timeout_ns = (long long)timeout_us * 1000;
  p.on = 1;
  return SKV_OK;
}

int skv_host_speculate_stats(skv_ctx* x, int64_t* hits, int64_t* misses) {
  if (!x) return fail(SKV_EINVAL, "null context");
  if (hits) *hits = x->spec.hits;
  if (misses) *misses = x->spec.misses;
  return SKV_OK;
}

int skv_decode_step_host(skv_ctx* x, const void* q, const void* k, const void* v, float* out, int record,
                         void* stream) {
  if (!x || !q || !k || !v || !out) return fail(SKV_EINVAL, "null argument");
  const int64_t qb = (int64_t)x->S * x->Hq * x->D * x->elt;
  const int64_t kb = (int64_t)x->S * x->Hkv * x->D * x->elt;
  const int64_t ob = (int64_t)x->S * x->Hq * x->D * sizeof(float);
  if (!x->stage_q) {
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t r) {
      if (e == cudaSuccess && r != cudaSuccess) e = r;
    };
    chk(x->alloc(&x->stage_q, qb * x->L));
    chk(x->alloc(&x->stage_k, kb * x->L));
    chk(x->alloc(&x->stage_v, kb * x->L));
    chk(x->alloc(&x->stage_out, ob * x->L));
    for (auto& s : x->hs) chk(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    x->ev_in.resize(x->L);
    x->ev_out.resize(x->L);
    for (int l = 0; l < x->L; ++l) {
      chk(cudaEventCreateWithFlags(&x->ev_in[l], cudaEventDisableTiming));
      chk(cudaEventCreateWithFlags(&x->ev_out[l], cudaEventDisableTiming));
    }
    chk(cudaEventCreateWithFlags(&x->ev_done, cudaEventDisableTiming));
    chk(cudaEventCreateWithFlags(&x->ev_entry, cudaEventDisableTiming));
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline setup");
  }
  if (x->spec.on && x->L <= 2 && !x->timing) {
    const int rc = spec_step(x, q, k, v, out, record, as_stream(stream));
    if (rc < 0) return rc;
    if (rc == 1) return check_sticky(x);
  } else {
    SPEC_CANCEL(x);
  }
  if (x->L <= 2) {
    cudaStream_t sc = as_stream(stream);  // (ordered after the caller's work: no event)
    // shallow models (config 0): the whole token on the caller's stream -- the
    // layers' launches reading q/k/v and storing the outputs through the
    // caller's mapped pinned buffers (a few KB: no copy operations), or copies
    // in and out around them; one synchronisation
    const bool zc = use_host_zc() && mapped_host(q) && mapped_host(k) && mapped_host(v) && mapped_host(out);
    const char* qs = static_cast<const char*>(zc ? q : x->stage_q);
    const char* ks = static_cast<const char*>(zc ? k : x->stage_k);
    const char* vs = static_cast<const char*>(zc ? v : x->stage_v);
    float* os = zc ? out : x->stage_out;
    if (!zc) {
      SKV_CK(cudaMemcpyAsync(x->stage_q, q, qb * x->L, cudaMemcpyHostToDevice, sc));
      SKV_CK(cudaMemcpyAsync(x->stage_k, k, kb * x->L, cudaMemcpyHostToDevice, sc));
      SKV_CK(cudaMemcpyAsync(x->stage_v, v, kb * x->L, cudaMemcpyHostToDevice, sc));
    }
    for (int l = 0; l < x->L; ++l) {
      const int rc = decode_layer_impl(x, l, qs + l * qb, ks + l * kb, vs + l * kb, nullptr,
                                       os + l * (ob / sizeof(float)), record, sc);
      if (rc) return rc;
    }
    if (!zc) SKV_CK(cudaMemcpyAsync(out, x->stage_out, ob * x->L, cudaMemcpyDeviceToHost, sc));
    SKV_CK(cudaStreamSynchronize(sc));
    return check_sticky(x);
  }
  cudaStream_t s_in = x->hs[0], s_c = x->hs[1], s_out = x->hs[2];
  // work the caller enqueued before this call (an eviction, a prefill chunk,
  // a state injection) completes before the pipeline reads or writes the cache
  SKV_CK(cudaEventRecord(x->ev_entry, as_stream(stream)));
  SKV_CK(cudaStreamWaitEvent(s_in, x->ev_entry, 0));
  SKV_CK(cudaStreamWaitEvent(s_c, x->ev_entry, 0));
  {
    const int rc = host_step_graph(x, q, k, v, out, record, s_c, qb, kb, ob);
    if (rc < 0) return rc;
    if (rc == 1) {
      SKV_CK(cudaStreamSynchronize(s_c));
      return check_sticky(x);
    }
  }
  if (layers_eligible(x)) {
    // all layers in one launch (decode_step_layers): whole-token copies around it
    const int ec = ensure_layer_counters(x);
    if (ec) return ec;
    SKV_CK(cudaMemcpyAsync(x->stage_q, q, qb * x->L, cudaMemcpyHostToDevice, s_c));
    SKV_CK(cudaMemcpyAsync(x->stage_k, k, kb * x->L, cudaMemcpyHostToDevice, s_c));
    SKV_CK(cudaMemcpyAsync(x->stage_v, v, kb * x->L, cudaMemcpyHostToDevice, s_c));
    const int lr = decode_step_layers(x, x->stage_q, x->stage_k, x->stage_v, x->stage_out, record, s_c);
    if (lr < 0) return lr;
    for (int l = 0; lr == 0 && l < x->L; ++l) {  // the clusters do not fit: per-layer launches
      const int rc = decode_layer_impl(x, l, static_cast<char*>(x->stage_q) + l * qb,
                                       static_cast<char*>(x->stage_k) + l * kb, static_cast<char*>(x->stage_v) + l * kb,
                                       nullptr, x->stage_out + l * (ob / sizeof(float)), record, s_c);
      if (rc) return rc;
    }
    SKV_CK(cudaMemcpyAsync(out, x->stage_out, ob * x->L, cudaMemcpyDeviceToHost, s_c));
    SKV_CK(cudaStreamSynchronize(s_c));
    return check_sticky(x);
  }
  // Layers in groups: one copy per tensor and group in, one out, so the copies
  // of group i+1 / i-1 overlap group i's kernels while the host issues few
  // runtime calls per token.  The first and the last group are one layer each:
  // only layer 0's inputs and layer L-1's outputs cross PCIe unoverlapped.
  static int ngroups = -1;  // SKV_HOST_GROUPS overrides the group count
  if (ngroups < 0) {
    const char* e = getenv("SKV_HOST_GROUPS");
    ngroups = e ? std::max(1, atoi(e)) : 4;
  }
  int bounds[66];
  int nb = 0;
  {
    const int g = std::min(ngroups, std::min(x->L, 64));
    bounds[nb++] = 0;
    if (g >= 3) {
      const int mid = x->L - 2, gm = g - 2;
      bounds[nb++] = 1;
      for (int i = 1; i <= gm; ++i) bounds[nb++] = 1 + (int)((int64_t)mid * i / gm);
      bounds[nb++] = x->L;
    } else {
      for (int i = 1; i <= g; ++i) bounds[nb++] = (int)((int64_t)x->L * i / g);
    }
  }
  for (int b = 0; b + 1 < nb; ++b) {
    const int l0 = bounds[b], nl = bounds[b + 1] - l0;
    if (nl <= 0) continue;
    SKV_CK(cudaMemcpyAsync(static_cast<char*>(x->stage_q) + l0 * qb, static_cast<const char*>(q) + l0 * qb, nl * qb,
                           cudaMemcpyHostToDevice, s_in));
    SKV_CK(cudaMemcpyAsync(static_cast<char*>(x->stage_k) + l0 * kb, static_cast<const char*>(k) + l0 * kb, nl * kb,
                           cudaMemcpyHostToDevice, s_in));
    SKV_CK(cudaMemcpyAsync(static_cast<char*>(x->stage_v) + l0 * kb, static_cast<const char*>(v) + l0 * kb, nl * kb,
                           cudaMemcpyHostToDevice, s_in));
    SKV_CK(cudaEventRecord(x->ev_in[l0], s_in));
    SKV_CK(cudaStreamWaitEvent(s_c, x->ev_in[l0], 0));
    for (int l = l0; l < l0 + nl; ++l) {
      int rc = decode_layer_impl(x, l, static_cast<char*>(x->stage_q) + l * qb, static_cast<char*>(x->stage_k) + l * kb,
                                 static_cast<char*>(x->stage_v) + l * kb, nullptr,
                                 x->stage_out + l * (ob / sizeof(float)), record, s_c);
      if (rc) return rc;
    }
    SKV_CK(cudaEventRecord(x->ev_out[l0], s_c));
    SKV_CK(cudaStreamWaitEvent(s_out, x->ev_out[l0], 0));
    SKV_CK(cudaMemcpyAsync(reinterpret_cast<char*>(out) + l0 * ob, x->stage_out + l0 * (ob / sizeof(float)), nl * ob,
                           cudaMemcpyDeviceToHost, s_out));
  }
  SKV_CK(cudaStreamSynchronize(s_out));
  SKV_CK(cudaStreamSynchronize(s_c));
  return check_sticky(x);
}

// ------------------------------------------------------------------- evict --

// mode 0: decide + compact; 1: write unbiased window-mean scores only (head-sharded
// partials, [S][L'][cap]); 2: decide from given scores (+bias) + compact.
static int evict_layers(skv_ctx* x, int l0, int l1, int32_t* kept_dev, int kept_ld, int kept_off, cudaStream_t st,
                        int mode = 0, float* scores_io = nullptr, int scores_ld = 0, int scores_off = 0) {
  // all layers in [l0, l1) share n / ring state (checked by caller)
  const int nl = l1 - l0;
  const int n = x->n[l0];
  const int m = n > x->B ? x->B : n;
  const bool all = (l0 == 0 && l1 == x->L);
  // block b enumerates (s, layer): contiguous when all layers are evicted together
  SelectArgs a{};
  a.row_stride = x->cap;
  a.ring_head = x->whead[l0];
  a.count = x->wcount[l0];
  a.W = x->W;
  a.n = n;
  a.l = x->cfg.recent_len;
  a.r = x->cfg.relevant_budget;
  a.bias = x->cfg.bias;
  a.apply_bias = mode == 1 ? 0 : 1;
  a.scores_only = mode == 1;
  a.pad = x->B;
  a.policy = x->cfg.policy;
  a.sink = x->cfg.sink_count;
  if (mode == 1 && n <= x->B) return SKV_OK;  // keep-all decision: nothing to score
  CompactArgs c{};
  c.heads = x->Hkv;
  c.row_bytes = x->D * x->elt;
  c.kv_hs = (int64_t)x->cap * x->D * x->elt;
  c.row_stride = x->cap;
  c.W = x->W;
  c.m = m;
  if (all) {
    a.rows = x->rows;
    a.r_bs = (int64_t)x->W * x->cap;
    a.wlen = x->wlen;
    a.w_bs = x->W;
    a.kept32 = x->kept;
    a.k_bs = x->B;
    a.scores = mode == 1 ? scores_io : x->scores;
    a.s_bs = x->cap;
    if (mode == 2) {
      a.scores_in = scores_io;
      a.si_bs = x->cap;
    }
    a.first_moved = x->first_moved;
    a.newlen = x->newlen;
    a.acc = x->acc;
    a.acc_bs = x->cap;
    if (x->slotmap) {
      a.perm = x->perm;
      a.pm_bs = x->cap;
      if (mode != 1) {
        a.moves = x->moves;
        a.mv_bs = 4 * (int64_t)x->cap;
        a.mcount = x->mcount;
        a.mc_bs = 1;
      }
    }
    cudaError_t e = launch_select(x->S * x->L, a, st);
    if (e != cudaSuccess) return cuda_fail(e, "select kernel launch");
    x->launches++;
    x->last_layer = -1;
    x->layers_chain = false;
    if (mode == 1) return SKV_OK;
    c.k = static_cast<char*>(x->k);
    c.v = static_cast<char*>(x->v);
    c.kv_bs = x->kv_layer_stride() * x->elt;
    c.pos = x->pos;
    c.modality = x->modality;
    c.round_id = x->round_id;
    c.m_bs = x->cap;
    c.rows = x->rows;
    c.r_bs = (int64_t)x->W * x->cap;
    c.wlen = x->wlen;
    c.newlen = x->newlen;
    c.w_bs = x->W;
    c.kept32 = x->kept;
    c.k_bs = x->B;
    c.first_moved = x->first_moved;
    c.len = x->len;
    c.len_bs = 1;
    c.acc = x->acc;
    c.acc_bs = x->cap;
    c.k_raw = static_cast<char*>(x->kraw);
    c.rope_cr = x->cfg.rope_mode == SKV_ROPE_CACHE_RELATIVE;
    if (x->slotmap) {
      c.moves = x->moves;
      c.mv_bs = 4 * (int64_t)x->cap;
      c.mcount = x->mcount;
      c.mc_bs = 1;
    }
    e = launch_compact(x->S * x->L, c, st);
    if (e != cudaSuccess) return cuda_fail(e, "compact kernel launch");
    x->launches++;
    x->last_layer = -1;
    x->layers_chain = false;
    if (c.rope_cr) {  // _refresh_rotations (engine.py:339-342): moved keys at their new slots
      int rc = rope_rows(x, 0, x->L, 0, m, x->first_moved, st);
      if (rc) return rc;
    }
  } else {
    for (int l = l0; l < l1; ++l) {
      const int64_t sl0 = l;  // block b = stream s -> (s*L + l)
      a.rows = x->rows + sl0 * x->W * x->cap;
      a.r_bs = (int64_t)x->L * x->W * x->cap;
      a.wlen = x->wlen + sl0 * x->W;
      a.w_bs = (int64_t)x->L * x->W;
      a.kept32 = x->kept + sl0 * x->B;
      a.k_bs = (int64_t)x->L * x->B;
      a.scores = mode == 1 ? scores_io + (int64_t)scores_off * x->cap : x->scores + sl0 * x->cap;
      a.s_bs = mode == 1 ? (int64_t)scores_ld * x->cap : (int64_t)x->L * x->cap;
      if (mode == 2) {
        a.scores_in = scores_io + (int64_t)scores_off * x->cap;
        a.si_bs = (int64_t)scores_ld * x->cap;
      }
      a.first_moved = x->first_moved + sl0 * x->S;  // scratch slice of S entries
      a.newlen = x->newlen + sl0 * x->W;
      a.acc = x->acc ? x->acc + sl0 * x->cap : nullptr;
      a.acc_bs = (int64_t)x->L * x->cap;
      if (x->slotmap) {
        a.perm = x->perm + sl0 * x->cap;
        a.pm_bs = (int64_t)x->L * x->cap;
        if (mode != 1) {
          a.moves = x->moves + sl0 * 4 * (int64_t)x->cap;
          a.mv_bs = (int64_t)x->L * 4 * x->cap;
          a.mcount = x->mcount + sl0;
          a.mc_bs = x->L;
        }
      }
      cudaError_t e = launch_select(x->S, a, st);
      if (e != cudaSuccess) return cuda_fail(e, "select kernel launch");
      x->launches++;
      x->last_layer = -1;
      x->layers_chain = false;
      if (mode == 1) continue;
      c.k = static_cast<char*>(x->k) + sl0 * x->kv_layer_stride() * x->elt;
      c.v = static_cast<char*>(x->v) + sl0 * x->kv_layer_stride() * x->elt;
      c.kv_bs = x->kv_stream_stride() * x->elt;
      c.pos = x->pos + sl0 * x->cap;
      c.modality = x->modality + sl0 * x->cap;
      c.round_id = x->round_id + sl0 * x->cap;
      c.m_bs = (int64_t)x->L * x->cap;
      c.rows = x->rows + sl0 * x->W * x->cap;
      c.r_bs = (int64_t)x->L * x->W * x->cap;
      c.wlen = x->wlen + sl0 * x->W;
      c.newlen = x->newlen + sl0 * x->W;
      c.w_bs = (int64_t)x->L * x->W;
      c.kept32 = x->kept + sl0 * x->B;
      c.k_bs = (int64_t)x->L * x->B;
      c.first_moved = a.first_moved;
      c.len = x->len + sl0;
      c.len_bs = x->L;
      c.acc = x->acc ? x->acc + sl0 * x->cap : nullptr;
      c.acc_bs = (int64_t)x->L * x->cap;
      c.k_raw = x->kraw ? static_cast<char*>(x->kraw) + sl0 * x->kv_layer_stride() * x->elt : nullptr;
      c.rope_cr = x->cfg.rope_mode == SKV_ROPE_CACHE_RELATIVE;
      if (x->slotmap) {
        c.moves = a.moves;
        c.mv_bs = a.mv_bs;
        c.mcount = a.mcount;
        c.mc_bs = a.mc_bs;
      }
      e = launch_compact(x->S, c, st);
      if (e != cudaSuccess) return cuda_fail(e, "compact kernel launch");
      x->launches++;
      x->last_layer = -1;
      x->layers_chain = false;
      if (c.rope_cr) {
        int rc = rope_rows(x, l, l + 1, 0, m, x->first_moved, st);
        if (rc) return rc;
      }
    }
  }
  if (mode == 1) return SKV_OK;
  if (kept_dev) {
    // [S][kept_ld][B] (rows kept_off .. kept_off+nl) out of the [S][L][B] scratch
    SKV_CK(cudaMemcpy2DAsync(kept_dev + (int64_t)kept_off * x->B, (size_t)kept_ld * x->B * sizeof(int32_t),
                             x->kept + (int64_t)l0 * x->B, (size_t)x->L * x->B * sizeof(int32_t),
                             (size_t)nl * x->B * sizeof(int32_t), x->S, cudaMemcpyDeviceToDevice, st));
  }
  for (int l = l0; l < l1; ++l) x->n[l] = m;
  return SKV_OK;
}

static int evict_common(skv_ctx* x, int layer, int32_t* kept_dev, void* stream, int mode, float* scores) {
  if (!x) return fail(SKV_EINVAL, "null argument");
  if (layer < -1 || layer >= x->L) return fail(SKV_EINVAL, "layer out of range");
  cudaStream_t st = as_stream(stream);
  const int l0 = layer < 0 ? 0 : layer, l1 = layer < 0 ? x->L : layer + 1;
  if (x->cfg.policy == SKV_POLICY_NONE) return SKV_OK;  // keep_all: nothing changes (engine.py:298-299)
  if (x->cfg.policy != SKV_POLICY_INF_MLLM && mode != 0)
    return fail(SKV_EINVAL, "score export / apply is defined for the Inf-MLLM policy only");
  for (int l = l0; l < l1; ++l)
    if (x->ragged[l]) return ragged_fail(x, l);
  for (int l = l0; l < l1; ++l) {
    if (x->cfg.policy == SKV_POLICY_INF_MLLM && x->wcount[l] == 0)
      return fail(SKV_EINVAL, "attention window is empty");
  }
  if (mode != 2) {
    for (int l = l0; l < l1; ++l) {
      int rc = flush_pending(x, l, st);
      if (rc) return rc;
    }
  }
  bool uniform = true;
  for (int l = l0 + 1; l < l1; ++l)
    uniform &= x->n[l] == x->n[l0] && x->whead[l] == x->whead[l0] && x->wcount[l] == x->wcount[l0];
  const int nl = l1 - l0;
  if (uniform && l0 == 0 && l1 == x->L) return evict_layers(x, l0, l1, kept_dev, nl, 0, st, mode, scores, nl, 0);
  for (int l = l0; l < l1; ++l) {
    int rc = evict_layers(x, l, l + 1, kept_dev, nl, l - l0, st, mode, scores, nl, l - l0);
    if (rc) return rc;
  }
  return SKV_OK;
}

int skv_evict(skv_ctx* x, int layer, int32_t* kept_dev, void* stream) {
  SPEC_CANCEL(x);
  return evict_common(x, layer, kept_dev, stream, 0, nullptr);
}

int skv_evict_scores(skv_ctx* x, int layer, float* scores_dev, void* stream) {
  SPEC_CANCEL(x);
  if (!scores_dev) return fail(SKV_EINVAL, "null argument");
  return evict_common(x, layer, nullptr, stream, 1, scores_dev);
}

int skv_evict_apply(skv_ctx* x, int layer, const float* scores_dev, int32_t* kept_dev, void* stream) {
  SPEC_CANCEL(x);
  if (!scores_dev) return fail(SKV_EINVAL, "null argument");
  return evict_common(x, layer, kept_dev, stream, 2, const_cast<float*>(scores_dev));
}

// ------------------------------------------------------------ state access --

int skv_length(const skv_ctx* x, int stream, int layer) {
  SPEC_CANCEL(x);
  if (!x || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  return x->ragged[layer] ? std::max(0, x->sn[(size_t)stream * x->L + layer]) : x->n[layer];
}

int skv_kv_view(skv_ctx* x, int stream, int layer, void** k, void** v) {
  SPEC_CANCEL(x);
  if (!x || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  const int64_t off = ((int64_t)stream * x->L + layer) * x->kv_layer_stride() * x->elt;
  // RoPE engines: the raw keys (KvCache.keys(), cache.py:93-96)
  if (k) *k = static_cast<char*>(x->kraw ? x->kraw : x->k) + off;
  if (v) *v = static_cast<char*>(x->v) + off;
  return SKV_OK;
}

// Current (length, window rows, ring head) of (stream, layer): the layer's
// mirror, or the stream's injected state while the layer is ragged.
static int stream_state(const skv_ctx* x, int stream, int layer, int* n, int* m, int* head) {
  if (!x->ragged[layer]) {
    *n = x->n[layer];
    *m = x->wcount[layer];
    *head = x->whead[layer];
    return SKV_OK;
  }
  const size_t sl = (size_t)stream * x->L + layer;
  if (x->sn[sl] < 0) return ragged_fail(x, layer);
  *n = x->sn[sl];
  *m = x->sm[sl];
  *head = x->sm[sl] % x->W;
  return SKV_OK;
}

// Host copy of the slot map of (stream, layer) (identity without one).
static int host_perm(const skv_ctx* x, int64_t sl, int n, std::vector<int32_t>& perm) {
  perm.resize(std::max(n, 1));
  if (!x->perm) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    return SKV_OK;
  }
  if (n > 0) SKV_CK(cudaMemcpy(perm.data(), x->perm + sl * x->cap, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  return SKV_OK;
}

int skv_positions(skv_ctx* x, int stream, int layer, int64_t* out, int cap) {
  SPEC_CANCEL(x);
  if (!x || !out || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  int nn, mm, hh;
  int rc = stream_state(x, stream, layer, &nn, &mm, &hh);
  if (rc) return rc;
  const int n = std::min(cap, nn);
  SKV_CK(cudaDeviceSynchronize());
  SKV_CK(cudaMemcpy(out, x->pos + ((int64_t)stream * x->L + layer) * x->cap, n * sizeof(int64_t),
                    cudaMemcpyDeviceToHost));
  rc = check_sticky(x);
  return rc ? rc : n;
}

int skv_window_rows(skv_ctx* x, int stream, int layer, float* rows_host, int32_t* lens_host) {
  SPEC_CANCEL(x);
  if (!x || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  int nn, count, head;
  int rc = stream_state(x, stream, layer, &nn, &count, &head);
  if (rc) return rc;
  if (!x->ragged[layer]) {
    rc = flush_pending(x, layer, nullptr);
    if (rc) return rc;
  }
  SKV_CK(cudaDeviceSynchronize());
  const int64_t sl = (int64_t)stream * x->L + layer;
  std::vector<int32_t> lens(x->W), perm;
  SKV_CK(cudaMemcpy(lens.data(), x->wlen + sl * x->W, x->W * sizeof(int32_t), cudaMemcpyDeviceToHost));
  rc = host_perm(x, sl, nn, perm);
  if (rc) return rc;
  std::vector<float> phys(std::max(nn, 1));
  for (int k = 0; k < count; ++k) {
    const int slot = ((head - count + k) % x->W + x->W) % x->W;
    const int len = std::min(lens[slot], nn);
    if (lens_host) lens_host[k] = len;
    if (rows_host && nn > 0) {  // values sit at physical rows: logical column c <- perm[c]
      SKV_CK(cudaMemcpy(phys.data(), x->rows + (sl * x->W + slot) * x->cap, (size_t)nn * sizeof(float),
                        cudaMemcpyDeviceToHost));
      for (int c = 0; c < len; ++c) rows_host[(int64_t)k * x->cap + c] = phys[perm[c]];
    }
  }
  rc = check_sticky(x);
  return rc ? rc : count;
}

int skv_state_dump(skv_ctx* x, int stream, int layer, int* n_out, int* m_out, void* k_host, void* v_host,
                   int64_t* pos_host, int8_t* modality_host, int32_t* round_host, float* rows_host,
                   int32_t* lens_host) {
  SPEC_CANCEL(x);
  if (!x || !n_out || !m_out || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L)
    return fail(SKV_EINVAL, "out of range");
  int n, m, head;
  int rc = stream_state(x, stream, layer, &n, &m, &head);
  if (rc) return rc;
  if (!x->ragged[layer]) {
    rc = flush_pending(x, layer, nullptr);  // the newest window row is materialised
    if (rc) return rc;
  }
  SKV_CK(cudaDeviceSynchronize());
  *n_out = n;
  *m_out = m;
  const int64_t sl = (int64_t)stream * x->L + layer;
  const size_t rb = (size_t)x->D * x->elt;
  const char* kd = static_cast<const char*>(x->kraw ? x->kraw : x->k) + sl * x->kv_layer_stride() * x->elt;
  const char* vd = static_cast<const char*>(x->v) + sl * x->kv_layer_stride() * x->elt;
  std::vector<int32_t> perm;
  rc = host_perm(x, sl, n, perm);
  if (rc) return rc;
  if (n > 0) {
    // K/V rows are physical: read the segment, emit logical row c = physical perm[c]
    std::vector<char> seg((size_t)n * rb);
    for (int pass = 0; pass < 2; ++pass) {
      char* dst = static_cast<char*>(pass ? v_host : k_host);
      if (!dst) continue;
      for (int h = 0; h < x->Hkv; ++h) {
        SKV_CK(cudaMemcpy(seg.data(), (pass ? vd : kd) + (size_t)h * x->cap * rb, (size_t)n * rb,
                          cudaMemcpyDeviceToHost));
        for (int c = 0; c < n; ++c)
          memcpy(dst + ((size_t)h * n + c) * rb, seg.data() + (size_t)perm[c] * rb, rb);
      }
    }
    if (pos_host) SKV_CK(cudaMemcpy(pos_host, x->pos + sl * x->cap, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (modality_host) SKV_CK(cudaMemcpy(modality_host, x->modality + sl * x->cap, n, cudaMemcpyDeviceToHost));
    if (round_host)
      SKV_CK(cudaMemcpy(round_host, x->round_id + sl * x->cap, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  if (m > 0 && (rows_host || lens_host)) {
    std::vector<int32_t> lens(x->W);
    std::vector<float> phys(std::max(n, 1));
    SKV_CK(cudaMemcpy(lens.data(), x->wlen + sl * x->W, x->W * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int k = 0; k < m; ++k) {
      const int slot = ((head - m + k) % x->W + x->W) % x->W;
      const int len = std::min(lens[slot], n);
      if (lens_host) lens_host[k] = len;
      if (rows_host) {
        if (n > 0)
          SKV_CK(cudaMemcpy(phys.data(), x->rows + (sl * x->W + slot) * x->cap, (size_t)n * sizeof(float),
                            cudaMemcpyDeviceToHost));
        for (int c = 0; c < n; ++c) rows_host[(int64_t)k * n + c] = c < len ? phys[perm[c]] : 0.f;
      }
    }
  }
  return check_sticky(x);
}

int skv_window_view(skv_ctx* x, int stream, int layer, float** rows_dev, int32_t** lens_dev, int* ring_head,
                    int* count) {
  SPEC_CANCEL(x);
  if (!x || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  int n, m, head;
  int rc = stream_state(x, stream, layer, &n, &m, &head);
  if (rc) return rc;
  if (!x->ragged[layer]) {
    rc = flush_pending(x, layer, nullptr);  // the newest recorded row is materialised (stream-ordered)
    if (rc) return rc;
  }
  const int64_t sl = (int64_t)stream * x->L + layer;
  if (rows_dev) *rows_dev = x->rows + sl * x->W * x->cap;
  if (lens_dev) *lens_dev = x->wlen + sl * x->W;
  if (ring_head) *ring_head = head;
  if (count) *count = m;
  return x->cap;  // row stride (floats)
}

int skv_positions_view(skv_ctx* x, int stream, int layer, int64_t** pos_dev) {
  SPEC_CANCEL(x);
  if (!x || !pos_dev || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L)
    return fail(SKV_EINVAL, "out of range");
  *pos_dev = x->pos + ((int64_t)stream * x->L + layer) * x->cap;
  return SKV_OK;
}

int skv_slot_map(skv_ctx* x, int stream, int layer, int32_t** perm_dev) {
  SPEC_CANCEL(x);
  if (!x || !perm_dev || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L)
    return fail(SKV_EINVAL, "out of range");
  *perm_dev = x->perm ? x->perm + ((int64_t)stream * x->L + layer) * x->cap : nullptr;
  return SKV_OK;
}

int skv_moved_rows(skv_ctx* x, int32_t* out_host) {
  SPEC_CANCEL(x);
  if (!x || !out_host) return fail(SKV_EINVAL, "null argument");
  if (!x->mcount) return fail(SKV_ESTATE, "no slot map: this engine compacts densely");
  SKV_CK(cudaDeviceSynchronize());
  SKV_CK(cudaMemcpy(out_host, x->mcount, x->sl_count() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  return SKV_OK;
}

int skv_sync(skv_ctx* x, void* stream) {
  SPEC_CANCEL(x);
  if (!x) return fail(SKV_EINVAL, "null argument");
  SKV_CK(cudaStreamSynchronize(as_stream(stream)));
  return check_sticky(x);
}

int skv_last_scores(skv_ctx* x, int stream, int layer, float* out, int cap) {
  SPEC_CANCEL(x);
  if (!x || !out || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  SKV_CK(cudaDeviceSynchronize());
  SKV_CK(cudaMemcpy(out, x->scores + ((int64_t)stream * x->L + layer) * x->cap,
                    (size_t)std::min(cap, x->cap) * sizeof(float), cudaMemcpyDeviceToHost));
  return SKV_OK;
}

int skv_state_inject(skv_ctx* x, int stream, int layer, int n, const void* k_host, const void* v_host,
                     const int64_t* pos_host, int m, const float* rows_host, const int32_t* lens_host) {
  SPEC_CANCEL(x);
  if (!x || stream < 0 || stream >= x->S || layer < 0 || layer >= x->L) return fail(SKV_EINVAL, "out of range");
  if (n < 0 || n > x->cap) return fail(SKV_EINVAL, "n exceeds capacity");
  if (m < 0 || m > x->W) return fail(SKV_EINVAL, "too many window rows");
  // window rows: 0 < len <= n, oldest first and never shrinking towards the
  // newest (AttentionWindow.push, policies.py:107-115)
  std::vector<int32_t> lens(x->W, 0);
  for (int k = 0; k < m; ++k) {
    lens[k] = lens_host ? lens_host[k] : n;
    if (lens[k] < 1 || lens[k] > n) return fail(SKV_EINVAL, "window row lengths must be in [1, n]");
    if (k > 0 && lens[k] < lens[k - 1]) return fail(SKV_EINVAL, "window rows may not shrink (oldest first)");
  }
  SKV_CK(cudaDeviceSynchronize());
  const int64_t sl = (int64_t)stream * x->L + layer;
  const size_t rb = (size_t)x->D * x->elt;
  // RoPE engines take raw keys (into the raw store) and rotate them below
  char* kd = static_cast<char*>(x->kraw ? x->kraw : x->k) + sl * x->kv_layer_stride() * x->elt;
  char* vd = static_cast<char*>(x->v) + sl * x->kv_layer_stride() * x->elt;
  if (k_host && v_host && n > 0) {
    SKV_CK(cudaMemcpy2D(kd, (size_t)x->cap * rb, k_host, (size_t)n * rb, (size_t)n * rb, x->Hkv,
                        cudaMemcpyHostToDevice));
    SKV_CK(cudaMemcpy2D(vd, (size_t)x->cap * rb, v_host, (size_t)n * rb, (size_t)n * rb, x->Hkv,
                        cudaMemcpyHostToDevice));
  }
  if (pos_host && n > 0) {
    SKV_CK(cudaMemcpy(x->pos + sl * x->cap, pos_host, n * sizeof(int64_t), cudaMemcpyHostToDevice));
    const int64_t nextp = pos_host[n - 1] + 1;
    SKV_CK(cudaMemcpy(x->next_pos + sl, &nextp, sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  const int32_t n32 = n;
  SKV_CK(cudaMemcpy(x->len + sl, &n32, sizeof(int32_t), cudaMemcpyHostToDevice));
  if (x->perm) {  // injected rows are in logical order: identity slot map
    SKV_CK(launch_iota(x->perm + sl * x->cap, x->cap, x->cap, nullptr));
    SKV_CK(cudaDeviceSynchronize());
  }
  for (int k = 0; k < m; ++k)
    if (rows_host)
      SKV_CK(cudaMemcpy(x->rows + (sl * x->W + k) * x->cap, rows_host + (int64_t)k * n, (size_t)lens[k] * sizeof(float),
                        cudaMemcpyHostToDevice));
  SKV_CK(cudaMemcpy(x->wlen + sl * x->W, lens.data(), x->W * sizeof(int32_t), cudaMemcpyHostToDevice));
  x->last_layer = -1;
  x->layers_chain = false;
  if (x->acc)  // heavy hitter: injected tokens start with no accumulated mass
    SKV_CK(cudaMemset(x->acc + ((int64_t)stream * x->L + layer) * x->cap, 0, (size_t)x->cap * sizeof(float)));
  if (x->kraw && n > 0) {  // rotated keys of the injected tokens (every stream of the layer)
    int rc = rope_rows(x, layer, layer + 1, 0, n, nullptr, nullptr);
    if (rc) return rc;
    SKV_CK(cudaDeviceSynchronize());
  }
  // host mirror: one state per layer.  Injecting one stream rewrites its ring
  // from slot 0, so the layer is unusable (ragged) until every stream of it has
  // been injected with the same n and row count.
  if (!x->ragged[layer])
    for (int s = 0; s < x->S; ++s) x->sn[(size_t)s * x->L + layer] = x->sm[(size_t)s * x->L + layer] = -1;
  x->sn[sl] = n;
  x->sm[sl] = m;
  bool rg = false;
  for (int s = 1; s < x->S; ++s)
    rg |= x->sn[(size_t)s * x->L + layer] != x->sn[layer] || x->sm[(size_t)s * x->L + layer] != x->sm[layer];
  x->ragged[layer] = rg;
  x->n[layer] = n;
  x->wcount[layer] = m;
  x->whead[layer] = m % x->W;
  x->pend_n[layer] = 0;
  return SKV_OK;
}

// ------------------------------------------------------------------ graphs --

int skv_capture_begin(skv_ctx* x, void* stream) {
  SPEC_CANCEL(x);
  if (!x) return fail(SKV_EINVAL, "null argument");
  // release the previous graph before capturing: destroying graph objects is not
  // permitted while a thread-local capture is active
  if (x->exec) {
    SKV_CK(cudaStreamSynchronize(as_stream(stream)));
    cudaGraphExecDestroy(x->exec);
    x->exec = nullptr;
  }
  if (x->graph) {
    cudaGraphDestroy(x->graph);
    x->graph = nullptr;
  }
  SKV_CK(cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeThreadLocal));
  x->gbegin = x->snap();
  return SKV_OK;
}

int skv_capture_end(skv_ctx* x, void* stream) {
  SPEC_CANCEL(x);
  if (!x) return fail(SKV_EINVAL, "null argument");
  x->gend = x->snap();
  x->restore(x->gbegin);  // nothing has executed yet
  SKV_CK(cudaStreamEndCapture(as_stream(stream), &x->graph));
  SKV_CK(cudaGraphInstantiate(&x->exec, x->graph, 0));
  return SKV_OK;
}

int skv_graph_launch(skv_ctx* x, void* stream) {
  SPEC_CANCEL(x);
  if (!x || !x->exec) return fail(SKV_ESTATE, "no captured graph");
  if (!(x->snap() == x->gbegin))
    return fail(SKV_ESTATE, "graph replay refused: engine state differs from the state at capture begin");
  SKV_CK(cudaGraphLaunch(x->exec, as_stream(stream)));
  x->restore(x->gend);
  return SKV_OK;
}

// ------------------------------------------------------- stand-alone policy --

int skv_top_k(const float* scores, int n, int k, int64_t* out, void* stream) {
  if (k < 0) return fail(SKV_EINVAL, "k must be >= 0");
  if (n < 0) return fail(SKV_EINVAL, "n must be >= 0");
  if (k == 0 || n == 0) return SKV_OK;
  cudaError_t e = launch_topk(scores, n, k, out, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "top-k kernel launch");
  return SKV_OK;
}

static int check_window(int m, int n, int recent_len) {
  if (m <= 0) return fail(SKV_EINVAL, "attention window is empty");
  if (m > 1024) return fail(SKV_EINVAL, "window holds more than 1024 rows");
  (void)n;
  (void)recent_len;
  return SKV_OK;
}

int skv_window_scores(const float* rows, int row_stride, const int32_t* lens, int m, int n, int recent_len,
                      float bias, int apply_bias, float* scores, void* stream) {
  int rc = check_window(m, n, recent_len);
  if (rc) return rc;
  if (n <= recent_len) return fail(SKV_EINVAL, "no scorable columns: n <= l");
  if (bias < 0) return fail(SKV_EINVAL, "bias must be >= 0");
  SelectArgs a{};
  a.rows = rows;
  a.row_stride = row_stride;
  a.wlen = lens;
  a.ring_head = m;
  a.count = m;
  a.W = m;
  a.n = n;
  a.l = recent_len;
  a.bias = bias;
  a.apply_bias = apply_bias;
  a.scores = scores;
  a.scores_only = 1;
  cudaError_t e = launch_select(1, a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "select kernel launch");
  return SKV_OK;
}

int skv_policy_decide(int policy, const float* acc, int n, int recent_len, int relevant_budget, int sink_count,
                      int64_t* kept, float* scores, void* stream) {
  if (n < 0) return fail(SKV_EINVAL, "n must be >= 0");
  if (policy == SKV_POLICY_WINDOW) {
    if (recent_len < 1) return fail(SKV_EINVAL, "budget must be >= 1");
    relevant_budget = 0;
    sink_count = 0;
  } else if (policy == SKV_POLICY_SINK_RECENT) {
    if (!(recent_len + relevant_budget > sink_count && sink_count >= 0))
      return fail(SKV_EINVAL, "require budget > sink_count >= 0");
  } else if (policy == SKV_POLICY_HEAVY_HITTER) {
    if (recent_len < 1 || relevant_budget < 0) return fail(SKV_EINVAL, "bad policy config");
    if (n > recent_len + relevant_budget && (!acc || !scores))
      return fail(SKV_EINVAL, "accumulator and scores scratch required when n > r + l");
  } else {
    return fail(SKV_EINVAL, "policy must be window, sink_recent or heavy_hitter");
  }
  if (n == 0) return 0;
  SelectArgs a{};
  a.W = 1;
  a.n = n;
  a.l = recent_len;
  a.r = relevant_budget;
  a.policy = policy;
  a.sink = sink_count;
  a.acc = acc;
  a.scores = scores;
  a.kept64 = kept;
  cudaError_t e = launch_select(1, a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "select kernel launch");
  return std::min(n, recent_len + relevant_budget);
}

int skv_project_row(const float* probs, int n, const int64_t* live, int m, float* out, void* stream) {
  if (n < 0 || m < 0) return fail(SKV_EINVAL, "lengths must be >= 0");
  if (m == 0) return SKV_OK;
  if (!probs || !live || !out) return fail(SKV_EINVAL, "null argument");
  cudaError_t e = launch_project_row(probs, n, live, m, out, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "projection kernel launch");
  return SKV_OK;
}

int skv_masked_row_sums(const float* rows, int row_stride, const int32_t* lens, int m, const int64_t* kept, int k,
                        double* out, void* stream) {
  if (m < 0 || k < 0 || row_stride < 0) return fail(SKV_EINVAL, "lengths must be >= 0");
  if (m == 0) return SKV_OK;
  if (!rows || !lens || !out || (k > 0 && !kept)) return fail(SKV_EINVAL, "null argument");
  cudaError_t e = launch_masked_row_sums(rows, row_stride, lens, m, kept, k, out, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "row-sum kernel launch");
  return SKV_OK;
}

int skv_hh_accumulate(const float* acc, int na, const float* row, int n, float* out, void* stream) {
  if (na < 0 || n < 0) return fail(SKV_EINVAL, "lengths must be >= 0");
  if (na > n) return fail(SKV_EINVAL, "accumulator longer than the new row");
  if (n == 0) return SKV_OK;
  cudaError_t e = launch_hh_accumulate(acc, na, row, n, out, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "accumulate kernel launch");
  return SKV_OK;
}

int skv_decide(const float* rows, int row_stride, const int32_t* lens, int m, int n, int recent_len,
               int relevant_budget, float bias, int64_t* kept, float* scores, void* stream) {
  int rc = check_window(m, n, recent_len);
  if (rc) return rc;
  if (recent_len < 1 || relevant_budget < 0 || bias < 0) return fail(SKV_EINVAL, "bad policy config");
  if (n <= recent_len + relevant_budget) {
    SelectArgs a{};
    a.rows = rows;
    a.row_stride = row_stride;
    a.wlen = lens;
    a.ring_head = m;
    a.count = m;
    a.W = m;
    a.n = n;
    a.l = recent_len;
    a.r = relevant_budget;
    a.kept64 = kept;
    cudaError_t e = launch_select(1, a, as_stream(stream));
    if (e != cudaSuccess) return cuda_fail(e, "select kernel launch");
    return n;
  }
  if (!scores) return fail(SKV_EINVAL, "scores scratch required when n > r + l");
  SelectArgs a{};
  a.rows = rows;
  a.row_stride = row_stride;
  a.wlen = lens;
  a.ring_head = m;
  a.count = m;
  a.W = m;
  a.n = n;
  a.l = recent_len;
  a.r = relevant_budget;
  a.bias = bias;
  a.apply_bias = 1;
  a.kept64 = kept;
  a.scores = scores;
  cudaError_t e = launch_select(1, a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "select kernel launch");
  return recent_len + relevant_budget;
}

int skv_gather_rows(void* base, int64_t block_stride, int blocks, int row_bytes, const int64_t* kept, int m,
                    void* stream) {
  if (row_bytes % 16) return fail(SKV_EINVAL, "row_bytes must be a multiple of 16");
  if (m <= 0 || blocks <= 0) return SKV_OK;
  CompactArgs c{};
  c.k = static_cast<char*>(base);
  c.kv_hs = block_stride;
  c.heads = blocks;
  c.row_bytes = row_bytes;
  c.kept64 = kept;
  c.m = m;
  cudaError_t e = launch_compact(1, c, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "compact kernel launch");
  return SKV_OK;
}

// Scratch for the stand-alone attend (drop-in API, not the engine hot path).
namespace {
struct AttendScratch {
  float* stats = nullptr;
  float* part = nullptr;
  int32_t* counters = nullptr;
  int32_t* sched = nullptr;
  size_t part_floats = 0;
  int heads = 0;
  int dev = -1;  // device the scratch lives on
};
thread_local AttendScratch g_att;
}  // namespace

int skv_attend(const float* keys, const float* values, int heads, int n, int head_dim, int64_t head_stride,
               const float* q, float* probs, float* out, void* stream) {
  if (heads < 1 || n < 1) return fail(SKV_EINVAL, "keys must be a non-empty sequence of vectors");
  if (head_dim != 64 && head_dim != 128) return fail(SKV_EINVAL, "device attend needs head_dim 64 or 128");
  // the stand-alone attend shares one scratch context: calls from several
  // host threads are serialised (engine contexts have no shared state)
  static std::mutex att_mu;
  std::lock_guard<std::mutex> lock(att_mu);
  cudaStream_t st = as_stream(stream);
  const int nt = (n + decode_tile_tokens() - 1) / decode_tile_tokens();
  const int ach = std::max(chunk_tiles(1), (nt + 127) / 128);  // at most 128 chunks (segment merge)
  const int nc = (nt + ach - 1) / ach;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = std::min(heads * nc, sms * decode_ctas_per_sm(SKV_DTYPE_F32, head_dim, 1));
  const size_t need = (size_t)heads * nc * (head_dim + 2);
  if (g_att.dev != dev) {  // this thread moved to another device: fresh scratch there
    g_att = AttendScratch{};
    g_att.dev = dev;
  }
  if (g_att.part_floats < need || g_att.heads < heads) {
    SKV_CK(cudaStreamSynchronize(st));
    if (g_att.stats) cudaFree(g_att.stats);
    if (g_att.part) cudaFree(g_att.part);
    if (g_att.counters) cudaFree(g_att.counters);
    const int hcap = std::max(heads, 64);
    const size_t pcap = std::max(need, (size_t)(hcap + 1024) * 130);
    SKV_CK(cudaMalloc(&g_att.stats, hcap * 2 * sizeof(float)));
    SKV_CK(cudaMalloc(&g_att.part, pcap * sizeof(float)));
    SKV_CK(cudaMalloc(&g_att.counters, 4 * hcap * sizeof(int32_t)));
    SKV_CK(cudaMemset(g_att.counters, 0, 4 * hcap * sizeof(int32_t)));
    if (!g_att.sched) {
      SKV_CK(cudaMalloc(&g_att.sched, 8 * sizeof(int32_t)));
      SKV_CK(cudaMemset(g_att.sched, 0, 8 * sizeof(int32_t)));
    }
    g_att.part_floats = pcap;
    g_att.heads = hcap;
  }
  AttnArgs a{};
  a.Hq = heads;
  a.Hkv = heads;
  a.n_old = n;
  a.append = 0;
  a.nt = nt;
  a.ch = ach;
  a.nc = nc;
  a.S = 1;
  a.sched = g_att.sched;
  a.done_self = nullptr;
  a.dctas = ctas;
  a.prefetch = 0;
  a.scale = (float)(1.0 / std::sqrt((double)head_dim));
  a.kc = const_cast<float*>(keys);
  a.vc = const_cast<float*>(values);
  a.c_ss = 0;
  a.c_hs = head_stride;
  a.q = q;
  a.kin = keys;  // unused (append = 0)
  a.vin = values;
  a.out = out;
  a.logits = probs;  // logits recorded in place, then normalised below
  a.l_hs = n;
  a.stats = g_att.stats;
  a.part = g_att.part;
  static int att_seq = 0;
  a.counters = g_att.counters + (size_t)(att_seq++ % 4) * g_att.heads;
  cudaError_t e = launch_decode(SKV_DTYPE_F32, head_dim, 1, ctas, a, st);
  if (e != cudaSuccess) return cuda_fail(e, "decode kernel launch");
  FoldArgs f{};
  f.logits = probs;
  f.l_hs = n;
  f.stats = g_att.stats;
  f.probs = probs;
  f.p_hs = n;
  f.n = n;
  f.mode = 2;
  e = launch_fold(1, std::max(1, std::min(64, (n + 127) / 128)), f, heads, st);
  if (e != cudaSuccess) return cuda_fail(e, "fold kernel launch");
  return SKV_OK;
}

int skv_prefill_profile(uint64_t* counters) {
  set_prefill_profile(reinterpret_cast<unsigned long long*>(counters));
  return SKV_OK;
}

int skv_prefill_attend(const void* q, int streams, int C, int Hq, int Hkv, const void* k_cache, const void* v_cache,
                       int L, int layer, int cap, int n0, float* out, int W, float* logits, int64_t lg_cap,
                       float* stats, void* stream) {
  if (!q || !k_cache || !v_cache || !out) return fail(SKV_EINVAL, "null argument");
  if (streams < 1 || C < 1 || Hq < 1 || Hkv < 1 || Hq % Hkv || L < 1 || layer < 0 || layer >= L)
    return fail(SKV_EINVAL, "bad prefill geometry");
  if (n0 < 0 || n0 + C > cap) return fail(SKV_EINVAL, "chunk exceeds the cache capacity");
  if (W < 0 || W > C) return fail(SKV_EINVAL, "W must be in [0, C]");
  // recorded logit rows hold n0 + C columns
  if (W > 0 && (!logits || !stats)) return fail(SKV_EINVAL, "W > 0 needs logits and stats buffers");
  if (W > 0 && lg_cap < (int64_t)n0 + C) return fail(SKV_EINVAL, "lg_cap must be >= n0 + C");
  PrefillArgs a{};
  a.C = C;
  a.n0 = n0;
  a.W = W;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.G = Hq / Hkv;
  a.L = L;
  a.layer = layer;
  a.cap = cap;
  a.scale = (float)(1.0 / std::sqrt(128.0));
  a.out = out;
  a.lg = W > 0 ? logits : nullptr;
  a.lg_cap = lg_cap;
#ifdef SKV_INSTRUMENT
  if (const char* e = getenv("SKV_PF_LGT")) a.lg_t = atoi(e) && lg_cap % 128 == 0;  // experiment: engine layout
#endif
  a.st = W > 0 ? stats : nullptr;
  const int64_t rows = (int64_t)streams * L * Hkv * cap;
  cudaError_t e = launch_prefill(q, streams, k_cache, v_cache, rows, a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "prefill kernel launch");
  return SKV_OK;
}

}  // extern "C"
