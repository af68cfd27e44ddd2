/*
 * streamkv_b200 -- C ABI of the B200 (sm_100a) Inf-MLLM streaming-decode hot path.
 *
 * The reference (`streamkv`, pure Python/NumPy) has no FFI; its boundary is the
 * public Python API re-exported by /root/reference/pkg/src/streamkv/__init__.py:3-32
 * plus the Session._attend call site (engine.py:269-271).  Every entry point
 * below replaces one piece of that API; the reference interface it stands in
 * for is cited beside it.  The Python drop-in (paper_2409_09086_b200/) binds
 * these with ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Every function returns 0 on success or a negative SKV_E* code; the message
 *     of the last error on the calling thread is returned by skv_last_error().
 *   - SKV_EINVAL is the reference's ValueError domain (shapes, index ranges,
 *     non-ascending kept sets, empty windows, n <= l, bad config).
 *   - Pointers named *_dev are device pointers; *_host are host pointers.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *     enqueued on it; functions that return host data synchronise it.
 *   - A context owns all its device buffers; nothing is allocated on the hot path.
 *   - Distinct contexts are independent; one context is externally serialised
 *     (reference SPEC.md:168).
 */
#ifndef STREAMKV_B200_H
#define STREAMKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKV_OK 0
#define SKV_EINVAL -1 /* domain error: the reference raises ValueError */
#define SKV_ECUDA -2  /* CUDA runtime error */
#define SKV_ENOMEM -3 /* device allocation failed */
#define SKV_ESTATE -4 /* call not valid in the current context state */

#define SKV_DTYPE_F32 0
#define SKV_DTYPE_BF16 1

/* Eviction policy: the Session's policy switch (engine.py:296-307). */
#define SKV_POLICY_INF_MLLM 0     /* inf_mllm_decide, policies.py:184-201 (the hot path) */
#define SKV_POLICY_WINDOW 1       /* sliding_window_decide(n, budget), policies.py:204-213 */
#define SKV_POLICY_SINK_RECENT 2  /* sink_recent_decide(n, sink_count, budget), policies.py:216-231 */
#define SKV_POLICY_HEAVY_HITTER 3 /* heavy_hitter_accumulate/decide, policies.py:234-256 */
#define SKV_POLICY_NONE 4         /* keep everything (EvictionDecision.keep_all, engine.py:298-299) */

/* Rotary positions of the cached keys (PositionMode, cache.py:24-34; the
 * Session's rotary helpers engine.py:198-233).  With RoPE on, q and k inputs
 * are pre-rotation: the engine rotates q and the new k at the token's
 * position, keeps raw keys (what cache.keys() returns) next to the rotated
 * keys it attends over, and after a compaction re-rotates the moved keys at
 * their new slots (cache-relative, _refresh_rotations engine.py:339-342). */
#define SKV_ROPE_NONE 0           /* inputs already rotated (the BASELINE configs) */
#define SKV_ROPE_CACHE_RELATIVE 1 /* PositionMode.CACHE_RELATIVE: position = cache slot */
#define SKV_ROPE_ORIGINAL 2       /* PositionMode.ORIGINAL: position = original stream position */

#define SKV_AGG_MEAN 0 /* aggregate_heads(.., "mean"), policies.py:261-262 */
#define SKV_AGG_MAX 1  /* aggregate_heads(.., "max"),  policies.py:263-264 */

/* Engine configuration.  Mirrors PolicyConfig (policies.py:28-59) plus the
 * cache shape of KvCache(layers, heads, head_dim) (cache.py:73-81) batched over
 * `streams` independent sessions, with GQA (heads_q a multiple of heads_kv). */
typedef struct skv_config {
  int32_t streams;         /* S independent sessions (no cross-session state) */
  int32_t layers;          /* L */
  int32_t heads_q;         /* query heads */
  int32_t heads_kv;        /* key/value heads (== heads_q in the reference) */
  int32_t head_dim;        /* D: 64 or 128 */
  int32_t dtype;           /* SKV_DTYPE_*: q/k/v inputs and the KV store */
  int32_t recent_len;      /* l  (PolicyConfig.recent_len) */
  int32_t relevant_budget; /* r  (PolicyConfig.relevant_budget) */
  float bias;              /* b  (PolicyConfig.bias) */
  int32_t window;          /* W rows of AttentionWindow(capacity=W), policies.py:98 */
  int32_t capacity;        /* max cached tokens per (stream, layer) */
  int32_t head_agg;        /* SKV_AGG_* */
  int32_t heads_q_total;   /* 0, or the query heads of all head shards: a shard's window rows are
                              its heads' probability sums / heads_q_total, so the shards' rows add
                              up to the reference head mean */
  int32_t policy;          /* SKV_POLICY_* (zero-initialised configs get the Inf-MLLM policy) */
  int32_t sink_count;      /* s  (PolicyConfig.sink_count) for SKV_POLICY_SINK_RECENT */
  int32_t rope_mode;       /* SKV_ROPE_* (0: q/k arrive rotated) */
  float rope_base;         /* ModelSpec.rope_base (engine.py:69), e.g. 10000 */
} skv_config;

typedef struct skv_ctx skv_ctx;

const char* skv_last_error(void);
int skv_version(void);

/* ---- lifetime ------------------------------------------------------------ */
int skv_create(const skv_config* cfg, skv_ctx** out);
int skv_destroy(skv_ctx* ctx);
/* Device bytes held by the context (KV store + window + scratch). */
int64_t skv_device_bytes(const skv_ctx* ctx);

/* ---- decode: append -> attend -> head aggregation -> window push -----------
 * Replaces, for one layer of every stream, the per-layer body of
 * Session.decode_step (engine.py:264-273): KvCache.append (cache.py:112-134),
 * Session._attend (engine.py:235-246), aggregate_heads (policies.py:259-265) and
 * AttentionWindow.push (policies.py:107-115).
 *   q_dev  [S][Hq][D], k_dev/v_dev [S][Hkv][D]  (config dtype)
 *   positions_host [S] original positions of the appended token (NULL: previous+1)
 *   out_dev [S][Hq][D] float32 attention output
 *   record  nonzero: the head-aggregated probability row is pushed to the window. */
int skv_decode_layer(skv_ctx* ctx, int layer, const void* q_dev, const void* k_dev, const void* v_dev,
                     const int64_t* positions_host, float* out_dev, int record, void* stream);

/* All layers of one token (Session.decode_step minus the tiny decoder):
 * q_dev [L][S][Hq][D], k_dev/v_dev [L][S][Hkv][D], out_dev [L][S][Hq][D] f32. */
int skv_decode_step(skv_ctx* ctx, const void* q_dev, const void* k_dev, const void* v_dev, float* out_dev,
                    int record, void* stream);

/* Same with HOST (pinned or pageable) buffers: copies in, decodes all layers
 * with layer-pipelined H2D/compute/D2H on internal streams, copies out.
 * Synchronous.  Work already enqueued on `stream` (an eviction, a prefill
 * chunk) completes before the pipeline touches the cache. */
int skv_decode_step_host(skv_ctx* ctx, const void* q_host, const void* k_host, const void* v_host,
                         float* out_host, int record, void* stream);

/* Speculative host steps for shallow (<= 2 layers, no RoPE) engines -- the
 * batch-1 Session.decode_step loop (engine.py:250-289) driven token by token
 * from the host.  With enable != 0, each skv_decode_step_host call also
 * launches the NEXT token's kernels behind a device-side gate that waits (at
 * most timeout_us) for the next call's doorbell in mapped pinned memory; the
 * call copies q/k/v into the engine's mapped buffers, rings, and spins on a
 * completion word instead of launching and synchronising.  Same kernels, same
 * results.  Any other entry point, or a call with a different `record`,
 * cancels the pending step first (its kernels exit without side effects);
 * while a step is pending, a device-wide synchronisation can wait up to
 * timeout_us.  Off by default.  No reference counterpart (a latency mode of
 * the host-buffer step). */
int skv_host_speculate(skv_ctx* ctx, int enable, int timeout_us);
/* Steps served from a pending launch / pending steps cancelled or expired. */
int skv_host_speculate_stats(skv_ctx* ctx, int64_t* hits, int64_t* misses);

/* ---- eviction: Algorithm 1 + compaction -------------------------------------
 * Replaces Session._evict_layer (engine.py:310-337) for every stream:
 * inf_mllm_decide (policies.py:184-201: window_mean_scores 130-147, bias_vector
 * 150-162, top_k_indices 165-181), KvCache.gather_keep (cache.py:136-156) and
 * AttentionWindow.remap (policies.py:117-124).
 *   layer  -1 = all layers (start_round's per-layer fan-out, engine.py:355-360)
 *   kept_dev optional [S][L'][r+l] int32 copy of the kept sets (L' = 1 or L),
 *            rows padded with -1 when the cache fits the budget (keep-all).
 * Returns SKV_EINVAL if a window is empty (policies.py:191-192). */
int skv_evict(skv_ctx* ctx, int layer, int32_t* kept_dev, void* stream);

/* Head-sharded eviction (KV heads split across GPUs, SURVEY 8e "layer" mode):
 * skv_evict_scores writes this shard's window-mean scores without the bias,
 * [S][L'][capacity] f32 (first n-l columns valid); the caller sums them across
 * shards (one all-reduce of (n-l) floats per (stream, layer)), then
 * skv_evict_apply adds the bias, selects and compacts exactly like skv_evict.
 * Every shard then holds the same kept sets. */
int skv_evict_scores(skv_ctx* ctx, int layer, float* scores_dev, void* stream);
int skv_evict_apply(skv_ctx* ctx, int layer, const float* scores_dev, int32_t* kept_dev, void* stream);

/* ---- state access --------------------------------------------------------
 * The streams of one layer run in lock step (one length per layer): a layer
 * whose streams were injected with different lengths or row counts refuses
 * decode / prefill / evict with SKV_ESTATE until every stream of it has been
 * injected alike (the reference's per-Session lengths, cache.py:90-91, are
 * only representable when they agree). */
/* Synchronise `stream` and report sticky device errors: SKV_EINVAL after a
 * chunked prefill read a value |v| >= 65504 (its fp16 P.V saturated).  Every
 * call that returns host data reports them too. */
int skv_sync(skv_ctx* ctx, void* stream);
/* Current cached length of (stream, layer): KvCache.length (cache.py:90-91). */
int skv_length(const skv_ctx* ctx, int stream, int layer);
/* Device pointers to the layer's key/value storage [Hkv][capacity][D]; the
 * first skv_length() rows of each head are live.  Engines with a slot map
 * (all but cache-relative RoPE) keep rows in PHYSICAL order: logical slot c
 * (KvCache.keys()[:, c], cache.py:93-100) is physical row perm[c] of
 * skv_slot_map().  An eviction then moves only the kept rows that lie beyond
 * the kept count (the survivors of the tokens appended since the previous
 * eviction) instead of shifting every row after the first evicted one. */
int skv_kv_view(skv_ctx* ctx, int stream, int layer, void** k_dev, void** v_dev);
/* Device view of the window ring of (stream, layer): rows [W][stride] f32
 * (values at PHYSICAL rows, see skv_slot_map), lengths [W], the ring head
 * (next slot) and row count (oldest = (head - count) mod W).  Returns the row
 * stride.  A pending recorded row is materialised first (stream-ordered on
 * the legacy stream). */
int skv_window_view(skv_ctx* ctx, int stream, int layer, float** rows_dev, int32_t** lens_dev, int* ring_head,
                    int* count);
/* Device pointer to the original positions [capacity] int64 of (stream, layer)
 * (logical order; first skv_length() valid). */
int skv_positions_view(skv_ctx* ctx, int stream, int layer, int64_t** pos_dev);
/* Device pointer to the slot map of (stream, layer): int32 [capacity],
 * perm[c] = physical row of logical slot c for c < skv_length(); null for
 * densely compacted engines (identity). */
int skv_slot_map(skv_ctx* ctx, int stream, int layer, int32_t** perm_dev);
/* Rows moved per (stream, layer) by the last eviction, int32 [S][L] host copy
 * (slot-map engines; SKV_ESTATE otherwise). */
int skv_moved_rows(skv_ctx* ctx, int32_t* out_host);
/* Original positions [n] of (stream, layer), host copy (cache.py:102-104). */
int skv_positions(skv_ctx* ctx, int stream, int layer, int64_t* out_host, int cap);
/* Window rows of (stream, layer) oldest-first into out_host [W][capacity] with
 * their lengths (AttentionWindow.rows); returns the row count. */
int skv_window_rows(skv_ctx* ctx, int stream, int layer, float* rows_host, int32_t* lens_host);
/* Biased scores computed at the last eviction of (stream, layer): [n-l] f32. */
int skv_last_scores(skv_ctx* ctx, int stream, int layer, float* out_host, int cap);
/* Dump (stream, layer) state to host buffers (KvCache.debug_snapshot,
 * cache.py:172-180, with the tensors): *n_out / *m_out receive the length and
 * window row count (call with null buffers first to size them); then
 * keys/values [Hkv][n][D] in config dtype (raw keys for RoPE engines),
 * positions [n], modality [n], round ids [n], window rows [m][n] oldest first
 * (row i zero-padded after lens[i]).  Any buffer may be null. */
int skv_state_dump(skv_ctx* ctx, int stream, int layer, int* n_out, int* m_out, void* k_host, void* v_host,
                   int64_t* pos_host, int8_t* modality_host, int32_t* round_host, float* rows_host,
                   int32_t* lens_host);
/* Overwrite (stream, layer) state from host data for state-injection parity:
 * keys/values [Hkv][n][D] in config dtype, positions [n], window rows [m][n]
 * (row i has length lens[i], 1 <= lens[i] <= n, non-decreasing oldest to
 * newest like AttentionWindow.push, policies.py:107-115; SKV_EINVAL otherwise). */
int skv_state_inject(skv_ctx* ctx, int stream, int layer, int n, const void* k_host, const void* v_host,
                     const int64_t* pos_host, int m, const float* rows_host, const int32_t* lens_host);

/* ---- CUDA graphs (replaces a tracing compiler) ---------------------------- */
int skv_capture_begin(skv_ctx* ctx, void* stream);
int skv_capture_end(skv_ctx* ctx, void* stream);
int skv_graph_launch(skv_ctx* ctx, void* stream);
/* Number of this library's kernels launched since creation (instrumentation). */
int64_t skv_kernel_launches(const skv_ctx* ctx);
/* Instrumentation: when enabled, every decode launch records the earliest CTA
 * start and latest CTA end (%globaltimer, ns) into a device ring of 8192 pairs;
 * skv_timing_read copies the pairs recorded since enabling (returns the count). */
int skv_timing(skv_ctx* ctx, int enable);
int skv_timing_read(skv_ctx* ctx, uint64_t* out_host, int max_pairs);
/* enable == 3 additionally records per-CTA [start, released, end] of the
 * launches in slots tcount % 64; skv_timing_cta copies one slot (max_ctas x 8). */
int skv_timing_cta(skv_ctx* ctx, int slot, uint64_t* out_host);
/* Instrumentation: a non-null device buffer of [L][148][16] u64 makes every
 * later all-layer persistent decode record per-CTA, per-layer %globaltimer
 * stamps (released, q loaded, K in, math done, published, merged). */
int skv_layers_timeline(skv_ctx* ctx, uint64_t* buf_dev);
/* Name of the kernel the last decode launch of this context ran
 * ("decode_tcd_kernel", "decode_tc_cluster_kernel", ...; "" before any). */
const char* skv_last_decode_kernel(const skv_ctx* ctx);
/* Instrumentation: a non-null device buffer of [CTAs][16] u64 makes every
 * later prefill launch accumulate per-CTA wait/busy cycle counters into it
 * (null turns it off). */
int skv_prefill_profile(uint64_t* counters_dev);

/* ---- chunked prefill (tcgen05) ------------------------------------------------
 * Causal attention of a C-token chunk whose k/v rows are already stored at
 * slots [n0, n0+C) of each (stream, layer, kv-head) segment: query i attends to
 * slots [0, n0+i].  This is the reference's per-token prompt loop
 * (Session.start_round, engine.py:350-353, each token through decode_step) as
 * one tensor-core pass.  bf16, head_dim 128.
 *   q_dev [S][C][Hq][128] bf16;  k_cache/v_cache [S][L][Hkv][cap][128] bf16
 *   out_dev [S][C][Hq][128] f32
 *   logits_dev (optional) [S][W][Hq][lg_cap] f32 scaled logits of the last W
 *   query rows; stats_dev [S][W][Hq][2] their (max, sum). */
/* Engine-level chunk: appends the chunk's k/v ([S][C][Hkv][128] bf16) and metadata
 * (modality, e.g. 1 for image tokens) to `layer`, runs the chunk attention
 * (q [S][C][Hq][128] bf16 -> out [S][C][Hq][128] f32) and pushes the head-mean
 * rows of the last min(W, C) tokens into the window, exactly as C calls of
 * skv_decode_layer would (Session.start_round's prompt loop). */
int skv_prefill_chunk(skv_ctx* ctx, int layer, const void* q_dev, const void* k_dev, const void* v_dev, int C,
                      int modality, float* out_dev, void* stream);
int skv_prefill_attend(const void* q_dev, int streams, int C, int heads_q, int heads_kv, const void* k_cache,
                       const void* v_cache, int layers, int layer, int capacity, int n0, float* out_dev, int W,
                       float* logits_dev, int64_t lg_cap, float* stats_dev, void* stream);

/* ---- stand-alone policy kernels (drop-in for the pure policy functions) ---- */
/* top_k_indices(scores, k) (policies.py:165-181) on device: ascending indices of
 * the k largest, ties to the larger index.  out_dev receives min(k, n) int64. */
int skv_top_k(const float* scores_dev, int n, int k, int64_t* out_dev, void* stream);
/* The Session's comparison baselines (engine.py:296-307), device-side:
 *   SKV_POLICY_WINDOW:       sliding_window_decide(n, budget=recent_len)   policies.py:204-213
 *   SKV_POLICY_SINK_RECENT:  sink_recent_decide(n, sink_count, recent_len + relevant_budget)
 *                                                                           policies.py:216-231
 *   SKV_POLICY_HEAVY_HITTER: heavy_hitter_decide(acc[n], n, relevant_budget, recent_len)
 *                                                                           policies.py:246-256
 * kept_dev receives the ascending kept set (sinks/relevant first); returns its
 * length, or a negative SKV_* code.  scores_dev (>= n floats) is scratch for the
 * heavy hitter. */
int skv_policy_decide(int policy, const float* acc_dev, int n, int recent_len, int relevant_budget, int sink_count,
                      int64_t* kept_dev, float* scores_dev, void* stream);
/* heavy_hitter_accumulate (policies.py:234-243): out[j] = row[j] + acc[j] (j < na), row[j] otherwise. */
int skv_hh_accumulate(const float* acc_dev, int na, const float* row_dev, int n, float* out_dev, void* stream);
/* Trace replay (replay.py:139-142): out[i] = f32(probs[live[i]] / total) with
 * the f64 total of the projected values -- a full-stream attention row seen
 * through the surviving cache columns. */
int skv_project_row(const float* probs_dev, int n, const int64_t* live_dev, int m, float* out_dev, void* stream);
/* retained_mass (metrics.py:46-62) per row: out_dev[r] = f64 sum of
 * rows[r][kept[i]] over kept[i] < lens[r]; rows_dev [m][row_stride]. */
int skv_masked_row_sums(const float* rows_dev, int row_stride, const int32_t* lens_dev, int m,
                        const int64_t* kept_dev, int k, double* out_dev, void* stream);
/* inf_mllm_decide over a device window: rows_dev [m][row_stride] f32 oldest
 * first, lens_dev [m] int32.  kept_dev [min(n, r+l)] int64; scores_dev optional
 * [n-l] f32 biased scores.  Returns the kept count (>= 0) or an error. */
int skv_decide(const float* rows_dev, int row_stride, const int32_t* lens_dev, int m, int n, int recent_len,
               int relevant_budget, float bias, int64_t* kept_dev, float* scores_dev, void* stream);
/* window_mean_scores (policies.py:130-147) + bias_vector (150-162) on device:
 * writes biased (bias applied) or raw scores [n-l]. */
int skv_window_scores(const float* rows_dev, int row_stride, const int32_t* lens_dev, int m, int n,
                      int recent_len, float bias, int apply_bias, float* scores_dev, void* stream);
/* In-place stable row compaction (gather_keep, cache.py:151-156) of `blocks`
 * independent row arrays: block b starts at base_dev + b*block_stride bytes, row
 * i is row_bytes wide; row i <- row kept[i] for i < m.  kept ascending, unique. */
int skv_gather_rows(void* base_dev, int64_t block_stride, int blocks, int row_bytes, const int64_t* kept_dev,
                    int m, void* stream);
/* Single-query attention over one layer: keys/values [H][n][D] f32 (stride
 * row_stride rows between heads), q [H][D] f32 -> probs [H][n], out [H][D]
 * (Session._attend, engine.py:235-246; tensorops.attn_probs/weighted_sum). */
int skv_attend(const float* keys_dev, const float* values_dev, int heads, int n, int head_dim,
               int64_t head_stride, const float* q_dev, float* probs_dev, float* out_dev, void* stream);

/* ---- single-row tensor ops (tensorops.py:26-111) --------------------------
 * Device float32 buffers; the host validates shapes / finiteness (where the
 * reference raises ValueError) before calling. */
/* softmax_row (tensorops.py:26-35): out = exp(x - max) / sum, n >= 1. */
int skv_softmax_row(const float* logits_dev, int n, float* out_dev, void* stream);
/* attn_probs (tensorops.py:86-102): softmax_row((keys @ q) * scale), keys [n][dim]. */
int skv_attn_probs(const float* q_dev, const float* keys_dev, int n, int dim, float scale, float* out_dev,
                   void* stream);
/* weighted_sum (tensorops.py:105-111): out[dim] = probs[n] @ values[n][dim]. */
int skv_weighted_sum(const float* probs_dev, const float* values_dev, int n, int dim, float* out_dev, void* stream);
/* aggregate_heads (policies.py:259-265): probs [heads][n] -> out [n]; mode
 * SKV_AGG_MEAN (sequential f32 head sum / heads) or SKV_AGG_MAX. */
int skv_aggregate_heads(const float* probs_dev, int heads, int n, int mode, float* out_dev, void* stream);
/* bias_vector (policies.py:150-162): out [n - recent_len] f32. */
int skv_bias_vector(int n, int recent_len, float bias, float* out_dev, void* stream);
/* rope_apply (tensorops.py:38-64): pairs rotated by position * base^(-2i/dim)
 * (angles in float64); synchronous. */
int skv_rope_apply(const float* v_dev, int dim, int64_t position, double base, float* out_dev, void* stream);

/* ---- batched trace replay (replay.py:72-180) --------
 * One trace layer's device state: its virtual cache of surviving stream column
 * ids, the window of projected rows (AttentionWindow(recent_len)) and, for the
 * heavy hitter, the accumulator plus staging rows.  All device pointers. */
typedef struct skv_replay_state {
  int64_t* live;      /* [cap] surviving stream column ids */
  float* ring;        /* [window][cap] projected rows */
  int32_t* ring_len;  /* [window] row lengths */
  int32_t* newlen;    /* [window] scratch: lengths after a remap */
  float* acc;         /* [cap] heavy-hitter accumulator, or null (not tracked) */
  float* stage;       /* [stage_rows][cap] projected rows of one batch (heavy hitter) */
  int32_t stage_rows;
  int32_t cap;        /* max live columns */
  int32_t window;     /* ring rows (= recent_len) */
} skv_replay_state;
/* Push R recorded rows of one layer (trace_rows + row_off[i], row_n[i] floats,
 * oldest first): each is projected onto live = live[0, nl_dec) ++ [n_dec, n_i)
 * and renormalised (f64 total), the last min(R, window) enter the ring from
 * slot ring_head on, and (acc != null) heavy_hitter_accumulate runs over all R
 * starting from an accumulator of acc_len columns. */
int skv_replay_rows(const skv_replay_state* st, const float* trace_rows, const int64_t* row_off,
                    const int32_t* row_n, int R, int nl_dec, int n_dec, int ring_head, int acc_len, void* stream);
/* One decision of a replayed layer: the policy (SKV_POLICY_*) over n live
 * columns and the ring (oldest at ring_head - ring_count), then the round's
 * metrics from the nraw raw rows (retained mass per row -> mass_out[nraw] f64;
 * counts_out[0] = |chosen relevant ids (first rc kept) & oracle top-r| or -1,
 * counts_out[1] = planted ids kept), then the remap of live ids, accumulator
 * and ring rows.  kept_out [r+l] int64 receives the kept indices (into live);
 * scores [>= max(n, stream_n)] f32 and top [relevant_budget] i32 are scratch.
 * Returns the kept count. */
/* A round's quality metrics on the device (metrics.py:46-73; the Session's
 * oracle metrics engine.py:314-331 and replay.py:150-166): kept stream ids
 * live[kept[i]] (i < km; the first rc are the relevant set), nrows scoring
 * rows rows_base + row_off[k] of row_n[k] floats in stream coordinates
 * (oldest first), stream length stream_n.  mass_out[k] = f64 mass of row k
 * on the kept ids; counts_out[0] = |relevant ids & oracle top-r| (-1 when
 * undefined), counts_out[1] = planted ids (truth[ntruth]) among the kept. */
int skv_round_metrics(const int64_t* kept, int km, int rc, const int64_t* live, const float* rows_base,
                      const int64_t* row_off, const int32_t* row_n, int nrows, int stream_n, int recent_len,
                      int relevant_budget, const int64_t* truth, int ntruth, float* scores, int32_t* top,
                      double* mass_out, int32_t* counts_out, void* stream);
int skv_replay_evict(const skv_replay_state* st, int policy, int n, int ring_head, int ring_count, int recent_len,
                     int relevant_budget, int sink_count, float bias, int rc, int64_t* kept_out, float* scores,
                     int32_t* top, const float* trace_rows, const int64_t* raw_off, const int32_t* raw_n, int nraw,
                     int stream_n, const int64_t* truth, int ntruth, double* mass_out, int32_t* counts_out,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STREAMKV_B200_H */
