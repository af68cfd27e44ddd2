// Internal kernel-argument structs and launchers shared by the .cu files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace skv {

// Kernel function attributes (dynamic shared memory opt-in) are per device:
// "set once" flags are kept per device so a process that drives several GPUs
// sets them on each.
constexpr int kMaxDevices = 64;
inline int device_slot() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
// Records the calling thread's error message (skv_last_error) and returns code.
int set_error(int code, const char* msg);

struct DevOnce {
  bool done[kMaxDevices] = {};
  bool& here() { return done[device_slot()]; }
};

// ----------------------------------------------------------------------------
// K1: split-KV flash-decode with fused append, logit record and split combine.
// Element (s, h, t, d) of the K store lives at kc + s*c_ss + h*c_hs + t*D + d.
// ----------------------------------------------------------------------------
struct FoldArgs {
  // Materialise the previous step's head-aggregated row from its recorded
  // logits and (max, sum) stats:  row[j] = agg_h expf(x[h][j]-M_h)/L_h.
  const float* logits;  // [s][hq][j]  (stream stride l_ss, head stride l_hs)
  int64_t l_ss, l_hs;
  const float* stats;   // [s][hq][2]  (stream stride st_ss)
  int64_t st_ss;
  float* rows;          // destination row of stream s: rows + s*r_ss
  int64_t r_ss;
  int32_t* wlen;        // optional: wlen[s*w_ss] = n
  int64_t w_ss;
  float* probs;         // mode 2: per-head probabilities probs + s*p_ss + h*p_hs + j
  int64_t p_ss, p_hs;
  int n;                // row length (0: nothing to fold)
  int mode;             // 0 mean over heads, 1 max over heads, 2 per-head probs
  int agg_div;          // mode 0 divisor (total query heads across shards; 0: Hq)
  int accum;            // heavy hitter: row[j] += value for j < n-1, row[n-1] = value
                        // (heavy_hitter_accumulate, policies.py:234-243)
};

struct AttnArgs {
  int32_t* err;         // sticky device error word (skv_ctx::err_word) or null
  int Hq, Hkv;          // group size G = Hq / Hkv is a template parameter
  int n_old;            // tokens cached before this step
  int append;           // 1: slot n_old is the new token taken from kin/vin
  // dynamic schedule: segment sigma = s*Hkv + g holds nt 32-token tiles split
  // into nc chunks of ch tiles; chunk tickets come from sched[0]; the partial
  // of chunk j of segment sigma lives in part slot sigma*nc + j.
  int nt;               // tiles per segment = ceil(n / 32)
  int ch, nc;           // tiles per chunk, chunks per segment
  int S;                // streams
  int stat;             // 1: static schedule, CTA c runs chunk c (grid = S*Hkv*nc)
  int32_t* sched;       // [4] ticket, grid-barrier and exit counters (zero between launches)
  int32_t* done_self;   // flag mode (else null): set to 1 by the merge kernel when this launch's outputs are complete
  const int32_t* done_prev;  // flag of the preceding merge (null: use griddepcontrol.wait)
  int dctas;            // decode grid size (the merge waits for this many finished CTAs)
  int prefetch;         // producer may stream cached K/V before griddepcontrol.wait
  int qpf;              // consumers prefetch the next chunk's q
  int late;             // dynamic schedule: hand out a segment's last chunk `late` segments later (0: all at the end)
  float scale;          // f32(1/sqrt(D)), engine.py:150
  void* kc;             // K store base (written for the appended row)
  void* vc;
  int64_t c_ss, c_hs;   // stream / head strides (elements)
  const void* q;        // q[s][hq][d]     stride q_ss per stream
  int64_t q_ss;
  const void* kraw;     // RoPE: the raw new k (same layout as kin), stored to kc_raw at slot n_old
  void* kc_raw;
  const void* kin;      // kin[s][g][d]    stride in_ss per stream
  const void* vin;
  int64_t in_ss;
  float* out;           // out[s][hq][d]   stride o_ss per stream
  int64_t o_ss;
  float* logits;        // optional record target [s][hq][j]
  int64_t l_ss, l_hs;
  float* stats;         // [s][hq][2] (M, L) of this step
  int64_t st_ss;
  float* part;          // scratch [sigma*nc + j][G][D + 2]
  int32_t* counters;    // [s*Hkv + g] chunk partials published; reset by the segment's merge CTA
  // appended token metadata
  int64_t* pos;         // pos[s*m_ss + t]
  int8_t* modality;
  int32_t* round_id;
  int64_t m_ss;
  int32_t* len;         // len[s*len_ss] = n after the step
  int64_t len_ss;
  int64_t* next_pos;    // next_pos[s*len_ss]
  const int64_t* pos_in;  // optional device [S] explicit positions
  int32_t round_value;
  FoldArgs fold;        // previous step's row (fold.n == 0: none)
  // tensor-core small-batch path (decode_tc.cu): whole-store views for TMA
  int L, layer, cap;
  const void* kc_base;  // K / V store bases, [total_rows][D]
  const void* vc_base;
  int64_t total_rows;
  unsigned long long* tstamp;  // optional [2]: min CTA start / max CTA end (%globaltimer ns)
  unsigned long long* ctat;    // optional [P][8]: per-CTA timeline (instrumentation)
  unsigned long long* mstamp;  // optional [8]: merge timeline (instrumentation)
  // speculative host steps (skv_host_speculate): this launch runs only if the
  // gate kernel ahead of it on the stream wrote 1 here (else both kernels exit
  // before touching any state)
  const int32_t* gate;
};

cudaError_t launch_decode(int dtype, int head_dim, int group, int ctas, const AttnArgs& a, cudaStream_t st);

// All layers of one token in one persistent launch (decode_tc_layers_kernel):
// AttnArgs describe layer 0; layer l's pointers advance by these strides.
// The segment merge runs inside the kernel (the CTA publishing a segment's
// last chunk merges it) and layer l+1's queries wait for layer l's outputs
// through layer_done[l] -- the model's layer-to-layer dependency, with no
// launch boundary on the chain.
struct LayerSteps {
  int L;                      // layers of the launch (layer 0 = args' layer)
  int64_t q_ls, in_ls, o_ls;  // elements between layers of q / new k,v / out
  int64_t kv_ls;              // K/V store elements between layers (kc, vc)
  int64_t m_ls;               // token metadata elements between layers
  int64_t lg_ls, st_ls;       // recorded logits / (max, sum) stats floats between layers
  int64_t fr_ls, fw_ls;       // pending fold: window row floats / lengths between layers
  int32_t* seg_count;         // [S*Hkv] published chunks (reset by the merging CTA)
  int32_t* layer_done;        // [L] merged segments per layer (reset by the last CTA out)
  int32_t* exit_count;        // [1]
  int prefetch0;              // 1: layer 0's cached K/V may stream before griddepcontrol.wait
  unsigned long long* tl;     // instrumentation (null: off): [L][148][16] %globaltimer per CTA and layer
  int late_prefetch;          // cluster kernel: 0 V after P.V, K after the combine; 1 both after the merge; 2 K after the merge
};
cudaError_t launch_decode_tc_layers(int group, int ctas, const AttnArgs& a, const LayerSteps& ls, cudaStream_t st);
// cluster variant: a.nc (<= 16) CTAs per segment form a cluster, chunks of up
// to mt (4..7) tiles; with max_clusters set, only reports how many such
// clusters can be co-resident
cudaError_t launch_decode_tc_cluster(int group, int mt, const AttnArgs& a, const LayerSteps& ls, cudaStream_t st,
                                     int* max_clusters = nullptr);
// dynamic-schedule launches (bf16, D = 128, any group) on mma.sync: decode_tcd_kernel + merge
cudaError_t launch_decode_tcd(int group, int ctas, const AttnArgs& a, cudaStream_t st);
// static-schedule GQA launches (bf16, D = 128, group 4 or 8, chunks <= 4 tiles) on mma.sync
cudaError_t launch_decode_tc(int group, int ctas, const AttnArgs& a, cudaStream_t st);
// the segment merge alone (PDL), after a decode launch
// Speculative host steps (skv_host_speculate): the gate kernel first copies
// the step ahead's outputs (out_src, device) to the host (out_dst, mapped) and
// signals `signal_tick` as done, then one thread waits for the host to ring
// `tick` (GO), cancel it, or `timeout_ns` to pass, and writes the decision to
// *gate (1 go, 2 cancelled, 3 expired); a GO copies the step's inputs from
// in_src (mapped) to in_dst (device).  hostw (mapped pinned): [0] bell,
// [1] done, [2] expired; *broken (device) = generation whose chain expired.
struct SpecGate {
  volatile int32_t* hostw;
  int32_t* gate;
  int32_t* broken;
  int signal_tick, tick, gen;
  long long timeout_ns;
  const int4* in_src;
  int4* in_dst;
  int in_vec;
  const int4* out_src;
  int4* out_dst;
  int out_vec;
  unsigned long long* dbg;  // probe: [64][4] gate start / go / signalled
};
cudaError_t launch_spec_gate(const SpecGate& g, cudaStream_t st);
cudaError_t launch_merge(int head_dim, int group, const AttnArgs& a, cudaStream_t st);
int decode_ctas_per_sm(int dtype, int head_dim, int group);
int decode_tile_tokens();
cudaError_t launch_fold(int streams, int pieces, const FoldArgs& f, int Hq, cudaStream_t st);

// ----------------------------------------------------------------------------
// K2: window-mean score + bias + radix top-k + recent merge (one CTA per window)
// ----------------------------------------------------------------------------
struct SelectArgs {
  const float* rows;    // rows of window b: rows + b*r_bs + slot*row_stride
  int64_t r_bs;
  int row_stride;
  const int32_t* wlen;  // wlen[b*w_bs + slot]
  int64_t w_bs;
  int ring_head;        // slot of the oldest row = (ring_head - count) mod W
  int count, W;         // rows held, ring size
  int n, l, r;
  float bias;
  int apply_bias;       // 0: raw window-mean scores (window_mean_scores only)
  int32_t* kept32;      // optional [b*k_bs + i] int32
  int64_t* kept64;      // optional int64 (stand-alone API)
  int64_t k_bs;
  float* scores;        // optional [b*s_bs + c]
  int64_t s_bs;
  int32_t* first_moved; // optional [b]: first i with kept[i] != i
  int32_t* newlen;      // optional [b*w_bs + slot] ring lengths after remap
  int scores_only;      // 1: stop after writing scores
  int pad;              // keep-all rows: write -1 into kept[n, pad)
  const float* scores_in;  // optional: window-mean scores given (e.g. reduced across head shards)
  int64_t si_bs;
  int policy;           // SKV_POLICY_* (0 Inf-MLLM, 1 window, 2 sink+recent, 3 heavy hitter)
  int sink;             // sink_count (policy 2)
  const float* acc;     // heavy-hitter accumulators acc + b*acc_bs (policy 3)
  int64_t acc_bs;
  // Slot map (engine evictions): perm + b*pm_bs maps logical slot c -> the
  // physical row holding it (identity beyond the last eviction's kept count).
  // Window rows and accumulators are stored by physical row and read through
  // it.  With `moves` set, the kernel also plans the compaction: the kept
  // tokens whose rows lie at or beyond m move into the rows in [0, m) freed by
  // evicted tokens (moves + b*mv_bs: [count][3] = src row, dst row, logical
  // index; mcount[b] = count) and perm is rewritten for the new order.
  int32_t* perm;
  int64_t pm_bs;
  int32_t* moves;
  int64_t mv_bs;
  int32_t* mcount;      // mcount[b * mc_bs]
  int64_t mc_bs;
};

cudaError_t launch_select(int batches, const SelectArgs& a, cudaStream_t st);
cudaError_t launch_project_row(const float* probs, int n, const int64_t* live, int m, float* out, cudaStream_t st);
cudaError_t launch_masked_row_sums(const float* rows, int row_stride, const int32_t* lens, int m, const int64_t* kept,
                                   int k, double* out, cudaStream_t st);
// heavy_hitter_accumulate (policies.py:234-243): out[j] = row[j] + (j < na ? acc[j] : 0)
cudaError_t launch_hh_accumulate(const float* acc, int na, const float* row, int n, float* out, cudaStream_t st);
cudaError_t launch_topk(const float* scores, int n, int k, int64_t* out, cudaStream_t st);

// ----------------------------------------------------------------------------
// K3: in-place stable compaction dst[i] = src[kept[i]] for i in [first, m)
// ----------------------------------------------------------------------------
struct CompactArgs {
  // KV rows: block (b, h): base + b*kv_bs + h*kv_hs bytes, rows of row_bytes
  char* k;
  char* v;
  int64_t kv_bs, kv_hs;  // bytes
  int heads;
  int row_bytes;
  // metadata per block b
  int64_t* pos;
  int8_t* modality;
  int32_t* round_id;
  int64_t m_bs;          // elements
  // window rows per block b: rows + b*r_bs + slot*row_stride, lengths wlen/newlen
  float* rows;
  int64_t r_bs;
  int row_stride;
  int32_t* wlen;
  const int32_t* newlen;
  int64_t w_bs;
  int W;
  // kept sets
  const int32_t* kept32;
  const int64_t* kept64;
  int64_t k_bs;
  const int32_t* first_moved;  // optional per block
  int m;                 // kept count
  int32_t* len;          // optional len[b*len_bs] = m
  int64_t len_bs;
  float* acc;            // optional heavy-hitter accumulators acc + b*acc_bs, gathered like a row of length n
  int64_t acc_bs;
  char* k_raw;           // RoPE: raw key store (layout of k), gathered too
  int rope_cr;           // RoPE cache-relative: gather raw keys + values only (the rotated
                         // rows are recomputed from the raw ones afterwards)
  // Slot-map compaction (SelectArgs::moves): with `moves` set, K/V (and raw
  // key) rows, window-row values and accumulators move only along the planned
  // (src -> dst) list; token metadata and window lengths are still gathered
  // in logical order from `kept`.
  const int32_t* moves;
  int64_t mv_bs;
  const int32_t* mcount;  // mcount[b * mc_bs]
  int64_t mc_bs;
};

cudaError_t launch_compact(int blocks, const CompactArgs& a, cudaStream_t st);
// p[i] = i % period, i < count (identity slot maps)
cudaError_t launch_iota(int32_t* p, int64_t count, int period, cudaStream_t st);
constexpr int kMaxMapRows = 8192 * 32;  // slot-map engines: capacity bound of the selection's row bitmap

// ----------------------------------------------------------------------------
// K4: chunked prefill attention (tcgen05), bf16, head_dim 128
// ----------------------------------------------------------------------------
struct PrefillArgs {
  int C, n0;            // chunk length; cached tokens before the chunk (chunk k/v already appended)
  int W;                // window rows recorded (the last W queries of the chunk)
  int Hq, Hkv, G;       // heads; G = Hq / Hkv
  int L, layer, cap;    // cache geometry: segment row = ((s*L + layer)*Hkv + g)*cap
  float scale;
  float* out;           // [S][C][Hq][128] f32
  float* lg;            // optional [S][W][Hq][lg_cap] f32 logits of the recorded rows
  int64_t lg_cap;
  float* st;            // optional [S][W][Hq][2] (max, sum)
  unsigned long long* prof;  // optional per-CTA cycle counters [grid][16] (instrumentation)
  int dbg;              // instrumentation: 1 skip softmax math, 2 skip MMAs
  int timeline;         // instrumentation: CTA 0's MMA-thread event timeline into prof
  int* ovf;             // optional: += count of V elements saturated to fp16 (|v| > 65504)
  int split;            // 1: a CTA with one Q tile splits its key tiles over both softmax warpgroups
  int order;            // CTA order: 0 head-major (pairs then the lone tile per head), 1 lone tiles last
  int S;                // streams (CTA order 1)
  int lg_t;             // 1: lg is [S][Hq][lg_cap/4][W][4] raw q.k (unscaled; column quads outermost: the
                        // recorded rows of a warp store 512 contiguous bytes per quad); lg_cap % 128 == 0
  int32_t* meta_len;    // optional (engine chunks): the streams' lengths := meta_n and next
  int64_t* meta_next;   //   original positions += C (stride meta_ss), stored by CTA 0 -- after
  int64_t meta_ss;      //   the chunk's append kernel, which read next_pos, in stream order
  int meta_n;
};

#include <cuda.h>
// 2-D TMA view of a [rows][128] bf16 store, 64-dim x box_rows boxes, 128-byte swizzle
cudaError_t make_kv_map(CUtensorMap* map, const void* base, int64_t rows, int box_rows);

cudaError_t launch_prefill(const void* q, int streams, const void* kbase, const void* vbase, int64_t kv_rows,
                           const PrefillArgs& a, cudaStream_t st);
void set_prefill_profile(unsigned long long* p);
cudaError_t launch_fold_rows(int streams, int rows, const FoldArgs& f, int Hq, int slot0, int Wring, int n_base,
                             int64_t lg_rs, int64_t st_rs, int64_t slot_stride, cudaStream_t st);
// fold of the recorded rows from the column-quad-major layout (PrefillArgs::lg_t)
cudaError_t launch_fold_rows_t(int streams, int rows, const FoldArgs& f, int Hq, int slot0, int Wring, int n_base,
                               int64_t lg_cap, int64_t slot_stride, float scale, cudaStream_t st);
// strides in 16-byte units; ss = stride of len / next_pos between streams
cudaError_t launch_append_chunk(const void* kin, const void* vin, void* kc, void* vc, int64_t c_ss_units,
                                int64_t c_hs_units, int S, int Hkv, int units, int n0, int C, int64_t* pos,
                                int8_t* modality, int32_t* round_id, int64_t m_ss, int64_t* next_pos, int32_t* len,
                                int64_t ss, int mod, int rnd, cudaStream_t st, const void* kraw_in,
                                void* kraw_c);

// ----------------------------------------------------------------------------
// RoPE (RoPE-enabled engines): rotate q / new k, and raw -> rotated key rows
// ----------------------------------------------------------------------------
struct RopeArgs {
  int Hq, Hkv, D;
  int mode;              // 1 cache-relative (position = slot index), 2 original position
  int64_t pos0;          // mode 1: position of token 0 (its cache slot)
  const int64_t* pos_in; // mode 2: explicit positions [S], else next_pos[s * np_ss]
  const int64_t* next_pos;
  int64_t np_ss;
  const double* inv_freq;  // [D/2] base^(-2i/D) in f64 (engine.py:176-178)
  const float* tcos;     // optional [tab_rows][D/2] f32 table for positions < tab_rows
  const float* tsin;
  int64_t tab_rows;
  const void* q;         // [S][T][Hq][D], stream stride q_ss
  void* qr;
  int64_t q_ss;
  const void* k;         // [S][T][Hkv][D], stream stride k_ss
  void* kr;
  int64_t k_ss;
};

struct RopeRowsArgs {
  RopeArgs ra;           // D, inv_freq, tables
  int D;
  const void* raw;       // raw key store, segment (b, h) at raw + b*bs + h*hs (elements)
  void* rot;             // rotated key store, same layout
  int64_t bs, hs;
  int r0, r1;            // rows [r0, r1) (r0 replaced by first[b] when given)
  const int32_t* first;  // optional per block
  const int64_t* pos;    // optional per-row positions pos[b*pos_bs + row] (original mode)
  int64_t pos_bs;
};

cudaError_t launch_rope_tokens(int dtype, int tokens, int streams, const RopeArgs& a, cudaStream_t st);
cudaError_t launch_rope_rows(int dtype, int heads, int blocks, const RopeRowsArgs& a, cudaStream_t st);

}  // namespace skv
