// Batched trace replay on the device (the reference's
// replay_trace, /root/reference/pkg/src/streamkv/replay.py:72-180).
//
// No decoder runs: each trace layer keeps a virtual cache of surviving stream
// column ids, a window of projected rows and (heavy hitter) an accumulator.
// The host plans everything from the trace alone -- every quantity that steers
// control flow (row lengths, live counts, kept counts) follows from the row
// sizes -- so the device runs, per layer and decision, one batched launch for
// all rows since the previous decision (projection onto the live columns +
// renormalisation + window push + accumulation), one selection launch (the
// shared select_kernel), one metrics launch and one remap launch, with no
// host synchronisation until the results are read at the end.
//
// Projection (replay.py:139-142): live_i = live_dec ++ [n_dec, n_i) -- the
// newest stream column always survives a decision, so the ids appended since
// it form a contiguous range --, out[j] = f32(f64(probs[live_i[j]]) / total)
// with the f64 total of the projected values (unnormalised when the total is 0).
// Accumulation (policies.py:234-243): acc[j] = row[j] + acc[j] row by row.
// Metrics (metrics.py:46-83): retained mass per raw row (f64 sums over the kept
// stream ids below the row's length), top-r overlap of the chosen relevant ids
// with the window-mean oracle over the raw rows (f32 oldest-first sums, IEEE
// division), planted recall (truth ids among the kept ids).
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/streamkv_b200.h"
#include "skv_common.cuh"
#include "skv_internal.h"
#include "skv_topk.cuh"

namespace skv {

constexpr int kRepThreads = 256;
constexpr int kMetThreads = 1024;

// One CTA per batch row: the projected row goes to the window ring (the last
// `window` rows of the batch) and, for the heavy hitter, to the staging rows.
__global__ void __launch_bounds__(kRepThreads)
    replay_project_kernel(const float* __restrict__ trows, const int64_t* __restrict__ row_off,
                          const int32_t* __restrict__ row_n, int R, const int64_t* __restrict__ live, int nl_dec,
                          int n_dec, float* ring, int32_t* ring_len, int ring_head, int window, int cap, float* stage) {
  __shared__ double part[kRepThreads / 32];
  const int i = blockIdx.x;
  const bool to_ring = i >= R - window;
  if (!to_ring && !stage) return;
  const float* probs = trows + row_off[i];
  const int n = row_n[i];
  const int nl = nl_dec + (n - n_dec);
  auto src = [&](int j) { return j < nl_dec ? live[j] : (int64_t)n_dec + (j - nl_dec); };
  double acc = 0.0;
  for (int j = threadIdx.x; j < nl; j += blockDim.x) acc += (double)probs[src(j)];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  double total = 0.0;
  for (int w = 0; w < kRepThreads / 32; ++w) total += part[w];
  float* rrow = to_ring ? ring + (int64_t)((ring_head + i) % window) * cap : nullptr;
  float* srow = stage ? stage + (int64_t)i * cap : nullptr;
  for (int j = threadIdx.x; j < nl; j += blockDim.x) {
    const double p = (double)probs[src(j)];
    const float v = total > 0.0 ? (float)(p / total) : (float)p;
    if (rrow) rrow[j] = v;
    if (srow) srow[j] = v;
  }
  if (threadIdx.x == 0 && to_ring) ring_len[(ring_head + i) % window] = nl;
  // the batch's last row materialises the stream ids appended since the last
  // decision (live[j] for j >= nl_dec is only read by later launches)
  if (i == R - 1)
    for (int j = nl_dec + threadIdx.x; j < nl; j += blockDim.x) const_cast<int64_t*>(live)[j] = (int64_t)n_dec + (j - nl_dec);
}

// heavy_hitter_accumulate over the batch rows in order: thread j owns column j.
__global__ void replay_accumulate_kernel(float* acc, int acc_len, const float* __restrict__ stage,
                                         const int32_t* __restrict__ row_n, int R, int nl_dec, int n_dec, int cap) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int nl_last = nl_dec + (row_n[R - 1] - n_dec);
  if (j >= nl_last) return;
  bool present = j < acc_len;
  float v = present ? acc[j] : 0.f;
  for (int i = 0; i < R; ++i) {
    const int len = nl_dec + (row_n[i] - n_dec);
    if (j < len) {
      const float x = stage[(int64_t)i * cap + j];
      v = present ? __fadd_rn(x, v) : x;
      present = true;
    }
  }
  acc[j] = v;
}

// One CTA per decision: kept / relevant stream ids, retained mass per raw
// row, oracle top-r overlap, planted recall.
__global__ void __launch_bounds__(kMetThreads)
    replay_metrics_kernel(const int64_t* __restrict__ kept, int km, int rc, const int64_t* __restrict__ live,
                          const float* __restrict__ trows, const int64_t* __restrict__ raw_off,
                          const int32_t* __restrict__ raw_n, int nraw, int stream_n, int l, int r,
                          const int64_t* __restrict__ truth, int ntruth, float* scores, int32_t* top,
                          double* mass_out, int32_t* counts_out) {
  extern __shared__ unsigned bits[];  // [2][words]: kept ids, oracle top-r
  __shared__ TopkSmem sm;
  __shared__ double part[kMetThreads / 32];
  const int tid = threadIdx.x;
  const int words = (stream_n + 31) / 32;
  unsigned* kbits = bits;
  unsigned* tbits = bits + words;
  for (int w = tid; w < 2 * words; w += blockDim.x) bits[w] = 0;
  __syncthreads();
  for (int i = tid; i < km; i += blockDim.x) {
    const int64_t id = live[kept[i]];
    if (id >= 0 && id < stream_n) atomicOr(&kbits[id >> 5], 1u << (id & 31));
  }
  __syncthreads();
  // retained mass: f64 sum of each raw row over the kept ids below its length
  for (int k = 0; k < nraw; ++k) {
    const float* row = trows + raw_off[k];
    const int len = min(raw_n[k], stream_n);
    double acc = 0.0;
    for (int c = tid; c < len; c += blockDim.x)
      if ((kbits[c >> 5] >> (c & 31)) & 1u) acc += (double)row[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) part[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kMetThreads / 32; ++w) t += part[w];
      mass_out[k] = t;
    }
    __syncthreads();
  }
  // planted recall: truth ids among the kept ids
  int hits = 0;
  for (int t = tid; t < ntruth; t += blockDim.x) {
    const int64_t id = truth[t];
    hits += (id >= 0 && id < stream_n) ? (int)((kbits[id >> 5] >> (id & 31)) & 1u) : 0;
  }
  int hits_total;
  block_excl_scan(hits, sm.scan, hits_total);
  // top-r overlap against the window-mean oracle over the raw rows
  int overlap = -1;
  if (stream_n > l && r >= 1) {
    const int cols = stream_n - l;
    const float inv = (float)nraw;
    for (int c = tid; c < cols; c += blockDim.x) {
      float acc = 0.f;
      for (int k = 0; k < nraw; ++k)
        if (c < raw_n[k]) acc = __fadd_rn(acc, trows[raw_off[k] + c]);
      scores[c] = __fdiv_rn(acc, inv);
    }
    __syncthreads();
    const int kk = min(r, cols);
    if (kk < cols) {
      topk_block(scores, cols, kk, top, nullptr, sm);
      for (int i = tid; i < kk; i += blockDim.x) atomicOr(&tbits[top[i] >> 5], 1u << (top[i] & 31));
    } else {
      for (int c = tid; c < cols; c += blockDim.x) atomicOr(&tbits[c >> 5], 1u << (c & 31));
    }
    __syncthreads();
    int ov = 0;
    for (int i = tid; i < rc; i += blockDim.x) {  // chosen relevant ids (distinct)
      const int64_t id = live[kept[i]];
      ov += (id >= 0 && id < cols) ? (int)((tbits[id >> 5] >> (id & 31)) & 1u) : 0;
    }
    int ov_total;
    block_excl_scan(ov, sm.scan, ov_total);
    overlap = ov_total;
  }
  if (tid == 0) {
    counts_out[0] = overlap;
    counts_out[1] = hits_total;
  }
}

}  // namespace skv

using namespace skv;

extern "C" {

int skv_replay_rows(const skv_replay_state* st, const float* trace_rows, const int64_t* row_off,
                    const int32_t* row_n, int R, int nl_dec, int n_dec, int ring_head, int acc_len, void* stream) {
  if (!st || !trace_rows || !row_off || !row_n) return set_error(SKV_EINVAL, "null argument");
  if (R <= 0) return SKV_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* stage = st->acc ? st->stage : nullptr;
  if (st->acc && (!st->stage || R > st->stage_rows)) return set_error(SKV_EINVAL, "staging rows too small");
  replay_project_kernel<<<R, kRepThreads, 0, s>>>(trace_rows, row_off, row_n, R, st->live, nl_dec, n_dec, st->ring,
                                                  st->ring_len, ring_head, st->window, st->cap, stage);
  if (cudaGetLastError() != cudaSuccess) return set_error(SKV_ECUDA, "replay projection launch");
  if (st->acc) {
    replay_accumulate_kernel<<<(st->cap + 255) / 256, 256, 0, s>>>(st->acc, acc_len, stage, row_n, R, nl_dec, n_dec,
                                                                   st->cap);
    if (cudaGetLastError() != cudaSuccess) return set_error(SKV_ECUDA, "replay accumulate launch");
  }
  return SKV_OK;
}

int skv_round_metrics(const int64_t* kept, int km, int rc, const int64_t* live, const float* rows_base,
                      const int64_t* row_off, const int32_t* row_n, int nrows, int stream_n, int recent_len,
                      int relevant_budget, const int64_t* truth, int ntruth, float* scores, int32_t* top,
                      double* mass_out, int32_t* counts_out, void* stream) {
  if (!kept || !live || !rows_base || !row_off || !row_n || !scores || !top || !mass_out || !counts_out)
    return set_error(SKV_EINVAL, "null argument");
  if (nrows < 1) return set_error(SKV_EINVAL, "retained_mass needs at least one scoring row");
  const int words = (std::max(stream_n, 1) + 31) / 32;
  const size_t smem = 2 * (size_t)words * sizeof(unsigned);
  if (smem > 160 * 1024) return set_error(SKV_EINVAL, "stream too long for the metrics kernel");
  static DevOnce attr;
  if (!attr.here()) {
    cudaFuncSetAttribute(replay_metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr.here() = true;
  }
  replay_metrics_kernel<<<1, kMetThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      kept, km, rc, live, rows_base, row_off, row_n, nrows, stream_n, recent_len, relevant_budget, truth, ntruth,
      scores, top, mass_out, counts_out);
  return cudaGetLastError() == cudaSuccess ? SKV_OK : set_error(SKV_ECUDA, "metrics kernel launch");
}

int skv_replay_evict(const skv_replay_state* st, int policy, int n, int ring_head, int ring_count, int recent_len,
                     int relevant_budget, int sink_count, float bias, int rc, int64_t* kept_out, float* scores,
                     int32_t* top, const float* trace_rows, const int64_t* raw_off, const int32_t* raw_n, int nraw,
                     int stream_n, const int64_t* truth, int ntruth, double* mass_out, int32_t* counts_out,
                     void* stream) {
  if (!st || !kept_out || !scores || !top || !mass_out || !counts_out) return set_error(SKV_EINVAL, "null argument");
  if (n < 1 || n > st->cap) return set_error(SKV_EINVAL, "live count out of range");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int l = recent_len;
  int r = relevant_budget;
  if (policy == SKV_POLICY_NONE) r = n;  // keep_all
  const int budget = r + l;
  const int km = n <= budget ? n : budget;
  // ---- decision (the engine's select kernel over the replay window)
  if (cudaMemsetAsync(st->newlen, 0, st->window * sizeof(int32_t), s) != cudaSuccess)
    return set_error(SKV_ECUDA, "memset");
  SelectArgs a{};
  a.rows = st->ring;
  a.row_stride = st->cap;
  a.wlen = st->ring_len;
  a.ring_head = ring_head;
  a.count = ring_count;
  a.W = st->window;
  a.n = n;
  a.l = l;
  a.r = r;
  a.bias = bias;
  a.apply_bias = 1;
  a.kept64 = kept_out;
  a.scores = scores;
  a.newlen = st->newlen;
  a.policy = policy == SKV_POLICY_NONE ? SKV_POLICY_INF_MLLM : policy;
  a.sink = sink_count;
  a.acc = st->acc;
  cudaError_t e = launch_select(1, a, s);
  if (e != cudaSuccess) return set_error(SKV_ECUDA, "replay select launch");
  // ---- metrics on the raw rows (before the live ids are remapped)
  const int words = (std::max(stream_n, 1) + 31) / 32;
  const size_t smem = 2 * (size_t)words * sizeof(unsigned);
  if (smem > 160 * 1024) return set_error(SKV_EINVAL, "stream too long for the replay metrics kernel");
  static DevOnce attr;
  if (!attr.here()) {
    cudaFuncSetAttribute(replay_metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr.here() = true;
  }
  replay_metrics_kernel<<<1, kMetThreads, smem, s>>>(kept_out, km, rc, st->live, trace_rows, raw_off, raw_n, nraw,
                                                     stream_n, l, relevant_budget, truth, ntruth, scores, top,
                                                     mass_out, counts_out);
  if (cudaGetLastError() != cudaSuccess) return set_error(SKV_ECUDA, "replay metrics launch");
  // ---- remap: live ids, accumulator and window rows restricted to the kept set
  if (km != n) {
    CompactArgs c{};
    c.heads = 0;
    c.pos = st->live;
    c.m_bs = 0;
    c.acc = st->acc;
    c.rows = st->ring;
    c.row_stride = st->cap;
    c.W = st->window;
    c.wlen = st->ring_len;
    c.newlen = st->newlen;
    c.kept64 = kept_out;
    c.m = km;
    e = launch_compact(1, c, s);
    if (e != cudaSuccess) return set_error(SKV_ECUDA, "replay remap launch");
  }
  return km;
}

}  // extern "C"
