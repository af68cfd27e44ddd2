// KvCache.append (cache.py:112-134) of a decode step's token, shared by the
// decode kernels: the token's k/v row goes to slot n_old of segment sigma and
// (kv-head 0 only) its metadata to the stream's arrays.  The CTA that holds a
// segment's last chunk calls this BEFORE it publishes that chunk's partial, so
// the segment merge -- and therefore the next launch, which is ordered after
// the merge -- always observes the appended row, its metadata and len/next_pos.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "skv_internal.h"

namespace skv {

template <typename T, int D>
__device__ __forceinline__ void append_row(const AttnArgs& a, int sigma, int n, int t, int nthreads) {
  constexpr int U = D * (int)sizeof(T) / 16;  // 16-byte units per row
  const int s = sigma / a.Hkv, g = sigma - s * a.Hkv;
  const int64_t dst = s * a.c_ss + (int64_t)g * a.c_hs + (int64_t)a.n_old * D;
  const int64_t in = s * a.in_ss + (int64_t)g * D;
  for (int q16 = t; q16 < U; q16 += nthreads) {
    reinterpret_cast<uint4*>(static_cast<T*>(a.kc) + dst)[q16] =
        reinterpret_cast<const uint4*>(static_cast<const T*>(a.kin) + in)[q16];
    reinterpret_cast<uint4*>(static_cast<T*>(a.vc) + dst)[q16] =
        reinterpret_cast<const uint4*>(static_cast<const T*>(a.vin) + in)[q16];
    if (a.kraw)  // RoPE: the raw key goes to the raw store (cache.keys())
      reinterpret_cast<uint4*>(static_cast<T*>(a.kc_raw) + dst)[q16] =
          reinterpret_cast<const uint4*>(static_cast<const T*>(a.kraw) + in)[q16];
  }
  if (g == 0 && t == 0) {
    int64_t* np = a.next_pos + s * a.len_ss;
    const int64_t pv = a.pos_in ? a.pos_in[s] : *np;
    a.pos[s * a.m_ss + a.n_old] = pv;
    a.modality[s * a.m_ss + a.n_old] = 0;
    a.round_id[s * a.m_ss + a.n_old] = a.round_value;
    *np = pv + 1;
    a.len[s * a.len_ss] = n;
  }
  // no fence here: the caller's barrier (__syncwarp / bar.sync) followed by the
  // gpu-scope release add of the chunk count is cumulative over these stores,
  // exactly as it is for the chunk partial itself
}

}  // namespace skv
