"""Seeded input recipes shared by the golden generator and the tests.

Shapes follow BASELINE.json configs (reduced in layers/streams/tokens where
the CPU oracle would otherwise take minutes).  Everything is regenerated from
seeds; only the reference's outputs are stored in ``tests/golden/*.npz``.
"""

from __future__ import annotations

import numpy as np

from oracle.streamkv_oracle import bf16_round

F32 = np.float32

CASES = {
    # BASELINE config 0 in full: 1 layer, 8 heads, D=64, fp32, 4096 tokens,
    # 4 saddle keys x6, budget 128 recent + 128 relevant, W=32, b=0.01, E=64.
    "cfg0": dict(S=1, L=1, Hq=8, Hkv=8, D=64, T=4096, l=128, r=128, W=32, b=0.01, E=64,
                 dtype="f32", seed=1000, saddles=4, saddle_gain=6.0, spike_prob=0.0,
                 spike_gain=1.0, out_every=64),
    # config-1 shape per head (32 x 128, bf16, 1% x4 key spikes), reduced budget.
    "cfg1_mini": dict(S=2, L=2, Hq=32, Hkv=32, D=128, T=640, l=128, r=128, W=32, b=0.01, E=128,
                      dtype="bf16", seed=1001, saddles=0, saddle_gain=1.0, spike_prob=0.01,
                      spike_gain=4.0, out_every=128),
    # config-3 GQA grouping (4 query heads per KV head), reduced.
    "gqa_mini": dict(S=1, L=2, Hq=8, Hkv=2, D=128, T=448, l=64, r=64, W=32, b=0.01, E=64,
                     dtype="bf16", seed=1003, saddles=0, saddle_gain=1.0, spike_prob=0.005,
                     spike_gain=4.0, out_every=32),
    # window longer than the eviction period: exercises window remap.
    "wide_window": dict(S=1, L=1, Hq=4, Hkv=4, D=64, T=320, l=16, r=32, W=40, b=0.1, E=16,
                        dtype="f32", seed=1004, saddles=3, saddle_gain=5.0, spike_prob=0.0,
                        spike_gain=1.0, out_every=16),
    # The Session's comparison baselines (engine.py:296-307):
    # heavy-hitter accumulated mass, sliding window, sink + recent.
    "hh_mini": dict(S=1, L=2, Hq=8, Hkv=8, D=64, T=384, l=32, r=32, W=16, b=0.01, E=32,
                    dtype="f32", seed=1005, saddles=4, saddle_gain=5.0, spike_prob=0.0,
                    spike_gain=1.0, out_every=32, policy="heavy_hitter"),
    "hh_gqa_bf16": dict(S=2, L=1, Hq=8, Hkv=2, D=128, T=320, l=48, r=80, W=16, b=0.01, E=64,
                        dtype="bf16", seed=1006, saddles=0, saddle_gain=1.0, spike_prob=0.01,
                        spike_gain=4.0, out_every=64, policy="heavy_hitter"),
    "window_mini": dict(S=1, L=1, Hq=4, Hkv=4, D=64, T=256, l=32, r=32, W=16, b=0.01, E=32,
                        dtype="bf16", seed=1007, saddles=0, saddle_gain=1.0, spike_prob=0.0,
                        spike_gain=1.0, out_every=32, policy="window"),
    "sink_mini": dict(S=2, L=1, Hq=4, Hkv=2, D=128, T=256, l=24, r=40, W=16, b=0.01, E=32,
                      dtype="bf16", seed=1008, saddles=0, saddle_gain=1.0, spike_prob=0.0,
                      spike_gain=1.0, out_every=32, policy="sink_recent", sink=4),
    # Rotary positions driven through the reference Session's own rotary
    # helpers (engine.py:198-233, 339-342): pre-rotation q/k inputs, raw keys
    # cached, cache-relative re-rotation after every compaction / original
    # stream positions.  f32 so the reference's rotated keys are reproduced.
    "rope_cr": dict(S=1, L=2, Hq=4, Hkv=4, D=64, T=256, l=32, r=32, W=16, b=0.01, E=32,
                    dtype="f32", seed=1009, saddles=3, saddle_gain=5.0, spike_prob=0.0,
                    spike_gain=1.0, out_every=32, rope="cache_relative", rope_base=10000.0),
    "rope_orig_gqa": dict(S=2, L=1, Hq=8, Hkv=2, D=128, T=224, l=32, r=48, W=16, b=0.01, E=32,
                          dtype="f32", seed=1010, saddles=0, saddle_gain=1.0, spike_prob=0.01,
                          spike_gain=4.0, out_every=32, rope="original", rope_base=500000.0),
    # aggregate_heads(.., "max") (policies.py:263-264) through the Session's
    # head_agg switch (engine.py:272): GQA bf16 and f32 with saddle keys.
    "max_mini": dict(S=2, L=2, Hq=8, Hkv=2, D=128, T=320, l=48, r=48, W=16, b=0.01, E=64,
                     dtype="bf16", seed=1011, saddles=0, saddle_gain=1.0, spike_prob=0.01,
                     spike_gain=4.0, out_every=64, head_agg="max"),
    "max_f32": dict(S=1, L=1, Hq=8, Hkv=8, D=64, T=256, l=32, r=32, W=32, b=0.01, E=32,
                    dtype="f32", seed=1012, saddles=3, saddle_gain=6.0, spike_prob=0.0,
                    spike_gain=1.0, out_every=32, head_agg="max"),
    # Session(oracle=True)'s live quality metrics against a never-evicted
    # shadow cache (engine.py:275-284, 314-331): retained mass and top-r
    # overlap at every eviction.
    "shadow_mini": dict(S=2, L=2, Hq=8, Hkv=2, D=64, T=384, l=32, r=32, W=16, b=0.01, E=64,
                        dtype="f32", seed=1013, saddles=4, saddle_gain=6.0, spike_prob=0.0,
                        spike_gain=1.0, out_every=64, shadow=True),
    # eight query heads per KV head (the widest GQA group the kernels take), bf16
    "gqa8_bf16": dict(S=2, L=2, Hq=16, Hkv=2, D=128, T=320, l=40, r=56, W=24, b=0.05, E=48,
                      dtype="bf16", seed=1014, saddles=0, saddle_gain=1.0, spike_prob=0.01,
                      spike_gain=4.0, out_every=48),
    # a long run with a short period: ~100 evictions, a large age bias
    "long_f32": dict(S=1, L=1, Hq=4, Hkv=4, D=64, T=1024, l=24, r=40, W=8, b=0.2, E=10,
                     dtype="f32", seed=1015, saddles=5, saddle_gain=5.0, spike_prob=0.0,
                     spike_gain=1.0, out_every=64),
}


def case_inputs(name: str):
    """Return q (T,L,S,Hq,D), k/v (T,L,S,Hkv,D) float32 for a case."""
    c = CASES[name]
    rng = np.random.default_rng(c["seed"])
    T, L, S, Hq, Hkv, D = c["T"], c["L"], c["S"], c["Hq"], c["Hkv"], c["D"]
    q = rng.standard_normal((T, L, S, Hq, D)).astype(F32)
    k = rng.standard_normal((T, L, S, Hkv, D)).astype(F32)
    v = rng.standard_normal((T, L, S, Hkv, D)).astype(F32)
    if c["saddles"]:
        pos = rng.choice(T, size=c["saddles"], replace=False)
        k[pos] *= F32(c["saddle_gain"])
    if c["spike_prob"] > 0:
        spikes = rng.random((T, L, S)) < c["spike_prob"]
        k[spikes] *= F32(c["spike_gain"])
    if c["dtype"] == "bf16":
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v


def kat_instances(count: int = 1000, seed: int = 20_26):
    """Algorithm-1 instances, drawn like the reference acceptance test
    (test_acceptance.py:39-68): ragged Dirichlet windows, n<=256, l<=32,
    r<=64, b in {0, 1e-3, 0.1, 1}."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(2, 257))
        l = int(rng.integers(1, 33))
        r = int(rng.integers(0, 65))
        b = float(rng.choice([0.0, 0.001, 0.1, 1.0]))
        m = int(rng.integers(1, l + 1))
        lengths = np.sort(rng.integers(1, n + 1, size=m))
        lengths[-1] = n
        rows = [rng.dirichlet(np.ones(int(length))).astype(F32) for length in lengths]
        out.append(dict(n=n, l=l, r=r, b=b, rows=rows))
    return out
