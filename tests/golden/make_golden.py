"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the dev container only (the reference is not present on GPU boxes):

    python tests/golden/make_golden.py

It imports ``streamkv`` from /root/reference/pkg/src and drives the hot path
exactly as SURVEY.md 7.1/8c describe (KvCache.append -> Session._attend ->
aggregate_heads -> AttentionWindow(W).push per step; every E steps
inf_mllm_decide -> gather_keep -> remap).  Inputs come from the seeded
recipes in ``oracle/streamkv_oracle.py`` so tests can regenerate them.  The
outputs are written to ``tests/golden/*.npz`` and committed; the oracle is
checked against them in ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import types  # noqa: E402

from streamkv.cache import KvCache, PositionMode, TokenMeta  # noqa: E402  (reference)
from collections import deque  # noqa: E402

from streamkv.engine import Session  # noqa: E402
from streamkv.metrics import retained_mass, topk_overlap  # noqa: E402
from streamkv.policies import (  # noqa: E402
    AttentionWindow,
    PolicyConfig,
    aggregate_heads,
    bias_vector,
    heavy_hitter_accumulate,
    heavy_hitter_decide,
    inf_mllm_decide,
    sink_recent_decide,
    sliding_window_decide,
    top_k_indices,
    window_mean_scores,
)

from tests.golden.cases import CASES, case_inputs, kat_instances  # noqa: E402

F32 = np.float32


class _ScaleHolder:
    def __init__(self, head_dim):
        self._scale = F32(1.0 / np.sqrt(head_dim))


def run_reference_case(name: str) -> dict:
    c = CASES[name]
    S, L, Hq, Hkv, D = c["S"], c["L"], c["Hq"], c["Hkv"], c["D"]
    G = Hq // Hkv
    policy = c.get("policy", "inf_mllm")
    cfg = PolicyConfig(recent_len=c["l"], relevant_budget=c["r"], bias=c["b"], sink_count=c.get("sink", 4),
                       head_agg=c.get("head_agg", "mean"))
    holder = _ScaleHolder(D)
    caches = [KvCache(L, Hkv, D) for _ in range(S)]
    windows = [[AttentionWindow(c["W"]) for _ in range(L)] for _ in range(S)]
    accs = [[np.zeros(0, dtype=F32) for _ in range(L)] for _ in range(S)]  # engine.py:274
    rope = c.get("rope")
    if rope:
        # the reference Session's rotary helpers on a holder with their state
        # (engine.py:175-180 init, 198-233 helpers)
        rot = types.SimpleNamespace()
        half = D // 2
        rot._inv_freq = c["rope_base"] ** (-2.0 * np.arange(half, dtype=np.float64) / D)
        rot._cos = np.zeros((0, half), dtype=F32)
        rot._sin = np.zeros((0, half), dtype=F32)
        rot._trig = types.MethodType(Session._trig, rot)
        mode = PositionMode.CACHE_RELATIVE if rope == "cache_relative" else PositionMode.ORIGINAL
        rstore = [[np.zeros((Hkv, 0, D), dtype=F32) for _ in range(L)] for _ in range(S)]
    # Session(oracle=True)'s shadow: a never-evicted cache and the last
    # recent_len head-aggregated rows over it (engine.py:142-151, 275-284)
    shadow = c.get("shadow", False)
    if shadow:
        scaches = [KvCache(L, Hkv, D) for _ in range(S)]
        srows = [[deque(maxlen=c["l"]) for _ in range(L)] for _ in range(S)]
    shadow_mass, shadow_overlap = [], []
    q_all, k_all, v_all = case_inputs(name)  # (T, L, S, H, D)
    T = q_all.shape[0]
    out_steps = []
    outs = []
    kept_log, score_log, evict_steps = [], [], []
    for t in range(T):
        step_out = np.zeros((L, S, Hq, D), dtype=F32)
        for layer in range(L):
            for s in range(S):
                caches[s].append(layer, k_all[t, layer, s], v_all[t, layer, s], TokenMeta(t))
                keys = caches[s].keys(layer)
                vals = caches[s].values(layer)
                qv = q_all[t, layer, s]
                if rope:  # engine.py:265-268
                    n = caches[s].length(layer)
                    p = n - 1 if mode == PositionMode.CACHE_RELATIVE else t
                    rk = Session._rotate_one(rot, k_all[t, layer, s], p)
                    rstore[s][layer] = np.concatenate([rstore[s][layer], rk[:, None, :]], axis=1)
                    keys = rstore[s][layer]
                    qv = Session._rotate_one(rot, qv, p)
                if G > 1:
                    keys = np.repeat(keys, G, axis=0)
                    vals = np.repeat(vals, G, axis=0)
                probs, o = Session._attend(holder, keys, vals, qv)
                row = aggregate_heads(probs, cfg.head_agg)  # engine.py:272
                windows[s][layer].push(row)
                accs[s][layer] = heavy_hitter_accumulate(accs[s][layer], row)
                step_out[layer, s] = o
                if shadow:
                    scaches[s].append(layer, k_all[t, layer, s], v_all[t, layer, s], TokenMeta(t))
                    sk, sv = scaches[s].keys(layer), scaches[s].values(layer)
                    if G > 1:
                        sk, sv = np.repeat(sk, G, axis=0), np.repeat(sv, G, axis=0)
                    sprobs, _ = Session._attend(holder, sk, sv, q_all[t, layer, s])
                    srows[s][layer].append(aggregate_heads(sprobs, cfg.head_agg))
        if t % c["out_every"] == 0 or t == T - 1:
            out_steps.append(t)
            outs.append(step_out)
        if (t + 1) % c["E"] == 0:
            evict_steps.append(t)
            for s in range(S):
                for layer in range(L):
                    n = caches[s].length(layer)
                    sc = np.zeros(0, dtype=F32)
                    # the Session's policy switch, engine.py:296-307
                    if policy == "heavy_hitter":
                        if n > cfg.budget:
                            sc = accs[s][layer][: n - cfg.recent_len].copy()
                        d = heavy_hitter_decide(accs[s][layer], n, cfg.relevant_budget, cfg.recent_len)
                    elif policy == "window":
                        d = sliding_window_decide(n, cfg.budget)
                    elif policy == "sink_recent":
                        d = sink_recent_decide(n, cfg.sink_count, cfg.budget)
                    else:
                        if n > cfg.budget:
                            sc = window_mean_scores(windows[s][layer], n, cfg.recent_len) + bias_vector(
                                n, cfg.recent_len, cfg.bias
                            )
                        d = inf_mllm_decide(windows[s][layer], n, cfg)
                    kept_log.append(d.kept.astype(np.int32))
                    score_log.append(sc.astype(F32))
                    if shadow:  # _evict_layer's oracle metrics, engine.py:314-331
                        orig = caches[s].original_positions(layer)
                        kept_ids, relevant_ids = orig[d.kept], orig[d.relevant]
                        rows = list(srows[s][layer])
                        shadow_mass.append(retained_mass(rows, kept_ids))
                        ov = np.nan
                        ns = scaches[s].length(layer)
                        if ns > cfg.recent_len and cfg.relevant_budget >= 1:
                            cols = ns - cfg.recent_len
                            acc = np.zeros(cols, dtype=F32)
                            for row in rows:
                                m = min(row.size, cols)
                                acc[:m] += row[:m]
                            ov = topk_overlap(acc / F32(len(rows)), relevant_ids, cfg.relevant_budget)
                        shadow_overlap.append(ov)
                    if d.kept.size != n:
                        caches[s].gather_keep(layer, d.kept)
                        windows[s][layer].remap(d.kept)
                        accs[s][layer] = accs[s][layer][d.kept]  # engine.py:335
                        if rope:  # _refresh_rotations, engine.py:339-342
                            rstore[s][layer] = Session._rotate_many(
                                rot, caches[s].keys(layer), caches[s].positions_for(layer, mode))
    final_keys = np.stack([np.stack([caches[s].keys(layer) for layer in range(L)]) for s in range(S)])
    final_pos = np.stack([np.stack([caches[s].original_positions(layer) for layer in range(L)]) for s in range(S)])
    return dict(
        out_steps=np.asarray(out_steps, np.int32),
        outs=np.stack(outs),
        evict_steps=np.asarray(evict_steps, np.int32),
        kept_off=np.cumsum([0] + [k.size for k in kept_log]).astype(np.int64),
        kept=np.concatenate(kept_log) if kept_log else np.zeros(0, np.int32),
        score_off=np.cumsum([0] + [s.size for s in score_log]).astype(np.int64),
        scores=np.concatenate(score_log) if score_log else np.zeros(0, F32),
        final_keys_sha=np.frombuffer(hashlib.sha256(final_keys.tobytes()).digest(), np.uint8),
        final_pos=final_pos,
        shadow_mass=np.asarray(shadow_mass, np.float64),
        shadow_overlap=np.asarray(shadow_overlap, np.float64),
    )


def run_kats() -> dict:
    """Algorithm-1 known answers on the acceptance-test instance recipe."""
    kept_log, score_sha = [], []
    for inst in kat_instances():
        w = AttentionWindow(len(inst["rows"]))
        for row in inst["rows"]:
            w.push(row)
        cfg = PolicyConfig(recent_len=inst["l"], relevant_budget=inst["r"], bias=inst["b"])
        d = inf_mllm_decide(w, inst["n"], cfg)
        kept_log.append(d.kept.astype(np.int32))
        if inst["n"] > inst["l"]:
            sc = window_mean_scores(w, inst["n"], inst["l"]) + bias_vector(inst["n"], inst["l"], inst["b"])
        else:
            sc = np.zeros(0, F32)
        score_sha.append(np.frombuffer(hashlib.sha256(sc.astype(F32).tobytes()).digest(), np.uint8))
    topk = []
    rng = np.random.default_rng(23)
    for _ in range(200):
        size = int(rng.integers(1, 50))
        scores = rng.choice([0.1, 0.2, 0.3, 0.5], size=size).astype(F32)
        k = int(rng.integers(0, size + 1))
        topk.append(top_k_indices(scores, k).astype(np.int32))
    return dict(
        kept_off=np.cumsum([0] + [k.size for k in kept_log]).astype(np.int64),
        kept=np.concatenate(kept_log),
        score_sha=np.stack(score_sha),
        topk_off=np.cumsum([0] + [t.size for t in topk]).astype(np.int64),
        topk=np.concatenate(topk),
    )


def main():
    only = set(sys.argv[1:])  # optional: regenerate just these cases
    for name in CASES:
        if only and name not in only:
            continue
        res = run_reference_case(name)
        np.savez_compressed(os.path.join(HERE, f"ref_{name}.npz"), **res)
        print(name, "evictions", res["evict_steps"].size, "kept entries", res["kept"].size)
    if only:
        return
    kat = run_kats()
    np.savez_compressed(os.path.join(HERE, "ref_kat_algorithm1.npz"), **kat)
    print("kat", kat["kept_off"].size - 1)


if __name__ == "__main__":
    main()
