"""Drive the CPU oracle over a golden case with the same logging schema as
``tests/golden/make_golden.py`` (test infrastructure)."""

from __future__ import annotations

import hashlib

import numpy as np

from oracle.streamkv_oracle import PolicyConfig, StreamOracle
from tests.golden.cases import CASES, case_inputs

F32 = np.float32


def run_oracle_case(name: str, kept_override=None) -> dict:
    """Run the oracle on a case.

    ``kept_override(t, s, layer, cpu_kept, cpu_scores, n)`` may return the kept
    set to apply instead of the oracle's (used to continue from the GPU's
    decisions so an allowed near-tie cannot cascade).
    """
    c = CASES[name]
    policy = c.get("policy", "inf_mllm")
    cfg = PolicyConfig(recent_len=c["l"], relevant_budget=c["r"], bias=c["b"], sink_count=c.get("sink", 4),
                       head_agg=c.get("head_agg", "mean"))
    orc = StreamOracle(c["S"], c["L"], c["Hq"], c["Hkv"], c["D"], cfg, window=c["W"], policy=policy,
                       rope=c.get("rope"), rope_base=c.get("rope_base", 10000.0))
    if c.get("shadow"):
        orc.enable_shadow()
    shadow_mass, shadow_overlap = [], []
    q_all, k_all, v_all = case_inputs(name)
    T = q_all.shape[0]
    out_steps, outs = [], []
    kept_log, score_log, evict_steps = [], [], []
    for t in range(T):
        step_out = np.zeros((c["L"], c["S"], c["Hq"], c["D"]), dtype=F32)
        for layer in range(c["L"]):
            o, _ = orc.step_layer(layer, q_all[t, layer], k_all[t, layer], v_all[t, layer])
            step_out[layer] = o
        orc.pos = [t + 1] * c["S"]
        if t % c["out_every"] == 0 or t == T - 1:
            out_steps.append(t)
            outs.append(step_out)
        if (t + 1) % c["E"] == 0:
            evict_steps.append(t)
            for s in range(c["S"]):
                for layer in range(c["L"]):
                    n = orc.length(s, layer)
                    if n <= cfg.budget or policy in ("window", "sink_recent", "none"):
                        sc = np.zeros(0, F32)
                    elif policy == "heavy_hitter":
                        sc = orc.acc[s][layer][: n - cfg.recent_len].copy()
                    else:
                        sc = orc.scores(s, layer)
                    dec = orc.decide(s, layer)
                    kept = dec.kept
                    if orc.shadow:
                        mass, ov = orc.shadow_metrics(s, layer, dec)
                        shadow_mass.append(mass)
                        shadow_overlap.append(np.nan if ov is None else ov)
                    if kept_override is not None:
                        kept = kept_override(t, s, layer, kept, sc, n)
                    kept_log.append(np.asarray(kept).astype(np.int32))
                    score_log.append(sc.astype(F32))
                    orc.apply(s, layer, kept)
    final_keys = np.stack([np.stack([orc.kv[s][layer].keys() for layer in range(c["L"])])
                           for s in range(c["S"])])
    final_pos = np.stack([np.stack([orc.kv[s][layer].pos[: orc.kv[s][layer].n] for layer in range(c["L"])])
                          for s in range(c["S"])])
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
        oracle=orc,
    )
