"""Golden fixture for the device trace replay, made
by running the REFERENCE (dev container only):

    python tests/golden/make_replay_golden.py

A planted-pattern trace from the reference generator (traceio.generate_synthetic)
plus extra layers of perturbed rows is serialised with the reference writer;
the reference ``replay_trace`` runs every policy over it.  The trace bytes,
the per-round kept sets and the metric rows go to tests/golden/ref_replay.npz;
a second trace (three layers, longer prompts, a wider budget, its own policy
config stored in the file) to tests/golden/ref_replay2.npz.
"""

from __future__ import annotations

import io
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from streamkv.policies import PolicyConfig  # noqa: E402  (reference)
from streamkv.replay import replay_trace  # noqa: E402
from streamkv.traceio import (  # noqa: E402
    AttnRow,
    SynthConfig,
    TraceHeader,
    generate_synthetic,
    read_trace,
    write_trace,
)

F32 = np.float32
POLICIES = ["inf-mllm", "heavy-hitter", "window", "sink-recent", "none"]
CFG = dict(recent_len=16, relevant_budget=24, bias=0.05, sink_count=3)


CFG2 = dict(recent_len=10, relevant_budget=40, bias=0.02, sink_count=5)


def make_trace(synth, layers: int, heads: int) -> bytes:
    events = []
    for ev in generate_synthetic(synth):
        events.append(ev)
        if isinstance(ev, AttnRow):  # extra layers with different (still normalised) mass
            n = ev.probs.size
            for layer in range(1, layers):
                w = ev.probs.astype(np.float64) * (1.0 + 0.5 * np.sin(np.arange(n) * (0.37 * layer)))
                events.append(AttnRow(layer, (w / w.sum()).astype(F32)))
    buf = io.BytesIO()
    write_trace(buf, TraceHeader(layers=layers, heads=heads), events)
    return buf.getvalue()


def main():
    synth1 = SynthConfig(rounds=9, prompt_len=24, decode_len=20, saddle_count=6, saddle_gain=6.0, shift_every=3,
                         sink_count=2, sink_gain=3.0, recent_gain=2.0, recent_len=12, seed=7)
    synth2 = SynthConfig(rounds=6, prompt_len=40, decode_len=30, saddle_count=9, saddle_gain=4.0, shift_every=2,
                         sink_count=4, sink_gain=2.5, recent_gain=1.5, recent_len=8, seed=19)
    write(make_trace(synth1, 2, 4), CFG, 16, "ref_replay.npz")
    write(make_trace(synth2, 3, 8), CFG2, 32, "ref_replay2.npz")


def write(data: bytes, cfg_kw: dict, head_dim: int, name: str):
    out = {"trace": np.frombuffer(data, dtype=np.uint8),
           "cfg": np.array([cfg_kw["recent_len"], cfg_kw["relevant_budget"], cfg_kw["sink_count"], head_dim],
                           dtype=np.int64),
           "bias": np.array([cfg_kw["bias"]], dtype=np.float64)}
    cfg = PolicyConfig(**cfg_kw)
    for pol in POLICIES:
        header, events = read_trace(io.BytesIO(data))
        res = replay_trace(header, list(events), pol, cfg, head_dim=head_dim)
        kept = [d.kept.astype(np.int32) for rnd in res.decisions_per_round for d in rnd]
        key = pol.replace("-", "_")
        out[f"{key}_kept_off"] = np.cumsum([0] + [k.size for k in kept]).astype(np.int64)
        out[f"{key}_kept"] = np.concatenate(kept) if kept else np.zeros(0, np.int32)
        nan = lambda v: np.nan if v is None else v
        out[f"{key}_metrics"] = np.array([[r.round_id, r.retained_mass, nan(r.topk_overlap), nan(r.planted_recall),
                                           r.cache_len, r.memory_bytes, r.flops_per_token] for r in res.rows],
                                         dtype=np.float64)
        print(name, pol, "rounds", len(res.rows), "decisions", len(kept))
    np.savez_compressed(os.path.join(HERE, name), **out)


if __name__ == "__main__":
    main()
