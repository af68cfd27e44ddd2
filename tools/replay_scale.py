"""Throughput of the batched device trace replay on a large synthetic trace.

The trace is generated here (seeded NumPy, planted persistent columns + recency
mass, rows normalised) -- the reference's generator is not on the GPU box.
  python tools/replay_scale.py            # device replay (GPU box)
  python tools/replay_scale.py --reference  # the reference replay_trace on the CPU (dev container)
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--rounds", type=int, default=32)
ap.add_argument("--prompt", type=int, default=64)
ap.add_argument("--decode", type=int, default=64)
ap.add_argument("--policy", default="inf-mllm")
ap.add_argument("--reference", action="store_true")
args = ap.parse_args()

rng = np.random.default_rng(2026)
F32 = np.float32
planted = set(int(x) for x in rng.choice(256, size=8, replace=False))
events = []
n = 0
for rnd in range(args.rounds):
    events.append(("round", rnd, args.prompt))
    for step in range(args.prompt + args.decode):
        n += 1
        base = rng.random(n) + 0.05
        base[-16:] += 3.0
        for c in planted:
            if c < n:
                base[c] += 6.0
        for layer in range(args.layers):
            row = (base * (1.0 + 0.2 * rng.random(n))).astype(np.float64)
            events.append(("row", layer, (row / row.sum()).astype(F32)))
rows = sum(1 for e in events if e[0] == "row")
print(f"trace: {args.layers} layers, {args.rounds} rounds, {rows} rows, stream length {n}, "
      f"{sum(e[2].size for e in events if e[0] == 'row') * 4 / 1e6:.0f} MB of probabilities")
if args.reference:
    sys.path.insert(0, "/root/reference/pkg/src")
    from streamkv.policies import PolicyConfig
    from streamkv.replay import replay_trace
    from streamkv.traceio import AttnRow, RoundStart, TraceHeader
else:
    import torch
    from paper_2409_09086_b200 import PolicyConfig
    from paper_2409_09086_b200.replay import replay_trace
    from paper_2409_09086_b200.traceio import AttnRow, RoundStart, TraceHeader
ev = [RoundStart(e[1], e[2]) if e[0] == "round" else AttnRow(e[1], e[2]) for e in events]
cfg = PolicyConfig(recent_len=256, relevant_budget=256, bias=0.01)
hdr = TraceHeader(layers=args.layers, heads=8)
if not args.reference:
    replay_trace(hdr, ev[: len(ev) // 8], args.policy, cfg)  # warm-up (module load, allocator)
    torch.cuda.synchronize()
t0 = time.perf_counter()
res = replay_trace(hdr, ev, args.policy, cfg)
if not args.reference:
    torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{'reference (CPU)' if args.reference else 'device'} replay_trace {args.policy}: {dt:.3f} s, "
      f"{rows / dt:.0f} rows/s, {len(res.rows)} metric rows, last retained mass {res.rows[-1].retained_mass:.6f}, "
      f"overlap {res.rows[-1].topk_overlap}")
