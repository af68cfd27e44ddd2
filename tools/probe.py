"""Component timing for the config-1 workload (decode-only graph, eviction,
per-launch decode events inside a graph).  Usage: python tools/probe.py [--ncu]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true", help="short run for a profiler")
ap.add_argument("--streams", type=int, default=8)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--hkv", type=int, default=32)
ap.add_argument("--budget", type=int, default=2048)
ap.add_argument("--period", type=int, default=128)
args = ap.parse_args()

S, L, H, Hkv, D = args.streams, args.layers, 32, args.hkv, 128
B, E, W = args.budget, args.period, 32
l = r = B // 2
dev = torch.device("cuda")
eng = StreamEngine(EngineConfig(S, L, H, Hkv, D, l, r, 0.01, W, B + E, torch.bfloat16))
g = torch.Generator(device=dev).manual_seed(1)
for s in range(S):
    for layer in range(L):
        kf, vf = eng.kv_full(s, layer)
        kf[:, :B] = torch.randn((Hkv, B, D), generator=g, device=dev).to(torch.bfloat16)
        vf[:, :B] = torch.randn((Hkv, B, D), generator=g, device=dev).to(torch.bfloat16)
        eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
q = torch.randn((E, L, S, H, D), generator=g, device=dev).to(torch.bfloat16)
k = torch.randn((E, L, S, Hkv, D), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((E, L, S, Hkv, D), generator=g, device=dev).to(torch.bfloat16)
out = torch.empty((L, S, H, D), dtype=torch.float32, device=dev)
if args.ncu:
    for t in range(3):
        eng.decode_step(q[t], k[t], v[t], out, record=True)
    eng.evict(-1)
    torch.cuda.synchronize()
    print("ncu probe done")
    sys.exit(0)

st = torch.cuda.Stream()


def timed(fn, reps=3):
    with torch.cuda.stream(st):
        fn()
        st.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
    st.synchronize()
    return a.elapsed_time(b) / reps


# warm: one period to reach steady ring state
eng.run_period(q, k, v, out, E, evict=True)
torch.cuda.synchronize()

# (a) decode-only graph of E steps (record last W) -- state restored by an eager evict afterwards
with torch.cuda.stream(st):
    eng.capture_begin()
    eng.run_period(q, k, v, out, E, evict=False)
    eng.capture_end()
with torch.cuda.stream(st):
    t_a = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.replay()
        b.record(st)
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        st.synchronize()
        print("replayed", flush=True)
        c0.record(st)
        eng.evict(-1)
        c1.record(st)
        st.synchronize()
        print("evicted", flush=True)
        t_a.append((a.elapsed_time(b), c0.elapsed_time(c1)))
print("decode-only period graph ms, eager evict ms:", t_a)
dec_ms = np.median([x[0] for x in t_a])
print(f"per token-step decode: {dec_ms / E * 1e3:.1f} us; per layer launch: {dec_ms / E / L * 1e3:.2f} us")
n_avg = B + (E + 1) / 2
bytes_layer = S * 2 * n_avg * Hkv * D * 2
print(f"decode HBM rate incl. launch gaps: {bytes_layer * L * E / (dec_ms * 1e-3) / 1e9:.0f} GB/s")

# (b) eager skv_decode_step (32 launches enqueued from C) bracketed by events
eng.evict(-1)
torch.cuda.synchronize()
res = []
with torch.cuda.stream(st):
    for t in range(8):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        eng.decode_step(q[t], k[t], v[t], out, record=False)
        e1.record(st)
        res.append((e0, e1))
st.synchronize()
d = [a.elapsed_time(b) * 1e3 / L for a, b in res]
print(f"decode launch avg (eager C loop): {np.mean(d):.2f} us  ({bytes_layer / (np.mean(d) * 1e-6) / 1e9:.0f} GB/s)")
eng.evict(-1)
torch.cuda.synchronize()
