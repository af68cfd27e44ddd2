"""Decode-launch timing variants (cfg1 shape): eager vs graph, record on/off."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

S, L, H, D, B, E, W = 8, 32, 32, 128, 2048, 128, 32
l = r = B // 2
dev = torch.device("cuda")
eng = StreamEngine(EngineConfig(S, L, H, H, D, l, r, 0.01, W, B + E, torch.bfloat16))
g = torch.Generator(device=dev).manual_seed(1)
for s in range(S):
    for layer in range(L):
        kf, vf = eng.kv_full(s, layer)
        kf[:, :B] = torch.randn((H, B, D), generator=g, device=dev).to(torch.bfloat16)
        vf[:, :B] = torch.randn((H, B, D), generator=g, device=dev).to(torch.bfloat16)
        eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
q = torch.randn((E, L, S, H, D), generator=g, device=dev).to(torch.bfloat16)
k = torch.randn((E, L, S, H, D), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((E, L, S, H, D), generator=g, device=dev).to(torch.bfloat16)
out = torch.empty((L, S, H, D), dtype=torch.float32, device=dev)
st = torch.cuda.Stream()
eng.run_period(q, k, v, out, E, evict=True)
torch.cuda.synchronize()
nbytes = S * 2 * (B + 8) * H * D * 2

def eager(steps, record):
    with torch.cuda.stream(st):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for t in range(steps):
            eng.decode_step(q[t], k[t], v[t], out, record=record)
        b.record(st)
    st.synchronize()
    ms = a.elapsed_time(b)
    eng.evict(-1); torch.cuda.synchronize()
    return ms * 1e3 / (steps * L)

def graph(steps, record):
    with torch.cuda.stream(st):
        eng.capture_begin()
        for t in range(steps):
            eng.decode_step(q[t], k[t], v[t], out, record=record)
        eng.capture_end()
        eng.replay()
        eng.evict(-1)
    st.synchronize()
    with torch.cuda.stream(st):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.replay()
        b.record(st)
        eng.evict(-1)
    st.synchronize()
    return a.elapsed_time(b) * 1e3 / (steps * L)

for name, fn in (("eager", eager), ("graph", graph)):
    for rec in (False, True):
        us = fn(16, rec)
        print(f"{name:5s} record={rec!s:5s}: {us:7.2f} us/launch  {nbytes / (us * 1e-6) / 1e9:6.0f} GB/s", flush=True)
