"""Where the host-buffer decode step spends its time (cfg0 / cfg3 shapes):
per-token wall time of (a) skv_decode_step_host, (b) device-buffer decode
steps launched back to back, (c) the same with a sync per token, (d) the
H2D+D2H copies alone with a sync per token."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

shape = os.environ.get("SHAPE", "cfg0")
if shape == "cfg0":
    S, L, Hq, Hkv, D, l, r, W, E, dt = 1, 1, 8, 8, 64, 128, 128, 32, 64, torch.float32
else:
    S, L, Hq, Hkv, D, l, r, W, E, dt = 1, 32, 32, 8, 128, 2048, 2048, 32, 256, torch.bfloat16
B = l + r
eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, dt))
g = torch.Generator(device="cuda").manual_seed(1)
for s in range(S):
    for layer in range(L):
        kf, vf = eng.kv_full(s, layer)
        kf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(dt)
        vf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(dt)
        eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
N = 48
q = torch.randn((N, L, S, Hq, D), device="cuda").to(dt)
k = torch.randn((N, L, S, Hkv, D), device="cuda").to(dt)
v = torch.randn((N, L, S, Hkv, D), device="cuda").to(dt)
out = torch.empty((L, S, Hq, D), device="cuda")
qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
oh = torch.empty(out.shape).pin_memory()

def run(name, fn, reps=N):
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(reps):
        fn(i)
    torch.cuda.synchronize()
    dt_us = (time.perf_counter() - t) / reps * 1e6
    print(f"{shape} {name:40s} {dt_us:9.1f} us/token  ({1e6 / dt_us:9.0f} tok/s)")

def evict_if_full():
    if eng.length(0, 0) + 1 > B + E:
        eng.evict(-1)
        torch.cuda.synchronize()

run("decode_step_host (pinned)", lambda i: (evict_if_full(), eng.decode_step_host(qh[i], kh[i], vh[i], oh, record=True)))
run("decode_step device, no sync", lambda i: (evict_if_full(), eng.decode_step(q[i], k[i], v[i], out, record=True)))
run("decode_step device + sync", lambda i: (evict_if_full(), eng.decode_step(q[i], k[i], v[i], out, record=True),
                                              torch.cuda.synchronize()))
def copies(i):
    q[0].copy_(qh[i], non_blocking=True); k[0].copy_(kh[i], non_blocking=True); v[0].copy_(vh[i], non_blocking=True)
    oh.copy_(out, non_blocking=True); torch.cuda.synchronize()
run("copies only + sync", copies)

# ---- where a host step's wall time goes (cfg0 shape)
import ctypes
if shape == "cfg0":
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    def slices(i):
        return qh[i % N], kh[i % N], vh[i % N]
    run("python: three tensor slices", lambda i: slices(i))
    run("ctypes skv_sync (stream sync)", lambda i: eng.lib.skv_sync(eng._h, sh))
    args = [ctypes.c_void_p(t.data_ptr()) for t in (qh[0], kh[0], vh[0], oh)]
    def raw(i):
        evict_if_full()
        eng.lib.skv_decode_step_host(eng._h, *args, 1, sh)
    run("raw ctypes skv_decode_step_host", raw)
