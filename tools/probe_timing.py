"""Per-launch device timestamps (first CTA start / last CTA end) for the
config-1 decode kernel inside a replayed period graph."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

S, L, H, D, W = int(os.environ.get("S", 8)), 32, 32, 128, 32
B, E = int(os.environ.get("B", 2048)), int(os.environ.get("E", 128))
Hkv = int(os.environ.get("HKV", 32))
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
st = torch.cuda.Stream()
eng.run_period(q, k, v, out, E, evict=True)
torch.cuda.synchronize()
eng.timing(True)
with torch.cuda.stream(st):
    eng.capture_begin()
    eng.run_period(q, k, v, out, E, evict=True)
    eng.capture_end()
    eng.replay()
st.synchronize()
eng.lib.skv_timing(eng._h, 2)  # clear values, keep the slots baked into the graph
with torch.cuda.stream(st):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st); eng.replay(); b.record(st)
st.synchronize()
period_ms = a.elapsed_time(b)
ts = eng.timing_read()  # slots assigned at capture time: E*L decode launches
n = E * L
ts = ts[:n].astype(np.int64)
dur = (ts[:, 1] - ts[:, 0]) / 1e3
gaps = (ts[1:, 0] - ts[:-1, 1]) / 1e3
nbytes = S * 2 * (B + E / 2) * Hkv * D * 2
print(f"period {period_ms:.2f} ms; decode span {(ts[-1,1]-ts[0,0])/1e6:.2f} ms; eviction+rest {period_ms - (ts[-1,1]-ts[0,0])/1e6:.2f} ms")
print(f"kernel duration us: mean {dur.mean():.2f} p10 {np.percentile(dur,10):.2f} p90 {np.percentile(dur,90):.2f}")
print(f"gap (next start - prev end) us: mean {gaps.mean():.2f} min {gaps.min():.2f} max {gaps.max():.2f}")
print(f"kernel-only HBM rate {nbytes/(dur.mean()*1e-6)/1e9:.0f} GB/s; incl gaps {nbytes/((dur.mean()+gaps.mean())*1e-6)/1e9:.0f} GB/s")
rec = dur.reshape(E, L)
print(f"record steps (last {W}): {rec[-W:].mean():.2f} us; non-record: {rec[:-W].mean():.2f} us")

# per-CTA timeline of a few consecutive launches (eager C loop of one step)
eng.lib.skv_timing(eng._h, 3)
eng.evict(-1); torch.cuda.synchronize()
with torch.cuda.stream(st):
    rec = bool(int(os.environ.get("REC", "0")))
    eng.decode_step(q[0], k[0], v[0], out, record=rec)
    eng.decode_step(q[1], k[1], v[1], out, record=rec)
st.synchronize()
import ctypes
P = None
t0 = None
for slot in range(40, 44):
    buf = np.zeros((4096, 8), dtype=np.uint64)
    P = eng.lib.skv_timing_cta(eng._h, slot, buf.ctypes.data_as(ctypes.c_void_p))
    mrow = buf[P].astype(np.int64)
    b = buf[:P].astype(np.int64)
    b = b[b[:, 0] > 0]
    if t0 is None:
        t0 = b[:, 0].min()
    rel = b[:, 1].min()
    if slot > 40:
        print(f"   release - previous release: {(rel - prev_rel) / 1e3:.1f} us; - previous last merge end {(rel - prev_mend) / 1e3:.1f} us")
    prev_rel, prev_mend = rel, mrow[2]
    st_, end, cend, pend = (b[:, 0] - rel) / 1e3, (b[:, 2] - rel) / 1e3, (b[:, 3] - rel) / 1e3, (b[:, 6] - rel) / 1e3
    chunks, ewait, taken = b[:, 4], b[:, 5] / 1e3, b[:, 7]
    if os.environ.get("DBGT"):
        qdone, t0done = (b[:, 5] - rel) / 1e3, (b[:, 4] - rel) / 1e3
        qq = lambda x: " ".join(f"{np.percentile(x, p):.1f}" for p in (0, 10, 50, 90, 100))
        print(f"   q loaded: {qq(qdone)}   tile0 done: {qq(t0done)}")
    q = lambda x: " ".join(f"{np.percentile(x, p):.1f}" for p in (0, 10, 50, 90, 100))
    print(f"launch {slot}: CTAs {len(b)} start(rel) [{st_.min():.1f},{st_.max():.1f}]")
    print(f"   producer end p0/10/50/90/100: {q(pend)}  tickets {q(taken)}")
    print(f"   consumer end: {q(cend)}  chunks {q(chunks)}  epi-wait us {q(ewait)}")
    print(f"   epilogue end: {q(end)}   merge seg0 start {(mrow[1] - rel) / 1e3:.1f}  last merge end {(mrow[2] - rel) / 1e3:.1f}")
    slow = np.argsort(end)[-3:]
    for j in slow:
        print(f"   slow CTA: start {st_[j]:.1f} prod_end {pend[j]:.1f} cons_end {cend[j]:.1f} epi_end {end[j]:.1f} chunks {chunks[j]} taken {taken[j]} epi_wait {ewait[j]:.1f}")
