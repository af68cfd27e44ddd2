import os, sys, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2409_09086_b200 import EngineConfig, StreamEngine
c = dict(bench.WORKLOADS["cfg2"])
L, H, D, S = c["layers"], c["heads_q"], c["head_dim"], c["streams"]
l, r, W, CI, CT = c["recent"], c["relevant"], c["window"], c["image"], c["text"]
B = l + r
dev = torch.device("cuda")
eng = StreamEngine(EngineConfig(S, L, H, H, D, l, r, c["bias"], W, B + CI + 64, torch.bfloat16))
g = torch.Generator(device=dev).manual_seed(99)
for s in range(S):
    for layer in range(L):
        kf, vf = eng.kv_full(s, layer)
        kf[:, :B] = torch.randn((H, B, D), generator=g, device=dev).to(torch.bfloat16)
        vf[:, :B] = torch.randn((H, B, D), generator=g, device=dev).to(torch.bfloat16)
        eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
mk = lambda C: [torch.randn((L, S, C, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(3)]
qi, ki, vi = mk(CI); qt, kt, vt = mk(CT)
oi = torch.empty((S, CI, H, D), dtype=torch.float32, device=dev); ot = torch.empty((S, CT, H, D), dtype=torch.float32, device=dev)
def frame():
    for layer in range(L): eng.prefill_chunk(layer, qi[layer], ki[layer], vi[layer], oi, modality=1)
    eng.evict(-1)
    for layer in range(L): eng.prefill_chunk(layer, qt[layer], kt[layer], vt[layer], ot, modality=0)
    eng.evict(-1)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3): frame()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10): frame()
    b.record(st)
st.synchronize(); print("eager frame ms", a.elapsed_time(b) / 10)
with torch.cuda.stream(st):
    eng.capture_begin(); frame(); eng.capture_end()
    for _ in range(3): eng.replay()
    a.record(st)
    for _ in range(10): eng.replay()
    b.record(st)
st.synchronize(); print("graph frame ms", a.elapsed_time(b) / 10)
