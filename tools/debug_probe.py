import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine
S, L, H, Hkv, D, B, E, W = 2, 4, 32, 32, 128, 256, 32, 8
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
def chk(msg):
    torch.cuda.synchronize(); print("ok:", msg, "n=", eng.length(0, 0), flush=True)
eng.run_period(q, k, v, out, E, evict=False); chk("eager period decode")
eng.evict(-1); chk("eager evict")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    eng.capture_begin(); eng.run_period(q, k, v, out, E, evict=False); eng.capture_end()
chk("captured")
with torch.cuda.stream(st):
    eng.replay()
chk("replay 1")
with torch.cuda.stream(st):
    eng.evict(-1)
chk("evict after replay")
with torch.cuda.stream(st):
    eng.replay()
chk("replay 2")
with torch.cuda.stream(st):
    eng.evict(-1)
chk("evict 2")
