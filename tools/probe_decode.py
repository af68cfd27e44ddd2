"""A few eager decode steps + one eviction at a configurable shape (for ncu
launch lists): S streams, HKV kv heads, budget B, period E (env)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

S, L, H, D, W = int(os.environ.get("S", 1)), int(os.environ.get("L", 4)), 32, 128, 32
B, E = int(os.environ.get("B", 4096)), int(os.environ.get("E", 256))
Hkv = int(os.environ.get("HKV", 8))
steps = int(os.environ.get("STEPS", 3))
l = r = B // 2
eng = StreamEngine(EngineConfig(S, L, H, Hkv, D, l, r, 0.01, W, B + E, torch.bfloat16))
g = torch.Generator(device="cuda").manual_seed(1)
for s in range(S):
    for layer in range(L):
        kf, vf = eng.kv_full(s, layer)
        kf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(torch.bfloat16)
        vf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(torch.bfloat16)
        eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
q = torch.randn((L, S, H, D), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, S, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, S, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
out = torch.empty((L, S, H, D), dtype=torch.float32, device="cuda")
for _ in range(steps):
    eng.decode_step(q, k, v, out, record=bool(int(os.environ.get("RECORD", "1"))))
torch.cuda.synchronize()
if int(os.environ.get("RECORD", "1")):
    eng.evict(-1)
torch.cuda.synchronize()
print("ok")
