"""Config-2 text chunks (32 tokens) through StreamEngine.prefill_chunk on 2
layers after an image chunk + eviction, for an ncu launch list."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

S, L, H, D, B, CI, CT = 4, 2, 32, 128, 4096, 576, int(os.environ.get("CT", 32))
eng = StreamEngine(EngineConfig(S, L, H, H, D, 2048, 2048, 0.01, 32, B + CI + 64, torch.bfloat16))
g = torch.Generator(device="cuda").manual_seed(1)
for s in range(S):
    for layer in range(L):
        kf, vf = eng.kv_full(s, layer)
        kf[:, :B] = torch.randn((H, B, D), generator=g, device="cuda").to(torch.bfloat16)
        vf[:, :B] = torch.randn((H, B, D), generator=g, device="cuda").to(torch.bfloat16)
        eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
mk = lambda C: [torch.randn((S, C, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3)]
qi, ki, vi = mk(CI)
qt, kt, vt = mk(CT)
oi = torch.empty((S, CI, H, D), dtype=torch.float32, device="cuda")
ot = torch.empty((S, CT, H, D), dtype=torch.float32, device="cuda")
for layer in range(L):
    eng.prefill_chunk(layer, qi, ki, vi, oi, modality=1)
eng.evict(-1)
for layer in range(L):
    eng.prefill_chunk(layer, qt, kt, vt, ot, modality=0)
eng.evict(-1)
torch.cuda.synchronize()
print("ok")
