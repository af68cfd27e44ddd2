"""Small runs of every kernel path for compute-sanitizer (memcheck / synccheck):
dynamic-schedule decode + merge + fold, the tensor-core GQA decode, eviction
(select + compaction), the tcgen05 prefill (two-tile, lone split tile, a
32-token chunk) with the window fold, and RoPE."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

g = torch.Generator(device="cuda").manual_seed(3)
bf = torch.bfloat16


def rnd(*shape):
    return torch.randn(shape, generator=g, device="cuda").to(bf)


def fill(eng, S, L, Hkv, D, n):
    for s in range(S):
        for layer in range(L):
            kf, vf = eng.kv_full(s, layer)
            kf[:, :n] = rnd(Hkv, n, D)
            vf[:, :n] = rnd(Hkv, n, D)
            eng.lib.skv_state_inject(eng._h, s, layer, n, None, None, None, 0, None, None)


# 1. dynamic-schedule decode (8 streams x 8 heads, MHA) + eviction
S, L, H, D, l, r, W, E = 8, 2, 8, 128, 256, 256, 8, 16
eng = StreamEngine(EngineConfig(S, L, H, H, D, l, r, 0.01, W, l + r + E, bf))
fill(eng, S, L, H, D, l + r)
for t in range(E):
    eng.decode_step(rnd(L, S, H, D), rnd(L, S, H, D), rnd(L, S, H, D), record=t >= E - W)
eng.evict(-1)
torch.cuda.synchronize()
print("decode (dynamic) + evict ok")

# 2. tensor-core GQA decode (batch 1, 32 q / 8 kv heads)
S, L, Hq, Hkv = 1, 2, 32, 8
eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, 512, 512, 0.01, W, 1024 + E, bf))
fill(eng, S, L, Hkv, D, 1024)
for t in range(E):
    eng.decode_step(rnd(L, S, Hq, D), rnd(L, S, Hkv, D), rnd(L, S, Hkv, D), record=t >= E - W)
eng.evict(-1)
torch.cuda.synchronize()
print("decode (tensor-core GQA) + evict ok")

# 3. prefill chunks: 200 tokens (two-tile CTA), 32 tokens (lone split tile), with folds
S, L, H = 2, 1, 4
eng = StreamEngine(EngineConfig(S, L, H, H, D, 256, 256, 0.01, 32, 512 + 256, bf))
fill(eng, S, L, H, D, 512)
for C in (200, 32):
    eng.prefill_chunk(0, rnd(S, C, H, D), rnd(S, C, H, D), rnd(S, C, H, D), modality=1)
    eng.evict(-1)
torch.cuda.synchronize()
print("prefill chunks + folds ok")

# 4. RoPE engine (cache-relative), a few decode steps and an eviction
eng = StreamEngine(EngineConfig(1, 1, 4, 4, 64, 32, 32, 0.01, 4, 64 + 8, bf, rope="cache_relative"))
fill(eng, 1, 1, 4, 64, 64)
for t in range(8):
    eng.decode_step(rnd(1, 1, 4, 64), rnd(1, 1, 4, 64), rnd(1, 1, 4, 64), record=t >= 4)
eng.evict(-1)
torch.cuda.synchronize()
print("rope ok")
