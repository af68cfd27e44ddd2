"""Timeline of the all-layer persistent decode (config-3 shape): per layer,
mean per-CTA stamps relative to the layer's first release."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine
S, L, Hq, Hkv, D, B, E, W = 1, 32, 32, 8, 128, int(os.environ.get("B", 4096)), 256, 32
eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, B // 2, B // 2, 0.01, W, B + E, torch.bfloat16))
g = torch.Generator(device="cuda").manual_seed(1)
for layer in range(L):
    kf, vf = eng.kv_full(0, layer)
    kf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(torch.bfloat16)
    vf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(torch.bfloat16)
    eng.lib.skv_state_inject(eng._h, 0, layer, B, None, None, None, 0, None, None)
q = torch.randn((8, L, S, Hq, D), device="cuda").to(torch.bfloat16)
k = torch.randn((8, L, S, Hkv, D), device="cuda").to(torch.bfloat16)
v = torch.randn((8, L, S, Hkv, D), device="cuda").to(torch.bfloat16)
tl = torch.zeros((L, 148, 16), dtype=torch.int64, device="cuda")
for t in range(4):
    eng.decode_step(q[t], k[t], v[t], record=bool(int(os.environ.get("REC", "0"))))
torch.cuda.synchronize()
eng.lib.skv_layers_timeline(eng._h, tl.data_ptr())
eng.decode_step(q[5], k[5], v[5], record=bool(int(os.environ.get("REC", "0"))))
torch.cuda.synchronize()
a = tl.cpu().numpy()
P = int((a[0, :, 0] > 0).sum())
a = a[:, :P]
names = ["released", "q+K in", "math done", "staged", "appended", "combined", "published", "all pub", "merge0", "merged"]
order = [0, 1, 2, 5, 8, 9, 3, 6, 7, 4]
prev = None
for l in range(L):
    r0 = a[l, :, 0].min()
    row = []
    for nm, i in zip(names, order):
        col = a[l, :, i]
        col = col[col > 0]
        if col.size == 0:
            row.append(f"{nm} -")
            continue
        row.append(f"{nm} {(np.median(col) - r0) / 1e3:5.2f}/{(col.max() - r0) / 1e3:5.2f}")
    gap = f" | layer period {(r0 - prev) / 1e3:5.2f}" if prev is not None else ""
    prev = r0
    if l < 6 or l > L - 3:
        print(f"L{l:02d} " + "  ".join(row) + gap)
# per-CTA phase durations (intra-CTA stamps are SM-cycle based), median / max over CTAs, layers 1..L-1
ph = a[1:, :, :]
print("phase (median/max us over CTAs and layers 1..):")
for k in range(1, len(order)):
    d = (ph[:, :, order[k]].astype(np.int64) - ph[:, :, order[k - 1]].astype(np.int64)) / 1e3
    ok = (ph[:, :, order[k]] > 0) & (ph[:, :, order[k - 1]] > 0)
    d = d[ok]
    if d.size:
        print(f"  {names[k - 1]:>9} -> {names[k]:<9} {np.median(d):5.2f} / {d.max():5.2f}")
# the last CTA to release each layer: its phases
print("last releaser per layer (CTA: phase durations us):")
for l in range(1, min(L, 8)):
    c = int(np.argmax(a[l, :, order[-1]]))
    r0 = a[l, :, 0].min()
    segs = [f"{(a[l, c, order[k]] - a[l, c, order[k - 1]]) / 1e3:4.2f}" for k in range(1, len(order))]
    print(f"  L{l:02d} cta {c:3d} start +{(a[l, c, 0] - r0) / 1e3:4.2f}: " + " ".join(segs) +
          f" | merged at {(a[l, c, order[-1]] - r0) / 1e3:4.2f}")
