"""Run the tcgen05 prefill kernel at the config-2 shape (for ncu / timing)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import _lib

lib = _lib.load()
S, C, H, D, L, n0 = int(os.environ.get("S", 4)), int(os.environ.get("C", 576)), 32, 128, 1, int(os.environ.get("N0", 4096))
cap = n0 + C + 64
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn((S, C, H, D), generator=g, device="cuda").to(torch.bfloat16)
kc = torch.randn((S, L, H, cap, D), generator=g, device="cuda").to(torch.bfloat16)
vc = torch.randn((S, L, H, cap, D), generator=g, device="cuda").to(torch.bfloat16)
out = torch.empty((S, C, H, D), dtype=torch.float32, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
reps = int(os.environ.get("REPS", 5))
W = int(os.environ.get("REC", 0))  # record the last W rows' logits + stats (engine path)
lg = torch.empty((S, max(W, 1), H, cap), dtype=torch.float32, device="cuda")
stt = torch.empty((S, max(W, 1), H, 2), dtype=torch.float32, device="cuda")
RA = (W, P(lg), cap, P(stt)) if W else (0, None, 0, None)
for i in range(2):
    _lib.check(lib.skv_prefill_attend(P(q), S, C, H, H, P(kc), P(vc), L, 0, cap, n0, P(out), *RA, st))
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for i in range(reps):
    _lib.check(lib.skv_prefill_attend(P(q), S, C, H, H, P(kc), P(vc), L, 0, cap, n0, P(out), *RA, st))
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
flops = 4 * D * (C * n0 + C * (C + 1) / 2) * S * H
print(f"prefill layer: {ms * 1e3:.1f} us, {flops / (ms * 1e-3) / 1e12:.1f} TFLOP/s useful")

if os.environ.get("PROF"):
    import numpy as np
    nqt = (C + 127) // 128
    grid = H * S * ((nqt + 1) // 2)
    buf = torch.zeros((grid * 16 + 4096,), dtype=torch.int64, device="cuda")
    _lib.check(lib.skv_prefill_profile(P(buf)))
    _lib.check(lib.skv_prefill_attend(P(q), S, C, H, H, P(kc), P(vc), L, 0, cap, n0, P(out), *RA, st))
    torch.cuda.synchronize()
    _lib.check(lib.skv_prefill_profile(None))
    ball = buf.cpu().numpy()
    b = ball[: grid * 16].reshape(grid, 16).astype(np.float64)
    if os.environ.get("SKV_PF_TL"):
        tl = ball[grid * 16:].reshape(-1, 2)
        tl = tl[tl[:, 1] > 0]
        t0 = tl[0, 1]
        names = {1: "q", 2: "k0", 10: "wait_v", 11: "v_ok", 20: "wait_p0", 21: "wait_p1", 30: "p0_ok", 31: "p1_ok",
                 40: "wait_k", 41: "k_ok", 50: "tile_done"}
        prev = t0
        for ev, t in tl[:120]:
            print(f"{names.get(int(ev), ev):10s} {t - t0:8d} (+{t - prev})")
            prev = t
    names = ["mma:k_full", "mma:pv_issue", "mma:v_full", "mma:p_full", "mma:total", "mma:s_issue",
             "wg0:s_full", "wg0:o_done", "wg0:rescales", "wg0:o_final", "wg0:total",
             "wg1:s_full", "wg1:o_done", "wg1:rescales", "wg1:o_final", "wg1:total"]
    for i, n in enumerate(names):
        if n != "-":
            print(f"{n:14s} mean {b[:, i].mean():12.0f}  max {b[:, i].max():12.0f}")
