"""Config-3 host-buffer steps in steady state (the bench's record pattern:
the last W of each 256-token period, eviction every period): per-token wall
time of skv_decode_step_host against its parts."""
import ctypes, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

S, L, Hq, Hkv, D, l, r, W, E = 1, 32, 32, 8, 128, 2048, 2048, 32, 256
B = l + r
eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, torch.bfloat16))
g = torch.Generator(device="cuda").manual_seed(1)
for layer in range(L):
    kf, vf = eng.kv_full(0, layer)
    kf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(torch.bfloat16)
    vf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda").to(torch.bfloat16)
    eng.lib.skv_state_inject(eng._h, 0, layer, B, None, None, None, 0, None, None)
N = 32
qh = torch.randn((N, L, S, Hq, D)).to(torch.bfloat16).pin_memory()
kh = torch.randn((N, L, S, Hkv, D)).to(torch.bfloat16).pin_memory()
vh = torch.randn((N, L, S, Hkv, D)).to(torch.bfloat16).pin_memory()
oh = torch.empty((L, S, Hq, D)).pin_memory()
qd, kd, vd = qh.cuda(), kh.cuda(), vh.cuda()
od = torch.empty((L, S, Hq, D), device="cuda")
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = lambda i: [ctypes.c_void_p(t.data_ptr()) for t in (qh[i % N], kh[i % N], vh[i % N], oh)]


def period(fn, tag):
    for t in range(E):
        fn(t, t >= E - W)
    eng.evict(-1)
    torch.cuda.synchronize()


def timeit(fn, tag, periods=3):
    period(fn, tag)  # warm: graphs of every state of the period
    t0 = time.perf_counter()
    for _ in range(periods):
        period(fn, tag)
    dt = (time.perf_counter() - t0) / (periods * E) * 1e6
    print(f"{tag:45s} {dt:8.1f} us/token ({1e6 / dt:7.0f} tok/s)")


timeit(lambda t, rec: eng.decode_step_host(qh[t % N], kh[t % N], vh[t % N], oh, record=rec), "decode_step_host (python)")
timeit(lambda t, rec: eng.lib.skv_decode_step_host(eng._h, *args(t), int(rec), sh), "raw ctypes skv_decode_step_host")
timeit(lambda t, rec: eng.decode_step(qd[t % N], kd[t % N], vd[t % N], od, record=rec), "device decode_step, no sync")
timeit(lambda t, rec: (eng.decode_step(qd[t % N], kd[t % N], vd[t % N], od, record=rec), torch.cuda.synchronize()),
       "device decode_step + sync")

# order check and the wrapper's own cost
timeit(lambda t, rec: eng.lib.skv_decode_step_host(eng._h, *args(t), int(rec), sh), "raw ctypes (again)")
timeit(lambda t, rec: eng.decode_step_host(qh[t % N], kh[t % N], vh[t % N], oh, record=rec), "decode_step_host (again)")
from paper_2409_09086_b200.engine import _stream_handle
for tag, fn in (("_stream_handle()", lambda: _stream_handle()), ("qh[i] view x3", lambda: (qh[3], kh[3], vh[3])),
                ("shape/dtype/is_cuda checks", lambda: [(t.shape != (L, S, Hq, D), t.dtype != torch.bfloat16, t.is_cuda)
                                                        for t in (qh[0], kh[0], vh[0])])):
    t0 = time.perf_counter()
    for _ in range(10000):
        fn()
    print(f"{tag:45s} {(time.perf_counter() - t0) / 10000 * 1e6:8.2f} us")
