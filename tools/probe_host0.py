"""Config-0 host-buffer steps in steady state (64-token periods, the last W
recorded, eviction every period): per-token wall time of skv_decode_step_host
against its parts and against the floor of one launch + one synchronisation."""
import ctypes, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_09086_b200 import EngineConfig, StreamEngine

S, L, Hq, Hkv, D, l, r, W, E = 1, 1, 8, 8, 64, 128, 128, 32, 64
B = l + r
eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, torch.float32))
g = torch.Generator(device="cuda").manual_seed(1)
kf, vf = eng.kv_full(0, 0)
kf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda")
vf[:, :B] = torch.randn((Hkv, B, D), generator=g, device="cuda")
eng.lib.skv_state_inject(eng._h, 0, 0, B, None, None, None, 0, None, None)
N = 32
qh = torch.randn((N, L, S, Hq, D)).pin_memory()
kh = torch.randn((N, L, S, Hkv, D)).pin_memory()
vh = torch.randn((N, L, S, Hkv, D)).pin_memory()
oh = torch.empty((L, S, Hq, D)).pin_memory()
qd, kd, vd = qh.cuda(), kh.cuda(), vh.cuda()
od = torch.empty((L, S, Hq, D), device="cuda")
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = lambda i: [ctypes.c_void_p(t.data_ptr()) for t in (qh[i % N], kh[i % N], vh[i % N], oh)]


def period(fn):
    for t in range(E):
        fn(t, t >= E - W)
    eng.evict(-1)
    torch.cuda.synchronize()


def timeit(fn, tag, periods=20):
    period(fn)
    t0 = time.perf_counter()
    for _ in range(periods):
        period(fn)
    dt = (time.perf_counter() - t0) / (periods * E) * 1e6
    print(f"{tag:45s} {dt:8.2f} us/token ({1e6 / dt:7.0f} tok/s)", flush=True)


timeit(lambda t, rec: eng.decode_step_host(qh[t % N], kh[t % N], vh[t % N], oh, record=rec), "decode_step_host (python)")
timeit(lambda t, rec: eng.lib.skv_decode_step_host(eng._h, *args(t), int(rec), sh), "raw ctypes skv_decode_step_host")
timeit(lambda t, rec: eng.decode_step(qd[t % N], kd[t % N], vd[t % N], od, record=rec), "device decode_step, no sync")
timeit(lambda t, rec: (eng.decode_step(qd[t % N], kd[t % N], vd[t % N], od, record=rec), torch.cuda.synchronize()),
       "device decode_step + sync")
x = torch.zeros(1, device="cuda")
timeit(lambda t, rec: (x.add_(1), torch.cuda.synchronize()), "torch add_ + sync (floor)")
timeit(lambda t, rec: (x.add_(1), x.add_(1), torch.cuda.synchronize()), "2x torch add_ + sync (floor)")
ev = torch.cuda.Event()


def spin():
    ev.record()
    while not ev.query():
        pass


timeit(lambda t, rec: (x.add_(1), spin()), "torch add_ + event spin")

eng.host_speculation(True, timeout_us=500)
timeit(lambda t, rec: eng.decode_step_host(qh[t % N], kh[t % N], vh[t % N], oh, record=rec), "speculative decode_step_host (python)")
timeit(lambda t, rec: eng.lib.skv_decode_step_host(eng._h, *args(t), int(rec), sh), "speculative raw ctypes")
print("speculation hits/misses", eng.host_speculation_stats())
