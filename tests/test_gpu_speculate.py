"""Speculative host steps (skv_host_speculate): each decode_step_host call
launches the next token's kernels behind a device-side doorbell gate.  These
tests drive the cases where the speculation is wrong -- a different `record`
flag, other entry points in between, a late call past the gate's timeout, a
device-wide synchronisation while a step is pending, the capacity limit --
and check every token's outputs and every period's kept sets against the
oracle, as if no speculation had happened."""
import os
import sys
import time

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.streamkv_oracle import PolicyConfig, StreamOracle, kept_sets_match  # noqa: E402
from tests.gpu_helpers import rel_err  # noqa: E402

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(S=1, L=1, Hq=8, Hkv=8, D=64, l=32, r=32, W=8, E=16, timeout_us=2000, seed=5):
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    B = l + r
    eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, torch.float32))
    orc = StreamOracle(S, L, Hq, Hkv, D, PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01), window=W)
    rng = np.random.default_rng(seed)
    for s in range(S):
        for layer in range(L):
            k = rng.standard_normal((Hkv, B, D)).astype(F32)
            v = rng.standard_normal((Hkv, B, D)).astype(F32)
            eng.inject(s, layer, k, v, np.arange(B, dtype=np.int64))
            for t in range(B):
                orc.kv[s][layer].append(k[:, t], v[:, t], t)
    orc.pos = [B] * S
    eng.host_speculation(True, timeout_us=timeout_us)
    return eng, orc, rng, (S, L, Hq, Hkv, D, l, r, W, E, B)


def _token(eng, orc, rng, dims, record, oh):
    S, L, Hq, Hkv, D = dims[:5]
    q = rng.standard_normal((L, S, Hq, D)).astype(F32)
    k = rng.standard_normal((L, S, Hkv, D)).astype(F32)
    v = rng.standard_normal((L, S, Hkv, D)).astype(F32)
    hq, hk, hv = (torch.from_numpy(a).pin_memory() for a in (q, k, v))
    oh.fill_(float("nan"))
    eng.decode_step_host(hq, hk, hv, oh, record=record)
    return rel_err(oh.numpy(), orc.step(q, k, v))


def _evict_check(eng, orc, dims, n=None):
    S, L, l, r, E, B = dims[0], dims[1], dims[5], dims[6], dims[8], dims[9]
    n = n or B + E
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    eng.evict(-1, kept)
    kc = kept.cpu().numpy()
    for s in range(S):
        for layer in range(L):
            ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer], n, cfg)
            assert ok, (s, layer, nbad, gap)
            orc.apply(s, layer, kc[s, layer].astype(np.int64))


@pytest.mark.parametrize("layers", [1, 2])
def test_speculation_survives_flag_flips_and_interleaved_calls(layers):
    """Record flips every few tokens, a length query / window read / device
    decode_step in the middle of periods: each cancels the pending step."""
    eng, orc, rng, dims = _setup(S=2, L=layers, Hq=8, Hkv=2)
    S, L, Hq, Hkv, D, l, r, W, E, B = dims
    oh = torch.empty((L, S, Hq, D), dtype=torch.float32).pin_memory()
    worst = 0.0
    for period in range(3):
        for t in range(E):
            rec = (t // 3) % 2 == 0 or t >= E - W
            worst = max(worst, _token(eng, orc, rng, dims, rec, oh))
            if t == 5:
                assert eng.length(0, 0) == B + t + 1
            if t == 9:
                q = rng.standard_normal((L, S, Hq, D)).astype(F32)
                k = rng.standard_normal((L, S, Hkv, D)).astype(F32)
                v = rng.standard_normal((L, S, Hkv, D)).astype(F32)
                od = eng.decode_step(*(torch.from_numpy(a).cuda() for a in (q, k, v)), record=True)
                worst = max(worst, rel_err(od.cpu().numpy(), orc.step(q, k, v)))
        _evict_check(eng, orc, dims)
    hits, misses = eng.host_speculation_stats()
    assert worst <= 1e-5, worst
    assert hits > E and misses > 0, (hits, misses)


def test_speculation_expired_gate_falls_back():
    """Calls that come after the gate's timeout: the pending step expires on
    the device (nothing of it runs) and the call takes the regular path."""
    eng, orc, rng, dims = _setup(timeout_us=100)
    S, L, Hq, Hkv, D, l, r, W, E, B = dims
    oh = torch.empty((L, S, Hq, D), dtype=torch.float32).pin_memory()
    worst = 0.0
    for period in range(2):
        for t in range(E):
            if t % 4 == 1:
                time.sleep(0.003)
            worst = max(worst, _token(eng, orc, rng, dims, t >= E - W, oh))
        _evict_check(eng, orc, dims)
    hits, misses = eng.host_speculation_stats()
    assert worst <= 1e-5, worst
    assert misses >= 4 and hits > 0, (hits, misses)


def test_device_synchronize_while_pending_is_bounded():
    """torch.cuda.synchronize() with a step pending returns once its gate
    expires; the next call then runs regularly."""
    eng, orc, rng, dims = _setup(timeout_us=1000)
    S, L, Hq, Hkv, D, l, r, W, E, B = dims
    oh = torch.empty((L, S, Hq, D), dtype=torch.float32).pin_memory()
    worst = _token(eng, orc, rng, dims, False, oh)
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 1.0
    for t in range(1, E):
        worst = max(worst, _token(eng, orc, rng, dims, t >= E - W, oh))
    _evict_check(eng, orc, dims)
    assert worst <= 1e-5, worst


def test_speculation_stops_at_capacity():
    """The last token that fits is served; the one after raises the same
    capacity error as without speculation, and an eviction recovers."""
    eng, orc, rng, dims = _setup()
    S, L, Hq, Hkv, D, l, r, W, E, B = dims
    oh = torch.empty((L, S, Hq, D), dtype=torch.float32).pin_memory()
    worst = 0.0
    fill = eng.cap - B  # (the engine rounds the capacity up to whole 32-token tiles)
    for t in range(fill):
        worst = max(worst, _token(eng, orc, rng, dims, t >= fill - W, oh))
    q = torch.zeros((L, S, Hq, D)).pin_memory()
    kv = torch.zeros((L, S, Hkv, D)).pin_memory()
    with pytest.raises(Exception, match="capacity"):
        eng.decode_step_host(q, kv, kv, oh, record=False)
    assert eng.length(0, 0) == eng.cap
    _evict_check(eng, orc, dims, n=eng.cap)
    for t in range(E):
        worst = max(worst, _token(eng, orc, rng, dims, t >= E - W, oh))
    _evict_check(eng, orc, dims)
    assert worst <= 1e-5, worst
