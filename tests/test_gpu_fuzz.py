"""Seeded shape fuzz: random engine shapes through whichever decode path the
engine picks for them (static / dynamic schedules, CUDA-core or tensor-core
chunk math, the all-layer cluster launch) against the oracle over two
eviction periods -- outputs every step, window rows, kept sets and the
compacted K/V after each eviction (stands in for the sanitizers the GPU pool
does not allow: any mis-indexed row or stale partial shows up as a mismatch).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.streamkv_oracle import PolicyConfig, StreamOracle, bf16_round, kept_sets_match  # noqa: E402
from tests.gpu_helpers import rel_err, tol_for  # noqa: E402

F32 = np.float32


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _shape(seed):
    rng = np.random.default_rng(1000 + seed)
    if seed >= 12:  # many segments: the dynamic (ticket) schedule
        G = int(rng.choice([1, 2, 4]))
        Hkv = int(rng.choice([8, 16]))
        l, r = int(rng.integers(256, 1025)), int(rng.integers(256, 1025))
        return dict(S=int(rng.choice([16, 24, 32])), L=int(rng.choice([1, 2])), Hq=G * Hkv, Hkv=Hkv, D=128, l=l,
                    r=r, W=int(rng.integers(4, 13)), E=int(rng.integers(12, 25)), dtype="bf16", seed=seed)
    dtype = "bf16" if seed % 4 else "f32"
    D = 128 if (dtype == "bf16" and seed % 3) else int(rng.choice([64, 128]))
    G = int(rng.choice([1, 2, 4, 8]))
    Hkv = int(rng.choice([1, 2, 4, 8] if G < 8 else [1, 2, 4]))
    S = int(rng.choice([1, 2, 3, 5, 8, 12, 24]))
    L = int(rng.choice([1, 2, 3, 4]))
    l = int(rng.integers(16, 385))
    r = int(rng.integers(16, 385))
    W = int(rng.integers(2, min(40, l) + 1))
    E = int(rng.integers(8, 65))
    return dict(S=S, L=L, Hq=G * Hkv, Hkv=Hkv, D=D, l=l, r=r, W=W, E=E, dtype=dtype, seed=seed)


@pytest.mark.parametrize("seed", list(range(20)))
def test_random_shapes_vs_oracle(seed):
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    c = _shape(seed)
    S, L, Hq, Hkv, D, l, r, W, E = (c[k] for k in ("S", "L", "Hq", "Hkv", "D", "l", "r", "W", "E"))
    B = l + r
    dt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    rnd = bf16_round if c["dtype"] == "bf16" else (lambda a: a)
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, dt))
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W)
    rng = np.random.default_rng(7 + seed)
    for s in range(S):
        for layer in range(L):
            k = rnd(rng.standard_normal((Hkv, B, D)).astype(F32))
            v = rnd(rng.standard_normal((Hkv, B, D)).astype(F32))
            eng.inject(s, layer, k, v, np.arange(B, dtype=np.int64))
            for t in range(B):
                orc.kv[s][layer].append(k[:, t], v[:, t], t)
    orc.pos = [B] * S
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    tol = tol_for(c["dtype"])
    worst = worst_row = 0.0
    kernels = set()
    for period in range(2):
        for t in range(E):
            q = rnd(rng.standard_normal((L, S, Hq, D)).astype(F32))
            k = rnd(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            v = rnd(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            got = eng.decode_step(*(torch.from_numpy(a).to("cuda", dt) for a in (q, k, v)),
                                  record=t >= E - W).cpu().numpy()
            kernels.add(eng.last_decode_kernel)
            worst = max(worst, rel_err(got, orc.step(q, k, v)))
        n = eng.length(0, 0)
        for s in range(S):
            for layer in range(L):
                for a_, b_ in zip(eng.window_rows(s, layer), orc.win[s][layer].rows[-W:]):
                    worst_row = max(worst_row, float(np.abs(a_ - b_).max() / np.abs(b_).max()))
        eng.evict(-1, kept)
        kc = kept.cpu().numpy()
        for s in range(S):
            for layer in range(L):
                ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer], n,
                                                cfg)
                assert ok, (c, period, s, layer, nbad, gap)
                orc.apply(s, layer, kc[s, layer].astype(np.int64))
                kg, vg = eng.kv(s, layer)
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][layer].values())
    print(f"fuzz {c}: kernels {sorted(kernels)} worst out {worst:.2e} rows {worst_row:.2e}")
    assert worst <= tol and worst_row <= tol, (c, worst, worst_row)


def _policy_shape(seed):
    rng = np.random.default_rng(5000 + seed)
    policy = ("window", "sink_recent", "heavy_hitter", "inf_mllm")[seed % 4]
    G = int(rng.choice([1, 2, 4]))
    Hkv = int(rng.choice([1, 2, 4, 8]))
    l, r = int(rng.integers(16, 257)), int(rng.integers(16, 257))
    return dict(policy=policy, head_agg="max" if policy == "inf_mllm" else "mean", sink=int(rng.integers(1, 9)),
                S=int(rng.choice([1, 3, 8, 16])), L=int(rng.choice([1, 2, 3])), Hq=G * Hkv, Hkv=Hkv, D=128, l=l, r=r,
                W=int(rng.integers(2, 17)), E=int(rng.integers(8, 33)), seed=seed)


@pytest.mark.parametrize("seed", list(range(8)))
def test_random_policies_vs_oracle(seed):
    """The Session policy switch (engine.py:296-307) under random shapes: window /
    sink_recent keep sets are index arithmetic (bit-exact), heavy_hitter ranks the
    accumulated attention mass, inf_mllm with head_agg="max" -- all vs the oracle
    over two eviction periods, with the compacted K/V compared exactly."""
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    c = _policy_shape(seed)
    S, L, Hq, Hkv, D, l, r, W, E = (c[k] for k in ("S", "L", "Hq", "Hkv", "D", "l", "r", "W", "E"))
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01, sink_count=c["sink"], head_agg=c["head_agg"])
    eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, torch.bfloat16, head_agg=c["head_agg"],
                                    policy=c["policy"], sink_count=c["sink"]))
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W, policy=c["policy"])
    rng = np.random.default_rng(11 + seed)
    for s in range(S):
        for layer in range(L):
            k = bf16_round(rng.standard_normal((Hkv, B, D)).astype(F32))
            v = bf16_round(rng.standard_normal((Hkv, B, D)).astype(F32))
            eng.inject(s, layer, k, v, np.arange(B, dtype=np.int64))
            for t in range(B):
                orc.kv[s][layer].append(k[:, t], v[:, t], t)
    orc.pos = [B] * S
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    worst = 0.0
    for period in range(2):
        for t in range(E):
            q, k, v = (bf16_round(rng.standard_normal(sh).astype(F32))
                       for sh in ((L, S, Hq, D), (L, S, Hkv, D), (L, S, Hkv, D)))
            got = eng.decode_step(*(torch.from_numpy(a).to("cuda", torch.bfloat16) for a in (q, k, v)),
                                  record=t >= E - W).cpu().numpy()
            worst = max(worst, rel_err(got, orc.step(q, k, v)))
        n = eng.length(0, 0)
        kept.fill_(-1)
        eng.evict(-1, kept)
        kc = kept.cpu().numpy()
        for s in range(S):
            for layer in range(L):
                want = orc.decide(s, layer).kept
                got_k = kc[s, layer, : want.size]
                if c["policy"] in ("window", "sink_recent"):
                    np.testing.assert_array_equal(got_k, want, err_msg=str((c, period, s, layer)))
                else:
                    sc = orc.acc[s][layer][: n - l] if c["policy"] == "heavy_hitter" else orc.scores(s, layer)
                    ok, nbad, gap = kept_sets_match(sc, want, got_k, n, cfg, rel_tol=1e-4)
                    assert ok, (c, period, s, layer, nbad, gap)
                orc.apply(s, layer, got_k.astype(np.int64))
                kg, vg = eng.kv(s, layer)
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][layer].values())
    print(f"policy fuzz {c}: worst out {worst:.2e}")
    assert worst <= tol_for("bf16"), (c, worst)


@pytest.mark.parametrize("seed", list(range(6)))
def test_random_host_steps_vs_oracle(seed):
    """decode_step_host (the e2e entry point: pinned host q/k/v in, f32 outputs
    out, per-state CUDA graphs, the all-layer cluster launch where eligible)
    under random shapes over two eviction periods against the oracle."""
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    rng = np.random.default_rng(7000 + seed)
    dtype = "f32" if seed == 5 else "bf16"
    G = int(rng.choice([1, 4, 8]))
    Hkv = int(rng.choice([1, 2, 4]))
    S, L = int(rng.choice([1, 2, 8])), int(rng.choice([1, 2, 4, 6]))
    Hq, D = G * Hkv, 128
    l, r = int(rng.integers(32, 257)), int(rng.integers(32, 257))
    W, E = int(rng.integers(2, 33)), int(rng.integers(8, 40))
    B = l + r
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rnd = bf16_round if dtype == "bf16" else (lambda a: a)
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + E, dt))
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W)
    for s in range(S):
        for layer in range(L):
            k = rnd(rng.standard_normal((Hkv, B, D)).astype(F32))
            v = rnd(rng.standard_normal((Hkv, B, D)).astype(F32))
            eng.inject(s, layer, k, v, np.arange(B, dtype=np.int64))
            for t in range(B):
                orc.kv[s][layer].append(k[:, t], v[:, t], t)
    orc.pos = [B] * S
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    oh = torch.empty((L, S, Hq, D), dtype=torch.float32).pin_memory()
    worst = 0.0
    for period in range(2):
        for t in range(E):
            q = rnd(rng.standard_normal((L, S, Hq, D)).astype(F32))
            k = rnd(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            v = rnd(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            qh, kh, vh = (torch.from_numpy(a).to(dt).pin_memory() for a in (q, k, v))
            eng.decode_step_host(qh, kh, vh, oh, record=True)
            worst = max(worst, rel_err(oh.numpy(), orc.step(q, k, v)))
        n = eng.length(0, 0)
        eng.evict(-1, kept)
        kc = kept.cpu().numpy()
        for s in range(S):
            for layer in range(L):
                ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer], n, cfg)
                assert ok, (seed, period, s, layer, nbad, gap)
                orc.apply(s, layer, kc[s, layer].astype(np.int64))
                kg, vg = eng.kv(s, layer)
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][layer].values())
    print(f"host-step fuzz seed {seed}: S={S} L={L} Hq={Hq} Hkv={Hkv} l={l} r={r} W={W} E={E} {dtype}: "
          f"worst {worst:.2e}")
    assert worst <= tol_for(dtype), (seed, worst)
