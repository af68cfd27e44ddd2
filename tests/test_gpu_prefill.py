"""GPU parity of the tcgen05 chunked-prefill kernel (K4) against a float32
PyTorch reference of the reference's per-token prompt loop: query i of the
chunk attends to the cached prefix and chunk tokens 0..i (engine.py:350-353)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ref(q, kc, vc, n0, C, W):
    """q [S][C][Hq][D] f32, kc/vc [S][Hkv][n0+C][D] f32 -> out, probs of last W rows."""
    S, _, Hq, D = q.shape
    Hkv = kc.shape[1]
    G = Hq // Hkv
    scale = np.float32(1.0 / np.sqrt(D))
    out = torch.zeros((S, C, Hq, D), dtype=torch.float32, device="cuda")
    logits_last = []
    for s in range(S):
        k = kc[s].repeat_interleave(G, dim=0)  # [Hq][N][D]
        v = vc[s].repeat_interleave(G, dim=0)
        lg = torch.einsum("chd,hnd->chn", q[s], k) * scale  # [C][Hq][N]
        n = torch.arange(n0 + C, device="cuda")
        mask = n[None, :] <= (n0 + torch.arange(C, device="cuda"))[:, None]  # [C][N]
        lg = lg.masked_fill(~mask[:, None, :], float("-inf"))
        p = torch.softmax(lg, dim=-1)
        out[s] = torch.einsum("chn,hnd->chd", p, v)
        logits_last.append(lg[C - W:])
    return out, logits_last


# lone Q tiles with enough keys split their key tiles over both warpgroups:
# (576, 1000) and (32, 513) split unevenly, (32, 2016) evenly, (64, 100) may
# not split (a row would see no key of the upper half's first tile)
@pytest.mark.parametrize("S,C,Hq,Hkv,n0,W", [(1, 128, 2, 2, 0, 32), (2, 576, 4, 4, 1000, 32), (1, 32, 8, 2, 513, 32),
                                             (2, 200, 4, 1, 300, 16), (1, 32, 4, 4, 2016, 32),
                                             (1, 64, 2, 2, 100, 32), (1, 1, 2, 2, 0, 1), (2, 1, 4, 1, 700, 1)])
def test_prefill_matches_torch(S, C, Hq, Hkv, n0, W):
    _check_prefill(S, C, Hq, Hkv, n0, W, 5)


def _fuzz_shape(seed):
    rng = np.random.default_rng(900 + seed)
    Hkv = int(rng.choice([1, 2, 4]))
    G = int(rng.choice([1, 2, 4, 8]))
    C = int(rng.choice([1, 7, 31, 33, 127, 129, 255, 256, 300, 511, 577, 700]))
    n0 = int(rng.choice([0, 1, 63, 128, 500, 1023, 2048, 2999]))
    W = int(min(C, rng.choice([0, 1, 5, 32, 32, 64, 64])))
    return int(rng.integers(1, 4)), C, G * Hkv, Hkv, n0, W


@pytest.mark.parametrize("seed", list(range(12)))
def test_prefill_fuzz_matches_torch(seed):
    """Seeded random chunk geometries (odd chunk lengths, lone and paired Q
    tiles, empty and tile-boundary prefixes, 0..64 recorded rows, GQA groups up
    to 8) against the float32 PyTorch prompt loop."""
    _check_prefill(*_fuzz_shape(seed), seed)


def _check_prefill(S, C, Hq, Hkv, n0, W, seed):
    from paper_2409_09086_b200 import _lib

    lib = _lib.load()
    D, L, layer = 128, 2, 1
    cap = ((n0 + C + 31) // 32) * 32 + 64
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn((S, C, Hq, D), generator=g, device="cuda").to(torch.bfloat16)
    kc = torch.randn((S, L, Hkv, cap, D), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((S, L, Hkv, cap, D), generator=g, device="cuda").to(torch.bfloat16)
    kc[:, :, :, ::97] *= 4  # key spikes
    out = torch.full((S, C, Hq, D), float("nan"), dtype=torch.float32, device="cuda")
    lg_cap = n0 + C
    logits = torch.zeros((S, max(W, 1), Hq, lg_cap), dtype=torch.float32, device="cuda")
    stats = torch.zeros((S, max(W, 1), Hq, 2), dtype=torch.float32, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    rc = lib.skv_prefill_attend(P(q), S, C, Hq, Hkv, P(kc), P(vc), L, layer, cap, n0, P(out), W, P(logits), lg_cap,
                                P(stats), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(rc)
    torch.cuda.synchronize()
    ref_out, ref_lg = _ref(q.float(), kc[:, layer, :, : n0 + C].float(), vc[:, layer, :, : n0 + C].float(), n0, C, W)
    err = ((out - ref_out).abs().amax(-1) / ref_out.abs().amax(-1)).max().item()
    print(f"prefill S={S} C={C} Hq={Hq} Hkv={Hkv} n0={n0}: output rel err {err:.2e}")
    assert torch.isfinite(out).all()
    assert err <= 2e-3
    for s in range(S):
        for w in range(W):
            i = C - W + w
            nv = n0 + i + 1
            got = logits[s, w, :, :nv]
            want = ref_lg[s][w, :, :nv]
            lerr = ((got - want).abs().amax(-1) / want.abs().amax(-1)).max().item()
            assert lerr <= 1e-5, (s, w, lerr)
            # (M, L) may carry a stale running maximum (lazy O rescale): only
            # p = exp(x - M) / L is the contract, and M may trail the row max
            # by at most 2^8 in the exponent
            M = stats[s, w, :, 0:1]
            Lsum = stats[s, w, :, 1:2]
            mx = want.amax(-1, keepdim=True)
            assert bool((M <= mx + 1e-5 * mx.abs() + 1e-6).all())
            assert bool(((want.amax(-1, keepdim=True) - M) * 1.4426950408889634 <= 8.0 + 1e-4).all())
            p_got = torch.exp(got - M) / Lsum
            p_ref = torch.softmax(want, -1)
            perr = ((p_got - p_ref).abs().amax(-1) / p_ref.amax(-1)).max().item()
            assert perr <= 1e-5, (s, w, perr)


@pytest.mark.parametrize(
    "S,l,W,agg,n_init",
    [(2, 256, 32, "mean", 0), (2, 256, 48, "mean", 0), (2, 256, 32, "max", 0),
     # BASELINE config 2's budget (l = r = 2048) from a full injected cache
     (1, 2048, 32, "mean", 4096)],
    ids=["l256-W32", "l256-W48", "l256-max", "cfg2-budget"],
)
def test_engine_prefill_chunks_match_oracle(S, l, W, agg, n_init):
    """Config-2 shape: 576-token image chunks (k/v = frame mean + 0.5 N(0,1))
    and 32-token text chunks through StreamEngine.prefill_chunk, eviction after
    every chunk, against the CPU oracle stepping the chunk token by token (the
    reference's prompt loop): outputs, window rows, kept sets, K/V after each
    compaction, positions.  W = 48 records more rows than one fold row-group
    (32) holds and wraps the window ring; "max" is aggregate_heads(.., "max")
    (policies.py:263-264) through the chunk fold; the last case runs config
    2's budget l = r = 2048 from a full cache."""
    from oracle.streamkv_oracle import PolicyConfig, StreamOracle, bf16_round, kept_sets_match
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    L, H, D = 1, 32, 128
    r = l
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01, head_agg=agg)
    eng = StreamEngine(EngineConfig(S, L, H, H, D, l, r, 0.01, W, B + 576 + 64, torch.bfloat16, head_agg=agg))
    orc = StreamOracle(S, L, H, H, D, cfg, window=W)
    rng = np.random.default_rng(31)
    F32 = np.float32
    worst = 0.0
    if n_init:
        for s in range(S):
            k0 = bf16_round(rng.standard_normal((H, n_init, D)).astype(F32))
            v0 = bf16_round(rng.standard_normal((H, n_init, D)).astype(F32))
            eng.inject(s, 0, k0, v0, np.arange(n_init, dtype=np.int64))
            for t in range(n_init):
                orc.kv[s][0].append(k0[:, t], v0[:, t], t)
        orc.pos = [n_init] * S
    kept_buf = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    for frame in range(2):
        for C, mod in ((576, 1), (32, 0)):
            q = rng.standard_normal((S, C, H, D)).astype(F32)
            if mod:
                mu_k = rng.standard_normal((S, 1, H, D)).astype(F32)
                mu_v = rng.standard_normal((S, 1, H, D)).astype(F32)
                k = mu_k + F32(0.5) * rng.standard_normal((S, C, H, D)).astype(F32)
                v = mu_v + F32(0.5) * rng.standard_normal((S, C, H, D)).astype(F32)
            else:
                k = rng.standard_normal((S, C, H, D)).astype(F32)
                v = rng.standard_normal((S, C, H, D)).astype(F32)
            q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
            dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.bfloat16)
            got = eng.prefill_chunk(0, dev(q), dev(k), dev(v), modality=mod).cpu().numpy()
            for i in range(C):
                want, _ = orc.step_layer(0, q[:, i][None][0], k[:, i], v[:, i])
                orc.advance()
                g = got[:, i].astype(np.float64)
                worst = max(worst, float((np.abs(g - want).max(-1) / np.abs(want).max(-1)).max()))
            n = orc.length(0, 0)
            rows_g = eng.window_rows(0, 0)
            rows_c = orc.win[0][0].rows
            assert [a.size for a in rows_g] == [b.size for b in rows_c]
            for a_, b_ in zip(rows_g, rows_c):
                assert float(np.abs(a_ - b_).max() / np.abs(b_).max()) <= 1e-5
            eng.evict(-1, kept_buf)
            kc = kept_buf.cpu().numpy()
            for s in range(S):
                if n > B:
                    ok, nbad, gap = kept_sets_match(orc.scores(s, 0), orc.decide(s, 0).kept, kc[s, 0], n, cfg)
                    assert ok, (frame, C, s, nbad, gap)
                    orc.apply(s, 0, kc[s, 0].astype(np.int64))
                else:
                    np.testing.assert_array_equal(kc[s, 0, :n], np.arange(n))
            for s in range(S):
                np.testing.assert_array_equal(eng.positions(s, 0), orc.kv[s][0].pos[: orc.kv[s][0].n])
                kg, vg = eng.kv(s, 0)  # compaction is a pure copy
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][0].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][0].values())
    print(f"engine prefill worst output rel err {worst:.2e}")
    assert worst <= 2e-3


def test_prefill_config2_full_shape():
    """BASELINE config 2's image chunk at full shape (4 streams x 32 heads,
    576 queries over a 4096-token cache + the chunk) against float32 torch,
    on a sample of heads per stream (all CTAs of the launch run)."""
    from paper_2409_09086_b200 import _lib

    lib = _lib.load()
    S, C, H, D, n0, L, W = 4, 576, 32, 128, 4096, 1, 32
    cap = n0 + C + 64
    g = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn((S, C, H, D), generator=g, device="cuda").to(torch.bfloat16)
    kc = torch.randn((S, L, H, cap, D), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((S, L, H, cap, D), generator=g, device="cuda").to(torch.bfloat16)
    kc[:, :, :, ::101] *= 4
    out = torch.full((S, C, H, D), float("nan"), dtype=torch.float32, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    _lib.check(lib.skv_prefill_attend(P(q), S, C, H, H, P(kc), P(vc), L, 0, cap, n0, P(out), 0, None, 0, None,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    scale = 1.0 / np.sqrt(D)
    worst = 0.0
    for s in range(S):
        for h in (0, 7, 19, 31):
            k = kc[s, 0, h, : n0 + C].float()
            v = vc[s, 0, h, : n0 + C].float()
            lg = (q[s, :, h].float() @ k.T) * scale  # [C][n]
            idx = torch.arange(n0 + C, device="cuda")
            mask = idx[None, :] <= (n0 + torch.arange(C, device="cuda"))[:, None]
            p = torch.softmax(lg.masked_fill(~mask, float("-inf")), dim=-1)
            ref = p @ v
            err = ((out[s, :, h] - ref).abs().amax(-1) / ref.abs().amax(-1)).max().item()
            worst = max(worst, err)
    print(f"config-2 full-shape prefill worst rel err {worst:.2e}")
    assert worst <= 2e-3


@pytest.mark.parametrize("seed", list(range(10)))
def test_engine_chunks_and_decode_fuzz(seed):
    """Random engines (1-2 streams and layers, GQA groups 1-4, budgets 64-300,
    W 8-40; seeds 6-9 with RoPE in both position modes) driven through a
    random mix of prefill chunks (1-600 tokens) and decode steps, evicting
    after each phase, against the oracle's per-token loop: chunk and step
    outputs, window rows, kept sets, compacted (raw) K/V."""
    from oracle.streamkv_oracle import PolicyConfig, StreamOracle, bf16_round, kept_sets_match
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    rng = np.random.default_rng(4200 + seed)
    S, L = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    Hkv, G = int(rng.choice([2, 4])), int(rng.choice([1, 2, 4]))
    Hq, D = Hkv * G, 128
    l, r, W = int(rng.integers(64, 301)), int(rng.integers(64, 301)), int(rng.choice([8, 32, 40]))
    B = l + r
    rope = None if seed < 6 else ("cache_relative", "original")[seed % 2]
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, B + 640, torch.bfloat16, rope=rope))
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W, rope=rope, rope_round=bf16_round if rope else None)
    F32 = np.float32
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.bfloat16)
    rnd = lambda *shape: bf16_round(rng.standard_normal(shape).astype(F32))
    kept_buf = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    worst = 0.0
    phases = []
    for _ in range(4):
        phases.append(("chunk", int(rng.choice([1, 17, 32, 129, 300, 576, 600]))))
        phases.append(("decode", int(rng.integers(1, 12))))
    for kind, count in phases:
        if kind == "chunk":
            q, k, v = rnd(L, S, count, Hq, D), rnd(L, S, count, Hkv, D), rnd(L, S, count, Hkv, D)
            got = [eng.prefill_chunk(layer, dev(q[layer]), dev(k[layer]), dev(v[layer])).cpu().numpy()
                   for layer in range(L)]
            for i in range(count):
                for layer in range(L):
                    want, _ = orc.step_layer(layer, q[layer][:, i], k[layer][:, i], v[layer][:, i])
                    g = got[layer][:, i].astype(np.float64)
                    worst = max(worst, float((np.abs(g - want).max(-1) / np.abs(want).max(-1)).max()))
                orc.advance()
        else:
            for _ in range(count):
                q, k, v = rnd(L, S, Hq, D), rnd(L, S, Hkv, D), rnd(L, S, Hkv, D)
                got = eng.decode_step(dev(q), dev(k), dev(v), record=True).cpu().numpy()
                want = orc.step(q, k, v)
                worst = max(worst, float((np.abs(got - want).max(-1) / np.abs(want).max(-1)).max()))
        n = orc.length(0, 0)
        for s in range(S):
            for layer in range(L):
                rows_g, rows_c = eng.window_rows(s, layer), orc.win[s][layer].rows
                assert [a.size for a in rows_g] == [b.size for b in rows_c[-len(rows_g):]] if rows_g else True
                for a_, b_ in zip(rows_g, rows_c[-len(rows_g):]):
                    assert float(np.abs(a_ - b_).max() / np.abs(b_).max()) <= 1e-5, (kind, s, layer)
        kept_buf.fill_(-1)
        eng.evict(-1, kept_buf)
        kc = kept_buf.cpu().numpy()
        for s in range(S):
            for layer in range(L):
                if n > B:
                    ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer], n,
                                                    cfg)
                    assert ok, (kind, count, s, layer, nbad, gap)
                    orc.apply(s, layer, kc[s, layer].astype(np.int64))
                else:
                    np.testing.assert_array_equal(kc[s, layer, :n], np.arange(n))
                kg, vg = eng.kv(s, layer)
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][layer].values())
    print(f"chunk+decode fuzz seed {seed}: S={S} L={L} Hq={Hq} Hkv={Hkv} l={l} r={r} W={W} rope={rope}: "
          f"worst {worst:.2e}")
    assert worst <= 2e-3
