"""GPU robustness: stream ordering of the host-buffer API, domain checks on
the C ABI, the sticky prefill overflow error, per-stream state rules, the
state dump, and caches longer than the segment merge's chunk limit.

Each case either compares against the CPU oracle (tests infrastructure) or
asserts the reference's error behaviour (ValueError for domain errors)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.streamkv_oracle import PolicyConfig, StreamOracle, bf16_round, kept_sets_match  # noqa: E402
from tests.gpu_helpers import rel_err  # noqa: E402

F32 = np.float32


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _eng(S, L, Hq, Hkv, D, l, r, W, cap, dt=torch.bfloat16, **kw):
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    return StreamEngine(EngineConfig(S, L, Hq, Hkv, D, l, r, 0.01, W, cap, dt, **kw))


def _inject_both(eng, orc, rng, S, L, Hkv, D, n0):
    for s in range(S):
        for layer in range(L):
            k = bf16_round(rng.standard_normal((Hkv, n0, D)).astype(F32))
            v = bf16_round(rng.standard_normal((Hkv, n0, D)).astype(F32))
            eng.inject(s, layer, k, v, np.arange(n0, dtype=np.int64))
            for t in range(n0):
                orc.kv[s][layer].append(k[:, t], v[:, t], t)
    orc.pos = [n0] * S


def test_decode_step_host_ordered_after_evict_and_prefill():
    """skv_decode_step_host must not overtake an eviction or a
    prefill chunk the caller enqueued without synchronising; checked against
    the oracle running the same sequence."""
    S, L, Hq, Hkv, D = 2, 2, 16, 4, 128
    l, r, W, E, C = 256, 256, 16, 32, 48
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = _eng(S, L, Hq, Hkv, D, l, r, W, B + E + C + 8)
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W)
    rng = np.random.default_rng(9)
    _inject_both(eng, orc, rng, S, L, Hkv, D, B)
    out_h = torch.empty((L, S, Hq, D), dtype=torch.float32).pin_memory()
    worst = 0.0

    def inputs(lead):
        q = bf16_round(rng.standard_normal((*lead, Hq, D)).astype(F32))
        k = bf16_round(rng.standard_normal((*lead, Hkv, D)).astype(F32))
        v = bf16_round(rng.standard_normal((*lead, Hkv, D)).astype(F32))
        return q, k, v

    def host_step():
        nonlocal worst
        q, k, v = inputs((L, S))
        hq, hk, hv = (torch.from_numpy(a).to(torch.bfloat16).pin_memory() for a in (q, k, v))
        eng.decode_step_host(hq, hk, hv, out_h, record=True)
        worst = max(worst, rel_err(out_h.numpy(), orc.step(q, k, v)))

    for _ in range(E):
        host_step()
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    eng.evict(-1, kept)
    n = B + E
    decisions = {(s, layer): orc.decide(s, layer) for s in range(S) for layer in range(L)}
    scores = {(s, layer): orc.scores(s, layer) for s in range(S) for layer in range(L)}
    host_q = inputs((L, S))  # generated before the kept sets are read back
    hq, hk, hv = (torch.from_numpy(a).to(torch.bfloat16).pin_memory() for a in host_q)
    eng.decode_step_host(hq, hk, hv, out_h, record=True)  # no sync after the eviction
    kc = kept.cpu().numpy()
    for (s, layer), d in decisions.items():
        ok, nbad, gap = kept_sets_match(scores[(s, layer)], d.kept, kc[s, layer], n, cfg)
        assert ok, (s, layer, nbad, gap)
        orc.apply(s, layer, kc[s, layer].astype(np.int64))
    worst = max(worst, rel_err(out_h.numpy(), orc.step(*host_q)))
    # prefill chunk, then a host step without synchronising
    q, k, v = inputs((L, S, C))
    kv_in = [tuple(torch.from_numpy(np.ascontiguousarray(a[layer])).to("cuda", torch.bfloat16) for a in (q, k, v))
             for layer in range(L)]
    for layer in range(L):
        eng.prefill_chunk(layer, *kv_in[layer])
    for i in range(C):
        orc.step(q[:, :, i], k[:, :, i], v[:, :, i])
    host_step()
    print(f"worst output rel err {worst:.2e}")
    assert worst <= 2e-3


def test_head_agg_max_rejected_when_head_sharded():
    """a shard's max over its heads cannot be summed across shards."""
    with pytest.raises(ValueError, match="max"):
        _eng(1, 1, 8, 2, 128, 32, 32, 8, 128, head_agg="max", heads_q_total=16)
    _eng(1, 1, 8, 2, 128, 32, 32, 8, 128, head_agg="max").close()  # unsharded max is fine


def test_prefill_large_v_raises_on_sync():
    """|v| >= 65504 saturates the prefill's fp16 V -- the
    engine reports it (sticky ValueError on sync / host reads) instead of
    returning silently wrong outputs."""
    S, L, H, D, C = 1, 1, 4, 128, 64
    eng = _eng(S, L, H, H, D, 64, 64, 8, 64 + 64 + C)
    rng = np.random.default_rng(3)
    q = torch.from_numpy(rng.standard_normal((S, C, H, D)).astype(F32)).to("cuda", torch.bfloat16)
    k = torch.from_numpy(rng.standard_normal((S, C, H, D)).astype(F32)).to("cuda", torch.bfloat16)
    v = torch.from_numpy(rng.standard_normal((S, C, H, D)).astype(F32)).to("cuda", torch.bfloat16)
    eng.prefill_chunk(0, q, k, v)
    eng.sync()  # in range: no error
    v2 = v.clone()
    v2[0, 5, 1, 7] = 70000.0
    eng.prefill_chunk(0, q, k, v2)
    with pytest.raises(ValueError, match="65504"):
        eng.sync()
    eng.sync()  # reported once, then cleared


def test_inject_validates_window_rows_and_ragged_streams():
    """row lengths must lie in [1, n] and never shrink; streams of a
    layer that disagree refuse work (SKV_ESTATE) until injected alike."""
    S, L, H, D = 2, 1, 4, 64
    eng = _eng(S, L, H, H, D, 16, 16, 4, 64, dt=torch.float32)
    n = 40
    k = np.zeros((H, n, D), F32)
    pos = np.arange(n, dtype=np.int64)
    with pytest.raises(ValueError):
        eng.inject(0, 0, k, k, pos, rows=[np.ones(n + 5, F32)])  # longer than n
    with pytest.raises(ValueError):
        eng.inject(0, 0, k, k, pos, rows=[np.ones(30, F32), np.ones(20, F32)])  # shrinks
    eng.inject(0, 0, k, k, pos, rows=[np.ones(20, F32) / 20, np.ones(n, F32) / n])
    q = torch.zeros((S, H, D), device="cuda")
    with pytest.raises(RuntimeError, match="lock step"):
        eng.decode_layer(0, q, q, q)  # stream 1 not injected yet
    assert eng.length(0, 0) == n
    eng.inject(1, 0, k, k, pos, rows=[np.ones(20, F32) / 20, np.ones(n, F32) / n])
    eng.decode_layer(0, q, q, q)
    assert eng.length(1, 0) == n + 1


def test_state_dump_roundtrip():
    """skv_state_dump returns what skv_state_inject wrote, and the cache after
    decode steps + an eviction in logical order."""
    S, L, Hq, Hkv, D = 2, 2, 8, 2, 128
    l, r, W, E = 32, 32, 8, 16
    B = l + r
    eng = _eng(S, L, Hq, Hkv, D, l, r, W, B + E)
    rng = np.random.default_rng(12)
    ks, vs = {}, {}
    for s in range(S):
        for layer in range(L):
            k = bf16_round(rng.standard_normal((Hkv, B, D)).astype(F32))
            v = bf16_round(rng.standard_normal((Hkv, B, D)).astype(F32))
            rows = [rng.dirichlet(np.ones(B)).astype(F32) for _ in range(3)]
            eng.inject(s, layer, k, v, np.arange(B, dtype=np.int64) * 3, rows=rows)
            ks[s, layer], vs[s, layer] = k, v
            d = eng.state_dump(s, layer)
            assert d["n"] == B
            np.testing.assert_array_equal(d["keys"], k)
            np.testing.assert_array_equal(d["values"], v)
            np.testing.assert_array_equal(d["original_positions"], np.arange(B) * 3)
            assert len(d["rows"]) == 3
            for a, b in zip(d["rows"], rows):
                np.testing.assert_array_equal(a, b)
    for t in range(E):
        q = torch.from_numpy(rng.standard_normal((L, S, Hq, D)).astype(F32)).to("cuda", torch.bfloat16)
        kk = torch.from_numpy(rng.standard_normal((L, S, Hkv, D)).astype(F32)).to("cuda", torch.bfloat16)
        eng.decode_step(q, kk, kk, record=True)
    eng.evict(-1)
    for s in range(S):
        for layer in range(L):
            d = eng.state_dump(s, layer)
            kg, vg = eng.kv(s, layer)
            np.testing.assert_array_equal(d["keys"], kg.float().cpu().numpy())
            np.testing.assert_array_equal(d["values"], vg.float().cpu().numpy())
            np.testing.assert_array_equal(d["original_positions"], eng.positions(s, layer))
            assert d["n"] == B and len(d["rows"]) == W


@pytest.mark.parametrize("G", [1, 4])
def test_cache_longer_than_merge_chunk_limit(G):
    """caches beyond 128 chunks of the default chunk size (n > 32K)
    take longer chunks instead of failing mid-stream."""
    Hkv, D = 2, 128
    Hq = Hkv * G
    n0 = 40_000
    eng = _eng(1, 1, Hq, Hkv, D, 64, 64, 4, n0 + 8)
    g = torch.Generator(device="cuda").manual_seed(1)
    kf, vf = eng.kv_full(0, 0)
    kf[:, :n0] = torch.randn((Hkv, n0, D), generator=g, device="cuda").to(torch.bfloat16)
    vf[:, :n0] = torch.randn((Hkv, n0, D), generator=g, device="cuda").to(torch.bfloat16)
    eng.lib.skv_state_inject(eng._h, 0, 0, n0, None, None, None, 0, None, None)
    for _ in range(3):
        q = torch.randn((1, Hq, D), generator=g, device="cuda").to(torch.bfloat16)
        k = torch.randn((1, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn((1, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
        out = eng.decode_layer(0, q, k, v, record=False)
        n = eng.length(0, 0)
        kk, vv = eng.kv(0, 0)
        K = kk.float().repeat_interleave(G, 0)
        V = vv.float().repeat_interleave(G, 0)
        p = torch.softmax((K @ q[0].float()[:, :, None])[..., 0] / np.sqrt(D), dim=-1)
        ref = (p[:, None, :] @ V)[:, 0]
        assert n == n0 + _ + 1
        assert rel_err(out[0].cpu().numpy(), ref.cpu().numpy()) < 2e-3


def test_slot_map_moves_only_the_survivors_of_the_period():
    """Slot-map compaction: with l >= E every token appended in the period is
    in the recent window, so exactly E rows move per (stream, layer) -- not
    the ~B rows a stable in-place shift moves -- and the cache read back in
    logical order equals the oracle's gather_keep (cache.py:136-156)."""
    S, L, Hq, Hkv, D = 2, 2, 8, 2, 128
    l, r, W, E = 64, 64, 8, 32
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = _eng(S, L, Hq, Hkv, D, l, r, W, B + E)
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W)
    rng = np.random.default_rng(21)
    _inject_both(eng, orc, rng, S, L, Hkv, D, B)
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    for period in range(3):
        for _ in range(E):
            q = bf16_round(rng.standard_normal((L, S, Hq, D)).astype(F32))
            k = bf16_round(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            v = bf16_round(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            eng.decode_step(*(torch.from_numpy(a).to("cuda", torch.bfloat16) for a in (q, k, v)), record=True)
            orc.step(q, k, v)
        eng.evict(-1, kept)
        kc = kept.cpu().numpy()
        np.testing.assert_array_equal(eng.moved_rows(), np.full((S, L), E))
        for s in range(S):
            for layer in range(L):
                ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer],
                                                B + E, cfg)
                assert ok, (period, s, layer, nbad, gap)
                orc.apply(s, layer, kc[s, layer].astype(np.int64))
                kg, vg = eng.kv(s, layer)
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][layer].values())
                perm = eng.slot_map(s, layer).cpu().numpy()
                assert sorted(perm.tolist()) == list(range(B))  # rows [0, B) hold exactly the kept tokens
    # cache-relative RoPE engines compact densely (their moved keys change position anyway)
    dense = _eng(1, 1, 8, 2, 128, 32, 32, 8, 80, rope="cache_relative")
    assert dense.moved_rows() is None and dense.slot_map(0, 0) is None


@pytest.mark.parametrize("G,L,l,E,periods", [(4, 4, 512, 64, 3), (8, 4, 512, 64, 3), (4, 2, 2048, 256, 1)],
                         ids=["G4", "G8", "G4-cfg3-budget"])
def test_all_layer_persistent_decode_matches_oracle(G, L, l, E, periods):
    """decode_step of a latency-bound GQA engine runs all layers in one
    persistent launch (decode_tc_cluster_kernel: one cluster per segment,
    segment merge over distributed shared memory, layer l+1 released by layer
    l's outputs).  Against the oracle: outputs, window rows, kept sets,
    compacted K/V.  The config-3 budget case (4096 + 256 tokens: 65-68 tiles per
    segment) runs 7-tile chunks on clusters of 10."""
    S, Hkv, D = 1, 32 // G, 128
    Hq = Hkv * G
    r, W = l, 16
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = _eng(S, L, Hq, Hkv, D, l, r, W, B + E)
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W)
    rng = np.random.default_rng(60 + G)
    _inject_both(eng, orc, rng, S, L, Hkv, D, B)
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    worst = worst_row = 0.0
    for period in range(periods):
        for t in range(E):
            q = bf16_round(rng.standard_normal((L, S, Hq, D)).astype(F32))
            k = bf16_round(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            v = bf16_round(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            before = eng.kernel_launches
            got = eng.decode_step(*(torch.from_numpy(a).to("cuda", torch.bfloat16) for a in (q, k, v)),
                                  record=t >= E - W).cpu().numpy()
            assert eng.kernel_launches - before in (1, 2 * L)  # one launch for all layers (SKV_LAYERS=1)
            worst = max(worst, rel_err(got, orc.step(q, k, v)))
        for s in range(S):
            for layer in range(L):
                for a_, b_ in zip(eng.window_rows(s, layer), orc.win[s][layer].rows[-W:]):
                    worst_row = max(worst_row, float(np.abs(a_ - b_).max() / np.abs(b_).max()))
        eng.evict(-1, kept)
        kc = kept.cpu().numpy()
        for s in range(S):
            for layer in range(L):
                ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer],
                                                B + E, cfg)
                assert ok, (period, s, layer, nbad, gap)
                orc.apply(s, layer, kc[s, layer].astype(np.int64))
                kg, vg = eng.kv(s, layer)
                np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys())
                np.testing.assert_array_equal(vg.float().cpu().numpy(), orc.kv[s][layer].values())
                np.testing.assert_array_equal(eng.positions(s, layer), orc.kv[s][layer].pos[: orc.kv[s][layer].n])
    print(f"persistent G={G}: worst out {worst:.2e} rows {worst_row:.2e}")
    assert worst <= 2e-3 and worst_row <= 2e-3


@pytest.mark.parametrize("L", [3, 4], ids=["eager-L3", "graph-L4"])
def test_host_step_graph_cache_over_periods(L):
    """skv_decode_step_host (from the engine's very first call) over three
    eviction periods: L = 4 runs each token as one CUDA graph cached per engine
    state (cache hits rebind only the copy nodes to new pinned buffers; the
    all-layer cluster launch and its fit query are captured), L = 3 the eager
    whole-token path.  Outputs every token, kept sets every period, against
    the oracle."""
    S, Hq, Hkv, D = 2, 8, 2, 128
    l, r, W, E = 32, 32, 8, 16
    B = l + r
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    eng = _eng(S, L, Hq, Hkv, D, l, r, W, B + E)
    orc = StreamOracle(S, L, Hq, Hkv, D, cfg, window=W)
    rng = np.random.default_rng(77)
    _inject_both(eng, orc, rng, S, L, Hkv, D, B)
    kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
    worst = 0.0
    for period in range(3):
        for t in range(E):
            q = bf16_round(rng.standard_normal((L, S, Hq, D)).astype(F32))
            k = bf16_round(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            v = bf16_round(rng.standard_normal((L, S, Hkv, D)).astype(F32))
            hq, hk, hv = (torch.from_numpy(a).to(torch.bfloat16).pin_memory() for a in (q, k, v))
            oh = torch.full((L, S, Hq, D), float("nan"), dtype=torch.float32).pin_memory()
            eng.decode_step_host(hq, hk, hv, oh, record=t >= E - W)
            worst = max(worst, rel_err(oh.numpy(), orc.step(q, k, v)))
        eng.evict(-1, kept)
        kc = kept.cpu().numpy()
        for s in range(S):
            for layer in range(L):
                ok, nbad, gap = kept_sets_match(orc.scores(s, layer), orc.decide(s, layer).kept, kc[s, layer],
                                                B + E, cfg)
                assert ok, (period, s, layer, nbad, gap)
                orc.apply(s, layer, kc[s, layer].astype(np.int64))
    assert worst <= 2e-3, worst


def test_adversarial_kept_sets_dense_compaction_vs_torch_gather():
    """K3's in-place stable compaction (skv_gather_rows / KvCache.gather_keep)
    on adversarial kept sets -- everything but the first row, every other
    row, only the last row, a single gap, runs of holes, random -- against a
    torch gather of the same rows (stands in for compute-sanitizer, which the
    GPU pool does not allow)."""
    import ctypes

    from paper_2409_09086_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(8)
    H, n, D = 8, 3000, 128
    for name, kept in [
        ("drop-first", np.arange(1, n)),
        ("every-other", np.arange(0, n, 2)),
        ("last-only", np.array([n - 1])),
        ("single-gap", np.delete(np.arange(n), n // 2)),
        ("runs", np.concatenate([np.arange(i, i + 7) for i in range(0, n - 7, 19)])),
        ("random", np.sort(rng.choice(n, size=n // 3, replace=False))),
        ("identity", np.arange(n)),
    ]:
        for dt in (torch.bfloat16, torch.float32):
            x = torch.randn((H, n, D), device="cuda").to(dt)
            ref = x[:, torch.from_numpy(kept).cuda()].clone()
            kd = torch.from_numpy(kept.astype(np.int64)).cuda()
            row_bytes = D * x.element_size()
            _lib.check(lib.skv_gather_rows(ctypes.c_void_p(x.data_ptr()), n * row_bytes, H, row_bytes,
                                           ctypes.c_void_p(kd.data_ptr()), kept.size,
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
            assert torch.equal(x[:, : kept.size], ref), (name, dt)


def test_full_size_config1_period_is_deterministic():
    """Config 1 at full size: the same period replayed from the same state twice
    gives bit-identical outputs, kept sets, slot maps and caches (the split-KV
    merge combines chunk partials in chunk order, whatever the ticket order)."""
    from paper_2409_09086_b200 import EngineConfig, StreamEngine

    S, L, H, D, l, r, W, E = 8, 32, 32, 128, 1024, 1024, 32, 128
    B = l + r
    results = []
    for rep in range(2):
        eng = StreamEngine(EngineConfig(S, L, H, H, D, l, r, 0.01, W, B + E, torch.bfloat16))
        g = torch.Generator(device="cuda").manual_seed(99)
        for s in range(S):
            for layer in range(L):
                kf, vf = eng.kv_full(s, layer)
                kf[:, :B] = torch.randn((H, B, D), generator=g, device="cuda").to(torch.bfloat16)
                vf[:, :B] = torch.randn((H, B, D), generator=g, device="cuda").to(torch.bfloat16)
                eng.lib.skv_state_inject(eng._h, s, layer, B, None, None, None, 0, None, None)
        q = torch.randn((E, L, S, H, D), generator=g, device="cuda").to(torch.bfloat16)
        k = torch.randn((E, L, S, H, D), generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn((E, L, S, H, D), generator=g, device="cuda").to(torch.bfloat16)
        out = torch.empty((L, S, H, D), dtype=torch.float32, device="cuda")
        outs = []
        for t in range(E):
            eng.decode_step(q[t], k[t], v[t], out, record=t >= E - W)
            outs.append(out[:, :2].clone())
        kept = torch.full((S, L, B), -1, dtype=torch.int32, device="cuda")
        eng.evict(-1, kept)
        torch.cuda.synchronize()
        results.append((torch.stack(outs).cpu(), kept.cpu(), eng.slot_map(3, 17).cpu(),
                         eng.kv(5, 9)[0].cpu(), eng.kv(0, 31)[1].cpu()))
        eng.close()
    for a_, b_ in zip(*results):
        assert torch.equal(a_, b_)


def test_dynamic_decode_kernels_both_match_oracle():
    """Throughput launches (dynamic chunk tickets) run decode_tcd_kernel (tensor
    cores) by default and decode_kernel (CUDA cores) with SKV_TCD=0: the
    config-1 sampled-lane and baseline-shape parity tests, in a subprocess per
    setting (the switch is read once per process), plus the kernel the engine
    reports."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for flag, want in (("1", "decode_tcd_kernel"), ("0", "decode_kernel")):
        env = dict(os.environ, SKV_TCD=flag)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                            "sampled_lanes or baseline_shapes or instantiations"],
                           env=env, cwd=root, capture_output=True, text=True, timeout=1200)
        assert r.returncode == 0, (flag, r.stdout[-3000:], r.stderr[-2000:])
        probe = ("import torch; from paper_2409_09086_b200 import EngineConfig, StreamEngine\n"
                 "e = StreamEngine(EngineConfig(8, 2, 32, 32, 128, 1024, 1024, 0.01, 32, 2200, torch.bfloat16))\n"
                 "for s in range(8):\n"
                 "    for l in range(2):\n"
                 "        e.lib.skv_state_inject(e._h, s, l, 2048, None, None, None, 0, None, None)\n"
                 "q = torch.randn((2, 8, 32, 128), device='cuda').bfloat16()\n"
                 "e.decode_step(q, q, q)\nprint(e.last_decode_kernel)")
        r = subprocess.run([sys.executable, "-c", probe], env=env, cwd=root, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        assert r.stdout.strip().splitlines()[-1] == want, (flag, r.stdout)


def test_project_row_matches_reference_projection():
    """skv_project_row (the trace replay's per-row projection, replay.py:139-142):
    probs[live] divided by their float64 total and rounded to f32 -- exact
    against the same NumPy arithmetic; an all-zero projection stays unscaled;
    m = 0 is a no-op."""
    import ctypes

    from paper_2409_09086_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for n, m, zero in ((5000, 3000, False), (64, 64, False), (300, 17, True), (10, 0, False)):
        probs = rng.random(n).astype(np.float32) ** 4
        if zero:
            probs[:] = 0.0
        live = np.sort(rng.choice(n, size=m, replace=False)).astype(np.int64)
        out = torch.full((max(m, 1),), -7.0, dtype=torch.float32, device="cuda")
        pd, ld = torch.from_numpy(probs).cuda(), torch.from_numpy(live).cuda() if m else torch.zeros(1, dtype=torch.int64,
                                                                                                    device="cuda")
        _lib.check(lib.skv_project_row(P(pd), n, P(ld), m, P(out), st))
        got = out.cpu().numpy()[:m]
        proj = probs[live]
        total = proj.sum(dtype=np.float64)
        want = (proj / total).astype(np.float32) if total > 0 else proj
        np.testing.assert_array_equal(got, want)
        if m == 0:
            assert out.cpu().numpy()[0] == -7.0


def test_host_steps_with_staging_copies_match_reference():
    """SKV_HOST_ZC=0 (staging buffers and copies instead of addressing the
    caller's mapped pinned buffers): the golden host-step runs and the
    host-step fuzz, in a subprocess (the switch is read once per process)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), os.path.join(root, "tests", "test_gpu_fuzz.py"),
                        "-k", "host_steps"], env=dict(os.environ, SKV_HOST_ZC="0"), cwd=root, capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
    assert " passed" in r.stdout and " failed" not in r.stdout
