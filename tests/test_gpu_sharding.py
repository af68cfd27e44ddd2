"""GPU parity of the head-sharded (config 3) path: two KV-head shards run as two
engines on one GPU (no rank waits on another: the cross-shard reduction is the
host-side sum that ``evict_head_sharded`` performs with an all-reduce on a
real multi-GPU job), compared with the unsharded reference-semantics oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.streamkv_oracle import PolicyConfig, StreamOracle, bf16_round, kept_sets_match, synth_step  # noqa: E402
from tests.gpu_helpers import rel_err  # noqa: E402

F32 = np.float32


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_two_kv_head_shards_match_unsharded_reference():
    from paper_2409_09086_b200 import EngineConfig, StreamEngine
    from paper_2409_09086_b200.sharding import shard_heads

    S, L, HQ, HKV, D = 1, 2, 32, 8, 128
    l, r, W, E, periods = 512, 512, 32, 128, 2
    B = l + r
    G = HQ // HKV
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    world = 2
    engines, blocks = [], []
    for rank in range(world):
        kvs, qs = shard_heads(HKV, G, world, rank)
        blocks.append((kvs, qs))
        engines.append(StreamEngine(EngineConfig(S, L, qs.stop - qs.start, kvs.stop - kvs.start, D, l, r, 0.01, W,
                                                 B + E, torch.bfloat16, heads_q_total=HQ)))
    orc = StreamOracle(S, L, HQ, HKV, D, cfg, window=W)
    rng = np.random.default_rng(99)
    for s in range(S):
        for layer in range(L):
            k = bf16_round(rng.standard_normal((HKV, B, D)).astype(F32))
            v = bf16_round(rng.standard_normal((HKV, B, D)).astype(F32))
            pos = np.arange(B, dtype=np.int64)
            for (kvs, _), eng in zip(blocks, engines):
                eng.inject(s, layer, k[kvs], v[kvs], pos)
            for t in range(B):
                orc.kv[s][layer].append(k[:, t], v[:, t], t)
    orc.pos = [B] * S
    worst = 0.0
    for period in range(periods):
        for t in range(E):
            qs_, ks_, vs_ = zip(*[synth_step(rng, S, HQ, HKV, D, 0.005, 4.0, True) for _ in range(L)])
            q, k, v = np.stack(qs_), np.stack(ks_), np.stack(vs_)
            want = orc.step(q, k, v)
            for (kvs, qsl), eng in zip(blocks, engines):
                dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.bfloat16)
                got = eng.decode_step(dev(q[:, :, qsl]), dev(k[:, :, kvs]), dev(v[:, :, kvs]), record=True)
                worst = max(worst, rel_err(got.cpu().numpy(), want[:, :, qsl]))
        n = orc.length(0, 0)
        # what evict_head_sharded does on a multi-GPU job: sum the shards' scores
        scores = sum(eng.evict_scores(-1) for eng in engines)
        kept = [torch.full((S, L, B), -1, dtype=torch.int32, device="cuda") for _ in engines]
        for eng, kb in zip(engines, kept):
            eng.evict_apply(scores, -1, kb)
        k0, k1 = kept[0].cpu().numpy(), kept[1].cpu().numpy()
        np.testing.assert_array_equal(k0, k1)
        for s in range(S):
            for layer in range(L):
                sc = orc.scores(s, layer)
                d = orc.decide(s, layer)
                ok, nbad, gap = kept_sets_match(sc, d.kept, k0[s, layer], n, cfg)
                assert ok, (period, s, layer, nbad, gap)
                orc.apply(s, layer, k0[s, layer].astype(np.int64))
                for (kvs, _), eng in zip(blocks, engines):
                    kg, _ = eng.kv(s, layer)
                    np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[s][layer].keys()[kvs])
    print(f"sharded worst output rel err {worst:.2e}")
    assert worst <= 2e-3


@pytest.mark.parametrize("world", [1, 2])
def test_kv_head_selection_matches_per_group_reference(world):
    """select="kv_head" (the collective-free mode): every
    KV-head group keeps its own window of G-head mean rows and its own
    Algorithm-1 decision.  Oracle: the reference pipeline run per group
    (StreamOracle over S*Hkv pseudo-streams of one KV head and G query heads).
    With world = 2 the KV heads split over two shard engines that never
    exchange anything."""
    from paper_2409_09086_b200 import EngineConfig
    from paper_2409_09086_b200.sharding import KvHeadEngine, shard_heads

    S, L, HQ, HKV, D = 1, 2, 32, 8, 128
    l, r, W, E, periods = 256, 256, 32, 64, 2
    B = l + r
    G = HQ // HKV
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.01)
    shards = []
    for rank in range(world):
        kvs, qs = shard_heads(HKV, G, world, rank)
        eng = KvHeadEngine(EngineConfig(S, L, qs.stop - qs.start, kvs.stop - kvs.start, D, l, r, 0.01, W, B + E,
                                        torch.bfloat16))
        shards.append((kvs, qs, eng))
    orc = StreamOracle(S * HKV, L, G, 1, D, cfg, window=W)  # one pseudo-stream per KV-head group
    rng = np.random.default_rng(123)
    for s in range(S):
        for layer in range(L):
            k = bf16_round(rng.standard_normal((HKV, B, D)).astype(F32))
            v = bf16_round(rng.standard_normal((HKV, B, D)).astype(F32))
            pos = np.arange(B, dtype=np.int64)
            for kvs, _, eng in shards:
                for gl, g in enumerate(range(kvs.start, kvs.stop)):
                    eng.inject_group(s, layer, gl, k[g:g + 1], v[g:g + 1], pos)
            for g in range(HKV):
                for t in range(B):
                    orc.kv[s * HKV + g][layer].append(k[g:g + 1, t], v[g:g + 1, t], t)
    orc.pos = [B] * (S * HKV)
    worst = 0.0
    for period in range(periods):
        for t in range(E):
            qs_, ks_, vs_ = zip(*[synth_step(rng, S, HQ, HKV, D, 0.005, 4.0, True) for _ in range(L)])
            q, k, v = np.stack(qs_), np.stack(ks_), np.stack(vs_)
            want = orc.step(q.reshape(L, S * HKV, G, D), k.reshape(L, S * HKV, 1, D), v.reshape(L, S * HKV, 1, D))
            want = want.reshape(L, S, HQ, D)
            for kvs, qsl, eng in shards:
                dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.bfloat16)
                got = eng.decode_step(dev(q[:, :, qsl]), dev(k[:, :, kvs]), dev(v[:, :, kvs]), record=True)
                worst = max(worst, rel_err(got.cpu().numpy(), want[:, :, qsl]))
        n = orc.length(0, 0)
        for kvs, _, eng in shards:
            hk = kvs.stop - kvs.start
            kept = torch.full((S, hk, L, B), -1, dtype=torch.int32, device="cuda")
            eng.evict(-1, kept)
            kc = kept.cpu().numpy()
            for s in range(S):
                for gl, g in enumerate(range(kvs.start, kvs.stop)):
                    ps = s * HKV + g
                    for layer in range(L):
                        d = orc.decide(ps, layer)
                        ok, nbad, gap = kept_sets_match(orc.scores(ps, layer), d.kept, kc[s, gl, layer], n, cfg)
                        assert ok, (period, s, g, layer, nbad, gap)
                        orc.apply(ps, layer, kc[s, gl, layer].astype(np.int64))
                        kg, _ = eng.inner.kv(s * hk + gl, layer)
                        np.testing.assert_array_equal(kg.float().cpu().numpy(), orc.kv[ps][layer].keys())
    print(f"kv_head world={world} worst output rel err {worst:.2e}")
    assert worst <= 2e-3
