"""Head-sharded (config 3) eviction logic on CPU with a world-size-2 gloo group.

Each rank owns half of the KV heads (and their query heads).  A CPU stand-in
engine built from the oracle provides the same ``evict_scores`` /
``evict_apply`` contract as ``StreamEngine``; the product function
``evict_head_sharded`` all-reduces the shard scores.  The kept sets must equal
the unsharded reference-semantics oracle (per-layer selection over all heads),
up to the near-tie rule.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from oracle.streamkv_oracle import (
    LayerKV,
    PolicyConfig,
    RowWindow,
    StreamOracle,
    age_bias,
    attend_heads,
    kept_sets_match,
    top_k_newer,
    window_scores,
)
from paper_2409_09086_b200.sharding import evict_head_sharded, shard_heads

F32 = np.float32
S, L, HQ, HKV, D = 2, 2, 8, 4, 64
l, r, W, E, T = 16, 16, 8, 16, 80
CAP = l + r + E


class OracleShard:
    """CPU stand-in with StreamEngine's sharded-eviction contract (test infra)."""

    def __init__(self, qs, kvs, hq_total, cfg):
        self.qs, self.kvs, self.hq_total, self.cfg = qs, kvs, hq_total, cfg
        self.G = (qs.stop - qs.start) // (kvs.stop - kvs.start)
        self.kv = [[LayerKV(kvs.stop - kvs.start, D) for _ in range(L)] for _ in range(S)]
        self.win = [[RowWindow(W) for _ in range(L)] for _ in range(S)]

    def step(self, t, q, k, v):  # full-model q (L,S,HQ,D), k/v (L,S,HKV,D)
        for layer in range(L):
            for s in range(S):
                st = self.kv[s][layer]
                st.append(k[layer, s, self.kvs], v[layer, s, self.kvs], t)
                keys = np.repeat(st.keys(), self.G, axis=0)
                vals = np.repeat(st.values(), self.G, axis=0)
                probs, _ = attend_heads(keys, vals, q[layer, s, self.qs], F32(1 / np.sqrt(D)))
                self.win[s][layer].push(probs.sum(axis=0, dtype=F32) / F32(self.hq_total))

    def evict_scores(self, layer=-1):
        out = torch.zeros((S, L, CAP), dtype=torch.float32)
        for s in range(S):
            for ly in range(L):
                n = self.kv[s][ly].n
                if n > l + r:
                    out[s, ly, : n - l] = torch.from_numpy(window_scores(self.win[s][ly], n, l))
        return out

    def evict_apply(self, scores, layer=-1, kept=None):
        res = []
        for s in range(S):
            per = []
            for ly in range(L):
                n = self.kv[s][ly].n
                if n <= l + r:
                    ks = np.arange(n)
                else:
                    biased = scores[s, ly, : n - l].numpy().astype(F32) + age_bias(n, l, self.cfg.bias)
                    ks = np.concatenate([top_k_newer(biased, r), np.arange(n - l, n)])
                if ks.size != n:
                    self.kv[s][ly].gather_keep(ks)
                    self.win[s][ly].remap(ks)
                per.append(ks)
            res.append(per)
        return res


def _worker(rank, world, port, q_all, k_all, v_all, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.05)
        kvs, qs = shard_heads(HKV, HQ // HKV, world, rank)
        eng = OracleShard(qs, kvs, HQ, cfg)
        decisions = []
        for t in range(T):
            eng.step(t, q_all[t], k_all[t], v_all[t])
            if (t + 1) % E == 0:
                decisions.append(evict_head_sharded(eng))
        ret[rank] = decisions
    finally:
        dist.destroy_process_group()


def test_head_sharded_eviction_matches_unsharded_oracle():
    rng = np.random.default_rng(77)
    q_all = rng.standard_normal((T, L, S, HQ, D)).astype(F32)
    k_all = rng.standard_normal((T, L, S, HKV, D)).astype(F32)
    v_all = rng.standard_normal((T, L, S, HKV, D)).astype(F32)
    k_all[rng.random((T, L, S)) < 0.05] *= F32(4)
    mgr = tmp.Manager()
    ret = mgr.dict()
    port = 29500 + int(rng.integers(0, 2000))
    tmp.spawn(_worker, args=(2, port, q_all, k_all, v_all, ret), nprocs=2, join=True)
    # both ranks must take identical decisions
    d0, d1 = ret[0], ret[1]
    assert len(d0) == len(d1) == T // E
    for a, b in zip(d0, d1):
        for s in range(S):
            for ly in range(L):
                np.testing.assert_array_equal(a[s][ly], b[s][ly])
    # and they must be the reference's (per-layer selection over all heads)
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.05)
    orc = StreamOracle(S, L, HQ, HKV, D, cfg, window=W)
    ei = 0
    for t in range(T):
        orc.step(q_all[t], k_all[t], v_all[t])
        if (t + 1) % E == 0:
            for s in range(S):
                for ly in range(L):
                    n = orc.length(s, ly)
                    want = orc.decide(s, ly).kept
                    got = d0[ei][s][ly]
                    if n > l + r:
                        ok, nbad, gap = kept_sets_match(orc.scores(s, ly), want, got, n, cfg)
                        assert ok, (t, s, ly, nbad, gap)
                    else:
                        np.testing.assert_array_equal(got, want)
                    orc.apply(s, ly, got)
            ei += 1


def test_shard_heads_partition():
    blocks = [shard_heads(8, 4, 4, rk) for rk in range(4)]
    assert [b[0] for b in blocks] == [slice(0, 2), slice(2, 4), slice(4, 6), slice(6, 8)]
    assert [b[1] for b in blocks] == [slice(0, 8), slice(8, 16), slice(16, 24), slice(24, 32)]
    with pytest.raises(ValueError):
        shard_heads(8, 4, 3, 0)


def _gather_worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_09086_b200.sharding import gather_results

        # rank r holds streams [2r, 2r + r + 1): ragged blocks along dim 0
        t = torch.arange(10 * rank, 10 * rank + 4 * (rank + 1), dtype=torch.int32).reshape(rank + 1, 4)
        ret[rank] = gather_results(t).numpy()
    finally:
        dist.destroy_process_group()


def test_gather_results_concatenates_rank_blocks():
    mgr = tmp.Manager()
    ret = mgr.dict()
    port = 31500 + int(np.random.default_rng().integers(0, 2000))
    tmp.spawn(_gather_worker, args=(2, port, ret), nprocs=2, join=True)
    want = np.concatenate([np.arange(0, 4).reshape(1, 4), np.arange(10, 18).reshape(2, 4)]).astype(np.int32)
    np.testing.assert_array_equal(ret[0], want)
    np.testing.assert_array_equal(ret[1], want)


# ---- select="kv_head": per KV-head-group decisions, no collective -------------

def _kvh_worker(rank, world, port, q_all, k_all, v_all, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_09086_b200.sharding import gather_results

        G = HQ // HKV
        kvs, qs = shard_heads(HKV, G, world, rank)
        hk = kvs.stop - kvs.start
        cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.05)
        # this rank's groups as pseudo-streams (KvHeadEngine's layout: unit = s*hk + local group)
        orc = StreamOracle(S * hk, L, G, 1, D, cfg, window=W)

        def forbidden(*a, **k):
            raise AssertionError("kv_head selection must not communicate on the hot path")

        real = dist.all_reduce, dist.all_gather
        dist.all_reduce = dist.all_gather = forbidden
        decisions = []
        try:
            for t in range(T):
                q = q_all[t][:, :, qs].reshape(L, S * hk, G, D)
                k = k_all[t][:, :, kvs].reshape(L, S * hk, 1, D)
                v = v_all[t][:, :, kvs].reshape(L, S * hk, 1, D)
                orc.step(q, k, v)
                if (t + 1) % E == 0:
                    per = np.full((S * hk, L, l + r), -1, np.int64)
                    for u in range(S * hk):
                        for ly in range(L):
                            ks = orc.decide(u, ly).kept
                            per[u, ly, : ks.size] = ks
                            orc.apply(u, ly, ks)
                    decisions.append(per.reshape(S, hk, L, l + r))
        finally:
            dist.all_reduce, dist.all_gather = real
        # results leave through the one collective outside the hot path
        ret[rank] = [gather_results(torch.from_numpy(d), dim=1).numpy() for d in decisions]
    finally:
        dist.destroy_process_group()


def test_kv_head_selection_sharded_without_collectives():
    """World-size-2 gloo: each rank decides for its own KV-head groups only
    (no collective until the result gather); the gathered decisions equal the
    reference pipeline run per group on one process."""
    rng = np.random.default_rng(78)
    q_all = rng.standard_normal((T, L, S, HQ, D)).astype(F32)
    k_all = rng.standard_normal((T, L, S, HKV, D)).astype(F32)
    v_all = rng.standard_normal((T, L, S, HKV, D)).astype(F32)
    k_all[rng.random((T, L, S)) < 0.05] *= F32(4)
    mgr = tmp.Manager()
    ret = mgr.dict()
    port = 27500 + int(rng.integers(0, 2000))
    tmp.spawn(_kvh_worker, args=(2, port, q_all, k_all, v_all, ret), nprocs=2, join=True)
    d0, d1 = ret[0], ret[1]
    assert len(d0) == len(d1) == T // E
    G = HQ // HKV
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=0.05)
    orc = StreamOracle(S * HKV, L, G, 1, D, cfg, window=W)
    ei = 0
    for t in range(T):
        orc.step(q_all[t].reshape(L, S * HKV, G, D), k_all[t].reshape(L, S * HKV, 1, D),
                 v_all[t].reshape(L, S * HKV, 1, D))
        if (t + 1) % E == 0:
            for s in range(S):
                for g in range(HKV):
                    for ly in range(L):
                        u = s * HKV + g
                        want = orc.decide(u, ly).kept
                        np.testing.assert_array_equal(d0[ei][s, g, ly, : want.size], want)
                        np.testing.assert_array_equal(d1[ei][s, g, ly, : want.size], want)
                        orc.apply(u, ly, want)
            ei += 1
