"""KV-head sharding of one stream across GPUs (BASELINE config 3).

Each rank owns a contiguous block of KV heads and their query heads and runs a
``StreamEngine`` with ``heads_q_total`` set to the model's query-head count, so
its window rows are its heads' probability sums divided by the total head
count.  The reference selects per layer over the head mean of *all* heads
(policies.py:259-263 via engine.py:272), so at an eviction the
ranks sum their window-mean scores -- one all-reduce of (n - l) floats per
(stream, layer), the only collective of the path -- and every rank then applies
the same bias, top-r and compaction (``select="layer"``, the parity mode).

``select="kv_head"`` (``KvHeadEngine``) is the north star's collective-free
variant: every KV-head group -- one KV head and its G query heads -- keeps its
own window of G-head mean rows and its own Algorithm-1 decision, i.e. the
reference's ``inf_mllm_decide`` applied per group.  Groups
never exchange anything, so KV heads shard across GPUs with no collective.
Its decisions are *not* the reference's per-layer semantics and every report
that uses it says so.
"""

from __future__ import annotations

from dataclasses import replace
from typing import Optional

import torch
import torch.distributed as dist


def shard_heads(heads_kv: int, group_size: int, world: int, rank: int):
    """Contiguous KV-head block of ``rank`` and the matching query-head block."""
    if heads_kv % world:
        raise ValueError(f"{heads_kv} KV heads do not split over {world} ranks")
    per = heads_kv // world
    kv = slice(rank * per, (rank + 1) * per)
    q = slice(kv.start * group_size, kv.stop * group_size)
    return kv, q


def evict_head_sharded(engine, layer: int = -1, kept: Optional[torch.Tensor] = None, group=None):
    """Per-layer (reference) selection across KV-head shards.

    ``engine`` provides ``evict_scores(layer)`` and ``evict_apply(scores, layer,
    kept)`` (``StreamEngine``, or any object with the same contract)."""
    scores = engine.evict_scores(layer)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(scores, op=dist.ReduceOp.SUM, group=group)
    return engine.evict_apply(scores, layer, kept)


def gather_results(t: torch.Tensor, dim: int = 0, group=None) -> torch.Tensor:
    """The one collective outside the hot path (SURVEY 8e "collective for
    results"): every rank's block of per-stream outputs / kept indices,
    concatenated along ``dim`` in rank order (all ranks receive it).  Single
    process: ``t`` itself.  Shapes may differ along ``dim`` only."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    world = dist.get_world_size(group)
    sizes = torch.tensor([t.shape[dim]], dtype=torch.int64, device=t.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    cap = int(max(int(x.item()) for x in all_sizes))
    pad = list(t.shape)
    pad[dim] = cap
    buf = torch.zeros(pad, dtype=t.dtype, device=t.device)
    buf.narrow(dim, 0, t.shape[dim]).copy_(t)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p.narrow(dim, 0, int(n.item())) for p, n in zip(parts, all_sizes)], dim=dim)


class KvHeadEngine:
    """``select="kv_head"``: one selection unit per (stream, KV-head group).

    A KV-head group (KV head g and query heads g*G .. g*G+G-1) attends, scores
    and evicts exactly like an independent stream with one KV head and G query
    heads, so the groups run as the streams of an inner ``StreamEngine``
    (streams = S * Hkv, heads_kv = 1, heads_q = G).  Inputs and outputs keep
    the model's layout: q (L,S,Hq,D) and k/v (L,S,Hkv,D) are contiguous, so
    (L, S*Hkv, G, D) / (L, S*Hkv, 1, D) are free views of them.  The oracle is
    the reference pipeline run per group (``StreamOracle(S*Hkv, L, G, 1, ...)``)."""

    def __init__(self, cfg):
        from .engine import StreamEngine

        if cfg.heads_q_total not in (0, cfg.heads_q):
            raise ValueError("kv_head selection needs no cross-shard head total")
        self.cfg = cfg
        self.G = cfg.heads_q // cfg.heads_kv
        self.inner = StreamEngine(replace(cfg, streams=cfg.streams * cfg.heads_kv, heads_kv=1, heads_q=self.G,
                                          heads_q_total=0))

    def _views(self, q, k, v, out, lead):
        S, Hkv, G, D = self.cfg.streams, self.cfg.heads_kv, self.G, self.cfg.head_dim
        q2 = q.view(*lead, S * Hkv, G, D)
        k2 = k.view(*lead, S * Hkv, 1, D)
        v2 = v.view(*lead, S * Hkv, 1, D)
        o2 = None if out is None else out.view(*lead, S * Hkv, G, D)
        return q2, k2, v2, o2

    @property
    def last_decode_kernel(self) -> str:
        return self.inner.last_decode_kernel

    def decode_step(self, q, k, v, out=None, record: bool = True):
        c = self.cfg
        if out is None:
            out = torch.empty((c.layers, c.streams, c.heads_q, c.head_dim), dtype=torch.float32, device=q.device)
        q2, k2, v2, o2 = self._views(q, k, v, out, (c.layers,))
        self.inner.decode_step(q2, k2, v2, o2, record=record)
        return out

    def decode_layer(self, layer: int, q, k, v, out=None, record: bool = True):
        c = self.cfg
        if out is None:
            out = torch.empty((c.streams, c.heads_q, c.head_dim), dtype=torch.float32, device=q.device)
        q2, k2, v2, o2 = self._views(q, k, v, out, ())
        self.inner.decode_layer(layer, q2, k2, v2, o2, record=record)
        return out

    def decode_step_host(self, q, k, v, out, record: bool = True):
        """decode_step with host (pinned) tensors through the host-buffer C entry point."""
        q2, k2, v2, o2 = self._views(q, k, v, out, (self.cfg.layers,))
        self.inner.decode_step_host(q2, k2, v2, o2, record=record)
        return out

    def evict(self, layer: int = -1, kept: Optional[torch.Tensor] = None):
        """``kept`` (optional, int32, (S, Hkv, L', r+l)): each group's kept set."""
        c = self.cfg
        inner_kept = None if kept is None else kept.view(c.streams * c.heads_kv, *kept.shape[2:])
        self.inner.evict(layer, inner_kept)
        return kept

    def length(self, stream: int = 0, layer: int = 0, group: int = 0) -> int:
        return self.inner.length(stream * self.cfg.heads_kv + group, layer)

    def kv(self, stream: int, layer: int):
        """Keys/values (Hkv, n, D) in logical order (every group holds n tokens)."""
        parts = [self.inner.kv(stream * self.cfg.heads_kv + g, layer) for g in range(self.cfg.heads_kv)]
        return torch.cat([p[0] for p in parts]), torch.cat([p[1] for p in parts])

    def positions(self, stream: int, layer: int, group: int) -> "object":
        return self.inner.positions(stream * self.cfg.heads_kv + group, layer)

    @property
    def kernel_launches(self) -> int:
        return self.inner.kernel_launches

    def capture_begin(self):
        self.inner.capture_begin()

    def capture_end(self):
        self.inner.capture_end()

    def replay(self):
        self.inner.replay()

    def inject_group(self, stream: int, layer: int, group: int, keys, values, positions, rows=None):
        self.inner.inject(stream * self.cfg.heads_kv + group, layer, keys, values, positions, rows)
