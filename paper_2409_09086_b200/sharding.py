"""KV-head sharding of one stream across GPUs (BASELINE config 3).

Each rank owns a contiguous block of KV heads and their query heads and runs a
``StreamEngine`` with ``heads_q_total`` set to the model's query-head count, so
its window rows are its heads' probability sums divided by the total head
count.  The reference selects per layer over the head mean of *all* heads
(policies.py:259-263 via engine.py:272), so at an eviction the
ranks sum their window-mean scores -- one all-reduce of (n - l) floats per
(stream, layer), the only collective of the path -- and every rank then applies
the same bias, top-r and compaction (``select="layer"``, the parity mode).

``select="kv_head"`` is the north star's collective-free variant: every rank
decides from its own heads only (each rank's engine is built with
``heads_q_total=0``).  Its decisions are *not* the reference semantics.
"""

from __future__ import annotations

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
