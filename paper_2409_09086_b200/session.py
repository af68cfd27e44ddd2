"""Live-session quality metrics on the device: the reference ``Session``'s
oracle mode (``Session(oracle=True)``, /root/reference/pkg/src/streamkv/engine.py:142-151
shadow cache and rows, 275-284 shadow step, 310-331 per-eviction metrics,
344-380 per-round MetricsRow, 391-451 ``attention_equivalence_check``).

``OracleSession`` runs the compressed-cache ``StreamEngine`` next to a shadow
``StreamEngine`` that never evicts (the full cache), both fed the same q/k/v.
The shadow keeps the last ``recent_len`` head-aggregated rows over the full
cache; at every eviction the kept / relevant ids of the compressed cache are
scored against them on the device (``skv_round_metrics``): retained
attention mass and top-r overlap with the full-cache window-mean oracle, per
(stream, layer), averaged over layers into one ``MetricsRow`` per stream --
one D2H read per eviction, after all layers are launched.
"""

from __future__ import annotations

import ctypes
from dataclasses import replace
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import check
from .engine import EngineConfig, StreamEngine
from .metrics import MetricsRow, flops_per_token
from .tensorops import attend

F32 = np.float32


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


class OracleSession:
    """Compressed cache + never-evicted shadow cache with live metrics."""

    def __init__(self, cfg: EngineConfig, max_tokens: int):
        if cfg.rope is not None:
            raise ValueError("OracleSession compares caches of pre-rotated keys (rope=None)")
        if max_tokens <= cfg.budget:
            raise ValueError("max_tokens must exceed the KV budget")
        self.cfg = cfg
        self.engine = StreamEngine(cfg)
        # the shadow records every step into a ring of recent_len rows
        # (deque(maxlen=recent_len), engine.py:148-150) and is never evicted
        self.shadow = StreamEngine(replace(cfg, window=cfg.recent_len, capacity=max_tokens, policy="inf_mllm",
                                           heads_q_total=0))
        self.metrics_rows: List[List[MetricsRow]] = []   # per eviction: one row per stream
        self.layer_metrics: List[np.ndarray] = []        # per eviction: [S][L][2] (mass, overlap or nan)
        self.round_id = -1
        lib = _lib.load()
        self.lib = lib
        S, L = cfg.streams, cfg.layers
        self._mass = torch.zeros((S, L, cfg.recent_len), dtype=torch.float64, device="cuda")
        self._count = torch.zeros((S, L, 2), dtype=torch.int32, device="cuda")
        self._iota = torch.arange(max(cfg.budget, 1), dtype=torch.int64, device="cuda")
        self._scores = torch.zeros(max_tokens, dtype=torch.float32, device="cuda")
        self._top = torch.zeros(max(1, cfg.relevant_budget), dtype=torch.int32, device="cuda")

    # ------------------------------------------------------------------ steps
    def decode_step(self, q, k, v, out=None, record: bool = True):
        """All layers of one token on both caches (engine.py:250-289 + 275-284)."""
        out = self.engine.decode_step(q, k, v, out, record=record)
        self.shadow.decode_step(q, k, v, record=True)
        return out

    def prefill_chunk(self, layer: int, q, k, v, out=None, modality: int = 0):
        """A chunk of one layer on both caches.  The shadow's rows record only
        the chunk's last min(recent_len, C) queries -- all its ring keeps."""
        out = self.engine.prefill_chunk(layer, q, k, v, out, modality)
        self.shadow.prefill_chunk(layer, q, k, v, None, modality)
        return out

    def _relevant_count(self, n: int) -> int:
        c = self.cfg
        if c.policy == "window":
            return 0
        if c.policy == "sink_recent":
            return n - min(c.budget - c.sink_count, n) if n <= c.budget else min(c.sink_count, n)
        if c.policy in ("inf_mllm", "heavy_hitter") and n > c.budget:
            return c.relevant_budget
        return n - min(c.recent_len, n)

    def evict(self, kept: Optional[torch.Tensor] = None) -> List[MetricsRow]:
        """_evict_layer for every (stream, layer) + the oracle metrics
        (engine.py:310-337) and start_round's MetricsRow (360-378), per stream."""
        c = self.cfg
        S, L = c.streams, c.layers
        n_before = [[self.engine.length(s, layer) for layer in range(L)] for s in range(S)]
        self.engine.evict(-1, kept)
        self.round_id += 1
        sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        meta = []
        for s in range(S):
            for layer in range(L):
                m = self.engine.length(s, layer)
                rc = self._relevant_count(n_before[s][layer])
                pos = ctypes.c_void_p()
                check(self.lib.skv_positions_view(self.engine._h, s, layer, ctypes.byref(pos)))
                rows, lens = ctypes.c_void_p(), ctypes.c_void_p()
                head, count = ctypes.c_int(), ctypes.c_int()
                stride = check(self.lib.skv_window_view(self.shadow._h, s, layer, ctypes.byref(rows),
                                                        ctypes.byref(lens), ctypes.byref(head),
                                                        ctypes.byref(count)))
                W = c.recent_len
                slots = [(head.value - count.value + i) % W for i in range(count.value)]
                slot_t = torch.tensor(slots, dtype=torch.int64, device="cuda")
                lens_t = _lens_view(lens.value, W).index_select(0, slot_t).contiguous()
                off_t = (slot_t * stride).contiguous()
                ns = self.shadow.length(s, layer)
                check(self.lib.skv_round_metrics(_p(self._iota), m, rc, ctypes.c_void_p(pos.value),
                                                 ctypes.c_void_p(rows.value), _p(off_t), _p(lens_t), count.value,
                                                 ns, c.recent_len, c.relevant_budget, None, 0, _p(self._scores),
                                                 _p(self._top), _p(self._mass[s, layer]), _p(self._count[s, layer]),
                                                 sh))
                meta.append((s, layer, count.value, m, (slot_t, lens_t, off_t)))  # keep inputs alive until read
        mass = self._mass.cpu().numpy()
        cnt = self._count.cpu().numpy()
        per_layer = np.full((S, L, 2), np.nan)
        for s, layer, nrows, m, _ in meta:
            total = 0.0
            for v in mass[s, layer, :nrows]:
                total += float(v)
            per_layer[s, layer, 0] = total / nrows
            if cnt[s, layer, 0] >= 0:
                per_layer[s, layer, 1] = int(cnt[s, layer, 0]) / c.relevant_budget
        self.layer_metrics.append(per_layer)
        rows = []
        for s in range(S):
            n0 = self.engine.length(s, 0)
            ov = [x for x in per_layer[s, :, 1] if not np.isnan(x)]
            mem = 2 * sum(self.engine.length(s, layer) for layer in range(L)) * c.head_dim * c.heads_kv * 4
            rows.append(MetricsRow(round_id=self.round_id, policy=c.policy,
                                   retained_mass=float(np.mean(per_layer[s, :, 0])),
                                   topk_overlap=float(np.mean(ov)) if ov else None, planted_recall=None,
                                   cache_len=n0, memory_bytes=mem,
                                   flops_per_token=flops_per_token(n0, L, c.heads_q, c.head_dim)))
        self.metrics_rows.append(rows)
        return rows

    # ---------------------------------------------------------------- checks
    def attention_equivalence_check(self, stream: int, layer: int, q) -> float:
        """Max deviation between attention over the compressed cache and over
        the shadow cache restricted to the kept tokens (engine.py:391-451 with
        matching positions): probabilities and outputs, every head."""
        c = self.cfg
        G = c.heads_q // c.heads_kv
        qq = torch.as_tensor(q).to(device="cuda", dtype=torch.float32).reshape(c.heads_q, c.head_dim)
        ka, va = (t.float().repeat_interleave(G, 0).contiguous() for t in self.engine.kv(stream, layer))
        ids = torch.from_numpy(self.engine.positions(stream, layer)).cuda()
        ks, vs = self.shadow.kv(stream, layer)
        kb = ks.index_select(1, ids).float().repeat_interleave(G, 0).contiguous()
        vb = vs.index_select(1, ids).float().repeat_interleave(G, 0).contiguous()
        pa, oa = attend(ka, va, qq)
        pb, ob = attend(kb, vb, qq)
        return float(max((oa - ob).abs().max().item(), (pa - pb).abs().max().item()))


def _lens_view(ptr: int, n: int) -> torch.Tensor:
    from .engine import _wrap

    return _wrap(ptr, (n,), torch.int32)
