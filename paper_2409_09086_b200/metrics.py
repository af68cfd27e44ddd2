"""Per-round policy quality measurements (reference metrics.py:34-90) on the
device: retained attention mass, top-k overlap with the full-cache oracle,
planted-saddle recall.  Index-set intersections of the
(small) kept / top-r sets and the final means are host arithmetic."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check
from .policies import _p, _sh, top_k_indices

F32 = np.float32


@dataclass
class MetricsRow:
    """metrics.py:34-43."""

    round_id: int
    policy: str
    retained_mass: Optional[float]
    topk_overlap: Optional[float]
    planted_recall: Optional[float]
    cache_len: int
    memory_bytes: int
    flops_per_token: int


def _dev_i64(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.int64).reshape(-1).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.int64)).reshape(-1)).cuda()


def _pack(rows: Sequence, width: int = 0):
    """Device rows -> [m][width] f32 buffer + int32 lengths."""
    rs = [r if isinstance(r, torch.Tensor) else torch.from_numpy(np.asarray(r, dtype=F32)) for r in rows]
    rs = [r.to(device="cuda", dtype=torch.float32).reshape(-1) for r in rs]
    width = max([width] + [r.numel() for r in rs])
    buf = torch.zeros((len(rs), max(1, width)), dtype=torch.float32, device="cuda")
    for i, r in enumerate(rs):
        buf[i, : r.numel()] = r
    lens = torch.tensor([r.numel() for r in rs], dtype=torch.int32, device="cuda")
    return buf, lens, max(1, width)


def retained_mass(oracle_rows: Sequence, kept) -> float:
    """metrics.py:46-62: mean over the rows of the f64 mass on ``kept``."""
    rows = list(oracle_rows)
    if not rows:
        raise ValueError("retained_mass needs at least one scoring row")
    buf, lens, width = _pack(rows)
    idx = _dev_i64(kept)
    out = torch.empty(len(rows), dtype=torch.float64, device="cuda")
    check(_lib.load().skv_masked_row_sums(_p(buf), width, _p(lens), len(rows), _p(idx) if idx.numel() else None,
                                          idx.numel(), _p(out), _sh()))
    total = 0.0
    for v in out.cpu().tolist():  # sequential f64, like the reference loop
        total += v
    return total / len(rows)


def topk_overlap(oracle_scores, relevant_ids, r: int) -> float:
    """metrics.py:65-73: |relevant ∩ oracle top-r| / r (device top-r)."""
    if r < 1:
        raise ValueError("r must be >= 1")
    top = top_k_indices(oracle_scores, r)
    top = top.cpu().numpy() if isinstance(top, torch.Tensor) else top
    rel = relevant_ids.cpu().numpy() if isinstance(relevant_ids, torch.Tensor) else np.asarray(relevant_ids)
    return len(set(int(i) for i in top) & set(int(i) for i in rel)) / r


def planted_recall(truth, kept) -> Optional[float]:
    """metrics.py:76-86 (None when nothing is planted)."""
    t = set(int(i) for i in (truth.cpu().numpy() if isinstance(truth, torch.Tensor) else np.asarray(truth)))
    if not t:
        return None
    k = set(int(i) for i in (kept.cpu().numpy() if isinstance(kept, torch.Tensor) else np.asarray(kept)))
    return len(t & k) / len(t)


def flops_per_token(cache_len: int, layers: int, heads: int, head_dim: int) -> int:
    """metrics.py:86-90: multiply-add proxy of one decode step."""
    if layers < 1 or heads < 1 or head_dim < 1 or cache_len < 0:
        raise ValueError("dimensions must be positive")
    return 4 * cache_len * head_dim * heads * layers


def window_oracle_scores(rows: Sequence, n: int, l: int):
    """The replay's full-cache oracle scores (replay.py:157-164): rows summed
    in order over the first n - l columns (shorter rows contribute their own
    columns), divided by the row count -- the K2 window-mean arithmetic."""
    buf, lens, width = _pack(rows, n)
    out = torch.empty(n - l, dtype=torch.float32, device="cuda")
    check(_lib.load().skv_window_scores(_p(buf), width, _p(lens), len(rows), n, l, ctypes.c_float(0.0), 0, _p(out),
                                        _sh()))
    return out
