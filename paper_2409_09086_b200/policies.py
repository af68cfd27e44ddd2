"""Drop-in for ``streamkv.policies`` (reference policies.py:28-265) on the GPU.

Same names, argument order, return types and ``ValueError`` domain errors.
The decision functions run the CUDA kernels of libstreamkv_b200.so:
``window_mean_scores`` / ``inf_mllm_decide`` the K2 score+bias+radix-select
kernel, ``top_k_indices`` its block radix top-k.  Inputs may be NumPy arrays /
lists (results come back as NumPy, like the reference) or CUDA tensors
(results stay on the device).  The Session's comparison baselines (sliding
window, sink+recent, heavy hitter; policies.py:204-256) run on the same select
kernel (``skv_policy_decide``) and a device accumulate kernel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List

import numpy as np
import torch

from . import _lib
from ._lib import check

F32 = np.float32

HEAD_AGG_MEAN = "mean"
HEAD_AGG_MAX = "max"


def _sh():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def _to_dev_f32(x):
    """(tensor on cuda f32, came_from_host)"""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return x.to(torch.float32).contiguous(), False
        return x.to(torch.float32).contiguous().cuda(), True
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=F32))).cuda(), True


def _out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


@dataclass
class PolicyConfig:
    """policies.py:28-59."""

    recent_len: int = 32
    relevant_budget: int = 2016
    bias: float = 0.1
    sink_count: int = 4
    head_agg: str = HEAD_AGG_MEAN

    def __post_init__(self):
        if self.recent_len < 1:
            raise ValueError("recent_len must be >= 1")
        if self.relevant_budget < 0:
            raise ValueError("relevant_budget must be >= 0")
        if self.bias < 0:
            raise ValueError("bias must be >= 0")
        if self.sink_count < 0:
            raise ValueError("sink_count must be >= 0")
        if self.head_agg not in (HEAD_AGG_MEAN, HEAD_AGG_MAX):
            raise ValueError(f"unknown head_agg {self.head_agg!r}")

    @property
    def budget(self) -> int:
        return self.recent_len + self.relevant_budget


@dataclass(frozen=True)
class EvictionDecision:
    """policies.py:62-84 (int64 index sets)."""

    relevant: object
    recent: object
    kept: object

    @staticmethod
    def from_sets(relevant, recent) -> "EvictionDecision":
        rel = np.asarray(sorted(set(int(i) for i in relevant)), dtype=np.int64)
        rec = np.asarray(sorted(set(int(i) for i in recent)), dtype=np.int64)
        return EvictionDecision(relevant=rel, recent=rec, kept=np.union1d(rel, rec).astype(np.int64))

    @staticmethod
    def keep_all(n: int, recent_len: int) -> "EvictionDecision":
        k = min(recent_len, n)
        return EvictionDecision(
            relevant=np.arange(0, n - k, dtype=np.int64),
            recent=np.arange(n - k, n, dtype=np.int64),
            kept=np.arange(n, dtype=np.int64),
        )


class AttentionWindow:
    """Rolling buffer of the last ``capacity`` rows (policies.py:87-127).

    The rows live in one device buffer [capacity][width] (width grows with the
    longest row) used as a ring, with their lengths: a push is one row copy,
    ``remap`` one gather of every row through the kept set (row i keeps its
    first #{kept < len_i} entries), and the policy kernels read the buffer
    oldest-first."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("window capacity must be >= 1")
        self.capacity = capacity
        self._buf = None        # [capacity][width] f32 device ring
        self._lens = []         # lengths, oldest first
        self._head = 0          # ring slot of the oldest row
        self._host = True

    def __len__(self) -> int:
        return len(self._lens)

    def _slot(self, i: int) -> int:
        return (self._head + i) % self.capacity

    @property
    def rows(self):
        out = [self._buf[self._slot(i), :n] for i, n in enumerate(self._lens)]
        return [r.cpu().numpy() for r in out] if self._host else [r.clone() for r in out]

    def push(self, row) -> None:
        r, host = _to_dev_f32(row)
        if r.ndim != 1 or r.numel() == 0:
            raise ValueError("row must be a non-empty vector")
        n = r.numel()
        if self._lens and n < self._lens[-1]:
            raise ValueError("row column count may not shrink between evictions")
        self._host = host
        if self._buf is None or self._buf.shape[1] < n:
            grown = torch.zeros((self.capacity, max(n, 2 * (self._buf.shape[1] if self._buf is not None else 0))),
                                dtype=torch.float32, device="cuda")
            if self._buf is not None:
                grown[:, : self._buf.shape[1]] = self._buf
            self._buf = grown
        if len(self._lens) == self.capacity:  # drop the oldest
            self._head = (self._head + 1) % self.capacity
            self._lens.pop(0)
        self._buf[self._slot(len(self._lens)), :n] = r
        self._lens.append(n)

    def remap(self, kept) -> None:
        if not self._lens:
            return
        idx = torch.as_tensor(np.asarray(kept, dtype=np.int64) if not isinstance(kept, torch.Tensor) else kept)
        idx = idx.to(device="cuda", dtype=torch.int64).reshape(-1)
        kh = idx.cpu().numpy()
        new_lens = [int(np.searchsorted(kh, n)) for n in self._lens]  # #{kept < len}, kept ascending
        width = self._buf.shape[1]
        gathered = self._buf.index_select(1, idx.clamp(max=width - 1))
        self._buf = torch.zeros_like(self._buf)
        self._buf[:, : gathered.shape[1]] = gathered
        self._lens = new_lens

    def clear(self) -> None:
        self._lens = []
        self._head = 0

    def _packed(self, n: int):
        """Oldest-first [m][width] view (one copy when the ring has wrapped) + lengths."""
        m = len(self._lens)
        if self._buf.shape[1] < n:
            self._buf = torch.nn.functional.pad(self._buf, (0, n - self._buf.shape[1]))
        order = [self._slot(i) for i in range(m)]
        if order == list(range(m)):
            buf = self._buf[:m]
        else:
            buf = self._buf.index_select(0, torch.tensor(order, dtype=torch.int64, device="cuda"))
        lens = torch.tensor(self._lens, dtype=torch.int32, device="cuda")
        return buf.contiguous(), lens, self._buf.shape[1]


def window_mean_scores(window: AttentionWindow, n: int, l: int):
    """policies.py:130-147 on device (bit-exact float32 order)."""
    if len(window) == 0:
        raise ValueError("attention window is empty")
    if n <= l:
        raise ValueError(f"no scorable columns: n={n} <= l={l}")
    buf, lens, width = window._packed(n)
    out = torch.empty(n - l, dtype=torch.float32, device="cuda")
    check(_lib.load().skv_window_scores(_p(buf), width, _p(lens), len(window), n, l, 0.0, 0, _p(out), _sh()))
    return _out(out, window._host)


def bias_vector(n: int, l: int, b: float):
    """policies.py:150-162: d = f32(b)/f32(n-l); bias[c] = (-d)*f32(n-l-1-c)."""
    if n <= l:
        raise ValueError(f"no scorable columns: n={n} <= l={l}")
    if b < 0:
        raise ValueError("bias must be >= 0")
    _lib.require_cuda()
    out = torch.empty(n - l, dtype=torch.float32, device="cuda")
    check(_lib.load().skv_bias_vector(n, l, ctypes.c_float(F32(b)), _p(out), _sh()))
    return out.cpu().numpy()


def top_k_indices(scores, k: int):
    """policies.py:165-181 on device: ascending indices, ties toward the larger index."""
    if k < 0:
        raise ValueError("k must be >= 0")
    s, host = _to_dev_f32(scores)
    s = s.reshape(-1)
    n = s.numel()
    m = min(k, n)
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    if m > 0:
        check(_lib.load().skv_top_k(_p(s), n, k, _p(out), _sh()))
    return _out(out, host)


def inf_mllm_decide(window: AttentionWindow, n: int, cfg: PolicyConfig) -> EvictionDecision:
    """policies.py:184-201 on device (K2: scores, bias, radix top-r, recent merge)."""
    if len(window) == 0:
        raise ValueError("attention window is empty")
    l, r = cfg.recent_len, cfg.relevant_budget
    if n <= r + l:
        return EvictionDecision.keep_all(n, l)
    buf, lens, width = window._packed(n)
    kept = torch.empty(r + l, dtype=torch.int64, device="cuda")
    scores = torch.empty(n - l, dtype=torch.float32, device="cuda")
    check(_lib.load().skv_decide(_p(buf), width, _p(lens), len(window), n, l, r, float(cfg.bias), _p(kept),
                                 _p(scores), _sh()))
    host = window._host
    kept_o = _out(kept, host)
    return EvictionDecision(relevant=kept_o[:r], recent=kept_o[r:], kept=kept_o)


_POLICY_WINDOW, _POLICY_SINK_RECENT, _POLICY_HEAVY_HITTER = 1, 2, 3


def _policy_decide(policy: int, acc, n: int, recent_len: int, relevant_budget: int, sink: int, host: bool):
    kept = torch.empty(max(1, min(n, recent_len + relevant_budget)), dtype=torch.int64, device="cuda")
    scores = torch.empty(max(1, n), dtype=torch.float32, device="cuda") if acc is not None else None
    m = check(_lib.load().skv_policy_decide(policy, _p(acc) if acc is not None else None, n, recent_len,
                                            relevant_budget, sink, _p(kept), _p(scores) if scores is not None else None,
                                            _sh()))
    return _out(kept[:m], host)


def sliding_window_decide(n: int, budget: int) -> EvictionDecision:
    """policies.py:204-213 on device: keep only the last ``budget`` positions."""
    if budget < 1:
        raise ValueError("budget must be >= 1")
    recent = _policy_decide(_POLICY_WINDOW, None, n, budget, 0, 0, True)
    return EvictionDecision(relevant=np.empty(0, dtype=np.int64), recent=recent, kept=recent)


def sink_recent_decide(n: int, s: int, budget: int) -> EvictionDecision:
    """policies.py:216-231 on device: the first ``s`` sinks plus the last ``budget - s``."""
    if not budget > s >= 0:
        raise ValueError("require budget > sink_count >= 0")
    if n <= budget:
        return EvictionDecision.keep_all(n, min(budget - s, n))
    kept = _policy_decide(_POLICY_SINK_RECENT, None, n, budget - s, s, s, True)
    return EvictionDecision(relevant=kept[:s], recent=kept[s:], kept=kept)


def heavy_hitter_accumulate(acc, new_row):
    """policies.py:234-243 on device: ``new_row`` plus the (shorter) running accumulator."""
    a, host_a = _to_dev_f32(acc)
    row, host = _to_dev_f32(new_row)
    a, row = a.reshape(-1), row.reshape(-1)
    if a.numel() > row.numel():
        raise ValueError("accumulator longer than the new row")
    out = torch.empty_like(row)
    check(_lib.load().skv_hh_accumulate(_p(a), a.numel(), _p(row), row.numel(), _p(out), _sh()))
    return _out(out, host)


def heavy_hitter_decide(acc, n: int, r: int, l: int) -> EvictionDecision:
    """policies.py:246-256 on device: the ``r`` largest accumulated masses of the
    first ``n - l`` columns (ties to the newer) plus the last ``l``."""
    a, host = _to_dev_f32(acc)
    a = a.reshape(-1)
    if a.numel() != n:
        raise ValueError(f"accumulator length {a.numel()} != n={n}")
    if n <= r + l:
        return EvictionDecision.keep_all(n, l)
    kept = _policy_decide(_POLICY_HEAVY_HITTER, a, n, l, r, 0, host)
    return EvictionDecision(relevant=kept[:r], recent=kept[r:], kept=kept)


def aggregate_heads(per_head, how: str):
    """policies.py:259-265: sequential float32 head sum / H (or max) on device."""
    if how not in (HEAD_AGG_MEAN, HEAD_AGG_MAX):
        raise ValueError(f"unknown head aggregation {how!r}")
    p, host = _to_dev_f32(per_head)
    if p.ndim != 2 or p.shape[0] == 0 or p.shape[1] == 0:
        raise ValueError("per_head must be a non-empty (heads, n) block")
    p = p.contiguous()
    out = torch.empty(p.shape[1], dtype=torch.float32, device="cuda")
    check(_lib.load().skv_aggregate_heads(_p(p), p.shape[0], p.shape[1], 1 if how == HEAD_AGG_MAX else 0, _p(out),
                                          _sh()))
    return _out(out, host)
