"""Batched streaming-decode engine over the C ABI (the B200 hot path).

``StreamEngine`` holds S independent streams (sessions) x L layers of a
size-constrained KV cache on one GPU and runs, through libstreamkv_b200.so:

* ``decode_layer`` / ``decode_step``: per layer, append the token's k/v, attend
  over the cache (including the new token), aggregate the per-head
  probabilities and push the row into the relevance window -- the hot body of
  ``Session.decode_step`` (reference engine.py:264-273);
* ``evict``: Algorithm 1 (window mean + attention bias + top-r + recent l) and
  in-place compaction of K/V, token metadata and the window rows --
  ``Session._evict_layer`` (engine.py:310-337) for every stream and layer;
* ``run_period``: E decode steps followed by one eviction, the eviction cadence
  of ``Session.start_round`` with an E-token prompt (engine.py:344-360).

Tensors are torch CUDA tensors; q/k/v use the engine dtype, outputs float32.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import SkvConfig, check


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(stream: Optional[torch.cuda.Stream] = None):
    if stream is None and _raw_stream is not None:  # (no Stream object per call: host steps are latency-bound)
        return _raw_stream(torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@dataclass(frozen=True)
class EngineConfig:
    streams: int
    layers: int
    heads_q: int
    heads_kv: int
    head_dim: int
    recent_len: int
    relevant_budget: int
    bias: float
    window: int
    capacity: int
    dtype: torch.dtype = torch.bfloat16
    head_agg: str = "mean"
    heads_q_total: int = 0  # head-sharded engines: query heads of all shards (0: heads_q)
    # Session policy switch (engine.py:296-307): "inf_mllm" (the hot path),
    # "window", "sink_recent", "heavy_hitter" or "none"
    policy: str = "inf_mllm"
    sink_count: int = 4
    # rotary positions (None: q/k arrive rotated, as in the BASELINE configs;
    # "cache_relative" / "original": PositionMode, cache.py:24-34)
    rope: Optional[str] = None
    rope_base: float = 10000.0

    @property
    def budget(self) -> int:
        return self.recent_len + self.relevant_budget


class StreamEngine:
    """S lock-stepped streams x L layers of the Inf-MLLM decode+evict path."""

    def __init__(self, cfg: EngineConfig):
        _lib.require_cuda()
        if cfg.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("dtype must be torch.float32 or torch.bfloat16")
        if cfg.head_agg not in ("mean", "max"):
            raise ValueError(f"unknown head_agg {cfg.head_agg!r}")
        if cfg.policy not in _lib.POLICIES:
            raise ValueError(f"unknown policy {cfg.policy!r}")
        if cfg.rope not in _lib.ROPE_MODES:
            raise ValueError(f"unknown rope mode {cfg.rope!r}")
        self.cfg = cfg
        self.lib = _lib.load()
        c = SkvConfig(
            streams=cfg.streams,
            layers=cfg.layers,
            heads_q=cfg.heads_q,
            heads_kv=cfg.heads_kv,
            head_dim=cfg.head_dim,
            dtype=_lib.DTYPE_BF16 if cfg.dtype == torch.bfloat16 else _lib.DTYPE_F32,
            recent_len=cfg.recent_len,
            relevant_budget=cfg.relevant_budget,
            bias=cfg.bias,
            window=cfg.window,
            capacity=cfg.capacity,
            head_agg=_lib.AGG_MAX if cfg.head_agg == "max" else _lib.AGG_MEAN,
            heads_q_total=cfg.heads_q_total,
            policy=_lib.POLICIES[cfg.policy],
            sink_count=cfg.sink_count,
            rope_mode=_lib.ROPE_MODES[cfg.rope],
            rope_base=cfg.rope_base,
        )
        handle = ctypes.c_void_p()
        torch.cuda.init()
        check(self.lib.skv_create(ctypes.byref(c), ctypes.byref(handle)))
        self._h = handle
        self.cap = (cfg.capacity + 31) // 32 * 32
        self.elt = 2 if cfg.dtype == torch.bfloat16 else 4

    # ---------------------------------------------------------------- life --
    def close(self):
        if getattr(self, "_h", None):
            self.lib.skv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(self.lib.skv_device_bytes(self._h))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.skv_kernel_launches(self._h))

    @property
    def last_decode_kernel(self) -> str:
        """The kernel the last decode launch ran (decode_tcd_kernel, decode_tc_cluster_kernel, ...)."""
        return self.lib.skv_last_decode_kernel(self._h).decode()

    # -------------------------------------------------------------- decode --
    def _check_io(self, q, k, v, out, lead):
        c = self.cfg
        for name, t, heads in (("q", q, c.heads_q), ("k", k, c.heads_kv), ("v", v, c.heads_kv)):
            want = (*lead, heads, c.head_dim)
            if tuple(t.shape) != want:
                raise ValueError(f"{name} shape {tuple(t.shape)} != {want}")
            if t.dtype != c.dtype or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CUDA {c.dtype} tensor")
        want = (*lead, c.heads_q, c.head_dim)
        if tuple(out.shape) != want or out.dtype != torch.float32 or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous float32 CUDA tensor of shape {want}")

    def decode_layer(self, layer: int, q, k, v, out=None, positions=None, record: bool = True):
        """q (S,Hq,D), k/v (S,Hkv,D) -> out (S,Hq,D) float32."""
        c = self.cfg
        if out is None:
            out = torch.empty((c.streams, c.heads_q, c.head_dim), dtype=torch.float32, device=q.device)
        self._check_io(q, k, v, out, (c.streams,))
        pos = None
        if positions is not None:
            arr = np.ascontiguousarray(np.asarray(positions, dtype=np.int64).reshape(c.streams))
            pos = arr.ctypes.data_as(ctypes.c_void_p)
        check(self.lib.skv_decode_layer(self._h, layer, _ptr(q), _ptr(k), _ptr(v), pos, _ptr(out),
                                        int(bool(record)), _stream_handle()))
        return out

    def decode_step(self, q, k, v, out=None, record: bool = True):
        """All layers of one token: q (L,S,Hq,D), k/v (L,S,Hkv,D) -> out (L,S,Hq,D)."""
        c = self.cfg
        if out is None:
            out = torch.empty((c.layers, c.streams, c.heads_q, c.head_dim), dtype=torch.float32,
                              device=q.device)
        self._check_io(q, k, v, out, (c.layers, c.streams))
        check(self.lib.skv_decode_step(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), int(bool(record)),
                                       _stream_handle()))
        return out

    def prefill_chunk(self, layer: int, q, k, v, out=None, modality: int = 0):
        """A C-token chunk of one layer on the tensor cores: q (S,C,Hq,D), k/v
        (S,C,Hkv,D) bf16 -> out (S,C,Hq,D) f32; equivalent to C decode_layer calls
        (the last min(W, C) rows enter the window)."""
        c = self.cfg
        S, C = q.shape[0], q.shape[1]
        if out is None:
            out = torch.empty((S, C, c.heads_q, c.head_dim), dtype=torch.float32, device=q.device)
        for name, t, heads in (("q", q, c.heads_q), ("k", k, c.heads_kv), ("v", v, c.heads_kv)):
            if tuple(t.shape) != (c.streams, C, heads, c.head_dim) or t.dtype != c.dtype or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous {c.dtype} tensor of shape {(c.streams, C, heads, c.head_dim)}")
        check(self.lib.skv_prefill_chunk(self._h, layer, _ptr(q), _ptr(k), _ptr(v), C, int(modality), _ptr(out),
                                         _stream_handle()))
        return out

    def decode_step_host(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
                         record: bool = True):
        """Same as decode_step with host (ideally pinned) tensors; synchronous.
        Work already enqueued on the current torch stream (evictions, prefill
        chunks) is ordered before it."""
        c = self.cfg
        shapes = self.__dict__.get("_host_shapes")
        if shapes is None:
            lead = (c.layers, c.streams)
            shapes = self._host_shapes = ((*lead, c.heads_q, c.head_dim), (*lead, c.heads_kv, c.head_dim))
        for name, t, shp in (("q", q, shapes[0]), ("k", k, shapes[1]), ("v", v, shapes[1])):
            if t.shape != shp or t.dtype != c.dtype or t.is_cuda:
                raise ValueError(f"{name} must be a host {c.dtype} tensor of shape {shp}")
        if out.is_cuda or out.dtype != torch.float32:
            raise ValueError("out must be a host float32 tensor")
        rc = self.lib.skv_decode_step_host(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                           1 if record else 0, _stream_handle())
        if rc < 0:
            check(rc)
        return out

    def host_speculation(self, enable: bool = True, timeout_us: int = 500):
        """Speculative host steps for shallow engines (<= 2 layers, no RoPE):
        each decode_step_host call also launches the next token behind a
        device-side doorbell gate, so the next call pays a PCIe round trip
        instead of launches plus a synchronisation.  Same kernels and results;
        any other engine call cancels the pending step.  While one is pending
        a device-wide synchronisation may wait up to ``timeout_us``."""
        check(self.lib.skv_host_speculate(self._h, 1 if enable else 0, int(timeout_us)))

    def host_speculation_stats(self):
        """(steps served from a pending launch, pending steps cancelled or expired)."""
        h, m = ctypes.c_int64(0), ctypes.c_int64(0)
        check(self.lib.skv_host_speculate_stats(self._h, ctypes.byref(h), ctypes.byref(m)))
        return h.value, m.value

    # --------------------------------------------------------------- evict --
    def evict(self, layer: int = -1, kept: Optional[torch.Tensor] = None):
        """Algorithm 1 + compaction for every stream of ``layer`` (-1: all layers).

        ``kept`` (optional, int32 CUDA, (S, L', r+l)) receives the kept sets;
        rows of a keep-all decision hold 0..n-1 padded with -1."""
        check(self.lib.skv_evict(self._h, int(layer), _ptr(kept), _stream_handle()))
        return kept

    def evict_scores(self, layer: int = -1) -> torch.Tensor:
        """This shard's unbiased window-mean scores, (S, L', capacity) f32 (first n-l valid).

        The tensor is the engine's persistent buffer for this shape: the next
        call overwrites it."""
        nl = self.cfg.layers if layer < 0 else 1
        # one persistent buffer per shape: a sharded period is captured in a CUDA
        # graph, whose replays must write memory that outlives the capture
        bufs = self.__dict__.setdefault("_score_bufs", {})
        scores = bufs.get(nl)
        if scores is None:
            scores = bufs[nl] = torch.empty((self.cfg.streams, nl, self.cap), dtype=torch.float32, device="cuda")
        scores.zero_()
        check(self.lib.skv_evict_scores(self._h, int(layer), _ptr(scores), _stream_handle()))
        return scores

    def evict_apply(self, scores: torch.Tensor, layer: int = -1, kept: Optional[torch.Tensor] = None):
        """Bias + top-r + recent merge + compaction from (reduced) window-mean scores."""
        check(self.lib.skv_evict_apply(self._h, int(layer), _ptr(scores.contiguous()), _ptr(kept),
                                       _stream_handle()))
        return kept

    def run_period(self, q, k, v, out, steps: int, evict: bool = True):
        """``steps`` decode steps (inputs indexed [t] along dim 0) + one eviction.

        Only the last ``window`` steps record window rows: older rows leave the
        window before the eviction reads it, so the decisions are identical to
        recording every step (AttentionWindow.push drops the oldest row,
        policies.py:113-115)."""
        first_rec = steps - self.cfg.window
        for t in range(steps):
            self.decode_step(q[t], k[t], v[t], out, record=t >= first_rec)
        if evict:
            self.evict(-1)
        return out

    # --------------------------------------------------------------- state --
    def sync(self):
        """Synchronise the current stream and raise the engine's sticky device
        errors (ValueError when a chunked prefill saturated |v| >= 65504)."""
        check(self.lib.skv_sync(self._h, _stream_handle()))

    def state_dump(self, stream: int, layer: int) -> dict:
        """Host copy of one (stream, layer) state (KvCache.debug_snapshot,
        cache.py:172-180, with the tensors): keys/values (Hkv, n, D) float32,
        positions, modalities, round ids, window rows (oldest first)."""
        n, m = ctypes.c_int(), ctypes.c_int()
        check(self.lib.skv_state_dump(self._h, stream, layer, ctypes.byref(n), ctypes.byref(m), *([None] * 7)))
        n, m = n.value, m.value
        c = self.cfg
        kt = torch.empty((c.heads_kv, n, c.head_dim), dtype=c.dtype)
        vt = torch.empty_like(kt)
        pos = np.zeros(n, np.int64)
        mod = np.zeros(n, np.int8)
        rnd = np.zeros(n, np.int32)
        rows = np.zeros((max(m, 1), max(n, 1)), np.float32)
        lens = np.zeros(max(m, 1), np.int32)
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        check(self.lib.skv_state_dump(self._h, stream, layer, ctypes.byref(ctypes.c_int()),
                                      ctypes.byref(ctypes.c_int()), _ptr(kt), _ptr(vt), P(pos), P(mod), P(rnd),
                                      P(rows), P(lens)))
        return {"n": n, "keys": kt.float().numpy(), "values": vt.float().numpy(), "original_positions": pos,
                "modalities": mod, "round_ids": rnd, "rows": [rows[i, : lens[i]].copy() for i in range(m)]}

    def length(self, stream: int = 0, layer: int = 0) -> int:
        return check(self.lib.skv_length(self._h, stream, layer))

    def slot_map(self, stream: int, layer: int) -> Optional[torch.Tensor]:
        """int32 (n,) view: logical slot -> physical row (None: identity)."""
        pp = ctypes.c_void_p()
        check(self.lib.skv_slot_map(self._h, stream, layer, ctypes.byref(pp)))
        if not pp.value:
            return None
        n = self.length(stream, layer)
        return _wrap(pp.value, (self.cap,), torch.int32)[:n]

    def kv(self, stream: int, layer: int):
        """Keys/values (Hkv, n, D) of (stream, layer) in logical (cache) order
        -- KvCache.keys()/values().  Without a slot map (or before the first
        eviction) these are views of the store; otherwise gathered copies."""
        kt, vt = self.kv_full(stream, layer)
        n = self.length(stream, layer)
        perm = self.slot_map(stream, layer)
        if perm is None:
            return kt[:, :n], vt[:, :n]
        idx = perm.long()
        if bool((idx == torch.arange(n, device=idx.device)).all()):
            return kt[:, :n], vt[:, :n]
        return kt.index_select(1, idx), vt.index_select(1, idx)

    def kv_full(self, stream: int, layer: int):
        """Views (Hkv, capacity, D) of the PHYSICAL key/value storage."""
        kp, vp = ctypes.c_void_p(), ctypes.c_void_p()
        check(self.lib.skv_kv_view(self._h, stream, layer, ctypes.byref(kp), ctypes.byref(vp)))
        c = self.cfg
        full = (c.heads_kv, self.cap, c.head_dim)
        return _wrap(kp.value, full, c.dtype), _wrap(vp.value, full, c.dtype)

    def moved_rows(self) -> Optional[np.ndarray]:
        """(S, L) rows moved by the last eviction (None: dense compaction)."""
        out = np.zeros((self.cfg.streams, self.cfg.layers), np.int32)
        rc = self.lib.skv_moved_rows(self._h, out.ctypes.data_as(ctypes.c_void_p))
        if rc == _lib.SKV_ESTATE:
            return None
        check(rc)
        return out

    def positions(self, stream: int, layer: int) -> np.ndarray:
        out = np.zeros(self.cap, dtype=np.int64)
        n = check(self.lib.skv_positions(self._h, stream, layer, out.ctypes.data_as(ctypes.c_void_p), self.cap))
        return out[:n]

    def window_rows(self, stream: int, layer: int):
        rows = np.zeros((self.cfg.window, self.cap), dtype=np.float32)
        lens = np.zeros(self.cfg.window, dtype=np.int32)
        m = check(self.lib.skv_window_rows(self._h, stream, layer, rows.ctypes.data_as(ctypes.c_void_p),
                                           lens.ctypes.data_as(ctypes.c_void_p)))
        return [rows[i, : lens[i]].copy() for i in range(m)]

    def last_scores(self, stream: int, layer: int, cols: int) -> np.ndarray:
        out = np.zeros(self.cap, dtype=np.float32)
        check(self.lib.skv_last_scores(self._h, stream, layer, out.ctypes.data_as(ctypes.c_void_p), self.cap))
        return out[:cols].copy()

    def inject(self, stream: int, layer: int, keys: np.ndarray, values: np.ndarray, positions: np.ndarray,
               rows=None):
        """State injection for parity: keys/values (Hkv, n, D) in engine dtype
        (float32 arrays are rounded to bf16 for a bf16 engine), positions (n,),
        rows: list of window rows (oldest first)."""
        c = self.cfg
        n = keys.shape[1]
        kt = torch.as_tensor(np.ascontiguousarray(keys, dtype=np.float32)).to(c.dtype).contiguous()
        vt = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float32)).to(c.dtype).contiguous()
        pos = np.ascontiguousarray(positions, dtype=np.int64)
        rows = rows or []
        m = len(rows)
        rbuf = np.zeros((max(m, 1), max(n, 1)), dtype=np.float32)
        lens = np.zeros(max(m, 1), dtype=np.int32)
        for i, r in enumerate(rows):
            rbuf[i, : r.size] = r
            lens[i] = r.size
        check(self.lib.skv_state_inject(self._h, stream, layer, n, _ptr(kt), _ptr(vt),
                                        pos.ctypes.data_as(ctypes.c_void_p), m,
                                        rbuf.ctypes.data_as(ctypes.c_void_p),
                                        lens.ctypes.data_as(ctypes.c_void_p)))

    def timing(self, enable: bool = True):
        """Record per-decode-launch device timestamps (first CTA start, last CTA end)."""
        check(self.lib.skv_timing(self._h, int(bool(enable))))

    def timing_read(self) -> np.ndarray:
        """(count, 2) uint64 ns: [start, end] of each decode launch since enabling."""
        buf = np.zeros((8192, 2), dtype=np.uint64)
        n = check(self.lib.skv_timing_read(self._h, buf.ctypes.data_as(ctypes.c_void_p), 8192))
        return buf[:n].copy()

    # -------------------------------------------------------------- graphs --
    def capture_begin(self):
        check(self.lib.skv_capture_begin(self._h, _stream_handle()))

    def capture_end(self):
        check(self.lib.skv_capture_end(self._h, _stream_handle()))

    def replay(self):
        check(self.lib.skv_graph_launch(self._h, _stream_handle()))


def _wrap(ptr: int, shape, dtype: torch.dtype) -> torch.Tensor:
    """Zero-copy torch view of engine-owned device memory."""
    typestr = {torch.float32: "<f4", torch.bfloat16: "<i2", torch.int32: "<i4"}[dtype]
    elt = 2 if dtype == torch.bfloat16 else 4

    class _Iface:
        __cuda_array_interface__ = {
            "shape": tuple(shape),
            "typestr": typestr,
            "data": (ptr, False),
            "version": 2,
            "strides": None,
        }

    t = torch.as_tensor(_Iface(), device="cuda")
    if dtype == torch.bfloat16:
        t = t.view(torch.bfloat16)
    assert t.element_size() == elt
    return t
