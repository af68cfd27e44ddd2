"""CPU oracle for the Inf-MLLM streaming-decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped path (``paper_2409_09086_b200``)
never imports anything under ``oracle/`` and fails loudly when its CUDA
library is missing.

It restates, in NumPy float32, the reference package ``streamkv``
(``/root/reference/pkg/src/streamkv``) for exactly the functions on the hot
path.  Every function cites the reference file:line it
follows.  The float32 operation sequence is kept identical to the reference
(same NumPy/BLAS calls on the same memory layout) so that, fed the same
inputs, the oracle reproduces the reference bit-for-bit; this is *pinned* by
``tests/test_oracle_golden.py`` against fixtures produced by running the
reference itself (``tests/golden/make_golden.py``).

Two things the reference does not have are expressed with reference
arithmetic, exactly as SURVEY.md 8a "divergences" prescribes:

* GQA: key/value heads are repeated ``Hq // Hkv`` times before the per-head
  attention loop (mathematically identical to grouped attention).
* bf16 inputs: callers pass bf16-rounded values upcast to float32.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

F32 = np.float32
I64 = np.int64


# --------------------------------------------------------------------------
# policy configuration / decision types
# --------------------------------------------------------------------------


@dataclass
class PolicyConfig:
    """Mirror of ``streamkv.policies.PolicyConfig`` (policies.py:28-59)."""

    recent_len: int = 32
    relevant_budget: int = 2016
    bias: float = 0.1
    sink_count: int = 4
    head_agg: str = "mean"

    def __post_init__(self):  # policies.py:45-55
        if self.recent_len < 1:
            raise ValueError("recent_len must be >= 1")
        if self.relevant_budget < 0:
            raise ValueError("relevant_budget must be >= 0")
        if self.bias < 0:
            raise ValueError("bias must be >= 0")
        if self.sink_count < 0:
            raise ValueError("sink_count must be >= 0")
        if self.head_agg not in ("mean", "max"):
            raise ValueError(f"unknown head_agg {self.head_agg!r}")

    @property
    def budget(self) -> int:  # policies.py:57-59
        return self.recent_len + self.relevant_budget


@dataclass(frozen=True)
class Decision:
    """relevant / recent / kept index sets (policies.py:62-84)."""

    relevant: np.ndarray
    recent: np.ndarray
    kept: np.ndarray

    @staticmethod
    def everything(n: int, recent_len: int) -> "Decision":  # policies.py:76-84
        k = min(recent_len, n)
        return Decision(
            relevant=np.arange(0, n - k, dtype=I64),
            recent=np.arange(n - k, n, dtype=I64),
            kept=np.arange(n, dtype=I64),
        )


# --------------------------------------------------------------------------
# rolling relevance window
# --------------------------------------------------------------------------


class RowWindow:
    """Rolling list of the last ``capacity`` head-aggregated rows.

    Follows ``AttentionWindow`` (policies.py:87-127): push drops the oldest
    row beyond capacity (107-115); rows may not shrink between evictions
    (111-112); ``remap`` keeps, per row, the kept indices that row covers
    (117-124).
    """

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("window capacity must be >= 1")
        self.capacity = capacity
        self.rows: List[np.ndarray] = []

    def __len__(self) -> int:
        return len(self.rows)

    def push(self, row) -> None:
        r = np.asarray(row, dtype=F32)
        if r.ndim != 1 or r.size == 0:
            raise ValueError("row must be a non-empty vector")
        if self.rows and r.size < self.rows[-1].size:
            raise ValueError("row column count may not shrink between evictions")
        self.rows.append(r)
        while len(self.rows) > self.capacity:
            self.rows.pop(0)

    def remap(self, kept) -> None:
        idx = np.asarray(kept, dtype=I64)
        self.rows = [row[idx[idx < row.size]] for row in self.rows]

    def clear(self) -> None:
        self.rows = []


# --------------------------------------------------------------------------
# Algorithm-1 selection pieces (bit-exact float32 contract)
# --------------------------------------------------------------------------


def window_scores(window: RowWindow, n: int, l: int) -> np.ndarray:
    """policies.py:130-147: oldest->newest f32 column sums, then / f32(m)."""
    if len(window) == 0:
        raise ValueError("attention window is empty")
    if n <= l:
        raise ValueError(f"no scorable columns: n={n} <= l={l}")
    cols = n - l
    total = np.zeros(cols, dtype=F32)
    for row in window.rows:
        upto = min(row.size, cols)
        total[:upto] += row[:upto]
    return total / F32(len(window))


def age_bias(n: int, l: int, b: float) -> np.ndarray:
    """policies.py:150-162: d = f32(b)/f32(cols); bias[c] = (-d) * f32(cols-1-c)."""
    if n <= l:
        raise ValueError(f"no scorable columns: n={n} <= l={l}")
    if b < 0:
        raise ValueError("bias must be >= 0")
    cols = n - l
    step = F32(b) / F32(cols)
    ages = np.arange(cols - 1, -1, -1, dtype=F32)
    return (-step) * ages


def top_k_newer(scores, k: int) -> np.ndarray:
    """policies.py:165-181: k largest, ties toward the larger index, ascending."""
    s = np.asarray(scores, dtype=F32)
    if k < 0:
        raise ValueError("k must be >= 0")
    if k == 0:
        return np.empty(0, dtype=I64)
    if k >= s.size:
        return np.arange(s.size, dtype=I64)
    idx = np.arange(s.size, dtype=I64)
    order = np.lexsort((-idx, -s))  # primary: score desc; secondary: index desc
    return np.sort(order[:k])


def biased_scores(window: RowWindow, n: int, cfg: PolicyConfig) -> np.ndarray:
    """The array Algorithm 1 ranks (policies.py:196-197)."""
    return window_scores(window, n, cfg.recent_len) + age_bias(n, cfg.recent_len, cfg.bias)


def saddle_decide(window: RowWindow, n: int, cfg: PolicyConfig) -> Decision:
    """``inf_mllm_decide`` (policies.py:184-201)."""
    if len(window) == 0:
        raise ValueError("attention window is empty")
    l, r = cfg.recent_len, cfg.relevant_budget
    if n <= r + l:
        return Decision.everything(n, l)
    relevant = top_k_newer(biased_scores(window, n, cfg), r)
    recent = np.arange(n - l, n, dtype=I64)
    return Decision(relevant=relevant, recent=recent, kept=np.concatenate([relevant, recent]))


# --------------------------------------------------------------------------
# comparison baselines: the Session's other policies
# --------------------------------------------------------------------------


def recent_only(n: int, budget: int) -> Decision:
    """``sliding_window_decide`` (policies.py:204-213): the last ``budget``."""
    if budget < 1:
        raise ValueError("budget must be >= 1")
    k = min(budget, n)
    recent = np.arange(n - k, n, dtype=I64)
    return Decision(relevant=np.empty(0, dtype=I64), recent=recent, kept=recent)


def sinks_plus_recent(n: int, s: int, budget: int) -> Decision:
    """``sink_recent_decide`` (policies.py:216-231): first ``s`` + last ``budget - s``."""
    if not budget > s >= 0:
        raise ValueError("require budget > sink_count >= 0")
    if n <= budget:
        return Decision.everything(n, min(budget - s, n))
    sinks = np.arange(min(s, n), dtype=I64)
    recent = np.arange(n - (budget - s), n, dtype=I64)
    keep_sinks = sinks[sinks < recent[0]] if recent.size else sinks
    return Decision(relevant=keep_sinks, recent=recent, kept=np.concatenate([keep_sinks, recent]))


def mass_accumulate(acc: np.ndarray, new_row) -> np.ndarray:
    """``heavy_hitter_accumulate`` (policies.py:234-243): row + acc, padded."""
    a = np.asarray(acc, dtype=F32)
    row = np.asarray(new_row, dtype=F32)
    if a.size > row.size:
        raise ValueError("accumulator longer than the new row")
    out = row.copy()
    out[: a.size] += a
    return out


def mass_decide(acc: np.ndarray, n: int, r: int, l: int) -> Decision:
    """``heavy_hitter_decide`` (policies.py:246-256): top-r accumulated mass + last l."""
    a = np.asarray(acc, dtype=F32)
    if a.size != n:
        raise ValueError(f"accumulator length {a.size} != n={n}")
    if n <= r + l:
        return Decision.everything(n, l)
    relevant = top_k_newer(a[: n - l], r)
    recent = np.arange(n - l, n, dtype=I64)
    return Decision(relevant=relevant, recent=recent, kept=np.concatenate([relevant, recent]))


POLICIES = ("inf_mllm", "window", "sink_recent", "heavy_hitter", "none")


def head_mean(per_head: np.ndarray, how: str = "mean") -> np.ndarray:
    """``aggregate_heads`` (policies.py:259-265)."""
    if how == "mean":
        return per_head.mean(axis=0, dtype=F32)
    if how == "max":
        return per_head.max(axis=0)
    raise ValueError(f"unknown head aggregation {how!r}")


# --------------------------------------------------------------------------
# single-query attention
# --------------------------------------------------------------------------


def attend_heads(keys: np.ndarray, values: np.ndarray, q: np.ndarray, scale) -> tuple:
    """``Session._attend`` (engine.py:235-246), f32 per-head loop.

    keys/values: (H, n, D) f32; q: (H, D) f32.  Returns probs (H, n) and
    out (H, D), both f32.
    """
    heads, n, dim = keys.shape
    probs = np.empty((heads, n), dtype=F32)
    out = np.empty((heads, dim), dtype=F32)
    scale = F32(scale)
    for h in range(heads):
        logits = (keys[h] @ q[h]) * scale
        logits -= logits.max()
        np.exp(logits, out=logits)
        probs[h] = logits / logits.sum(dtype=F32)
        out[h] = probs[h] @ values[h]
    return probs, out


# --------------------------------------------------------------------------
# KV store
# --------------------------------------------------------------------------


class LayerKV:
    """One layer's (H, cap, D) f32 key/value store plus token metadata.

    Storage, growth and compaction follow ``_LayerStore`` / ``KvCache``
    (cache.py:44-67 layout + doubling growth, 112-134 append, 136-156
    gather_keep).  Head-major (H, cap, D) is kept so each head's keys are a
    contiguous (n, D) block, exactly what the reference hands to BLAS.
    """

    def __init__(self, heads: int, head_dim: int):
        self.n = 0
        cap = 64
        self.k = np.zeros((heads, cap, head_dim), dtype=F32)
        self.v = np.zeros((heads, cap, head_dim), dtype=F32)
        self.pos = np.zeros(cap, dtype=I64)
        self.modality = np.zeros(cap, dtype=np.int8)
        self.round_id = np.zeros(cap, dtype=np.int32)

    def _grow(self) -> None:
        cap = self.k.shape[1] * 2
        for name in ("k", "v"):
            old = getattr(self, name)
            new = np.zeros((old.shape[0], cap, old.shape[2]), dtype=F32)
            new[:, : self.n] = old[:, : self.n]
            setattr(self, name, new)
        for name in ("pos", "modality", "round_id"):
            old = getattr(self, name)
            new = np.zeros(cap, dtype=old.dtype)
            new[: self.n] = old[: self.n]
            setattr(self, name, new)

    def append(self, k: np.ndarray, v: np.ndarray, pos: int, modality: int = 0, round_id: int = 0):
        if self.n > 0 and pos <= self.pos[self.n - 1]:
            raise ValueError("original_position must be strictly increasing")
        if self.n == self.k.shape[1]:
            self._grow()
        self.k[:, self.n] = k
        self.v[:, self.n] = v
        self.pos[self.n] = pos
        self.modality[self.n] = modality
        self.round_id[self.n] = round_id
        self.n += 1

    def gather_keep(self, kept) -> None:
        idx = np.asarray(kept, dtype=I64)
        if idx.ndim != 1:
            raise ValueError("kept must be a 1-D index set")
        if idx.size:
            if idx[0] < 0 or idx[-1] >= self.n:
                raise ValueError(f"kept indices out of range [0, {self.n})")
            if np.any(np.diff(idx) <= 0):
                raise ValueError("kept indices must be strictly ascending")
        m = idx.size
        self.k[:, :m] = self.k[:, idx]
        self.v[:, :m] = self.v[:, idx]
        self.pos[:m] = self.pos[idx]
        self.modality[:m] = self.modality[idx]
        self.round_id[:m] = self.round_id[idx]
        self.n = m

    def keys(self) -> np.ndarray:
        return self.k[:, : self.n]

    def values(self) -> np.ndarray:
        return self.v[:, : self.n]


# --------------------------------------------------------------------------
# rotary positions
# --------------------------------------------------------------------------


class Rotary:
    """The reference Session's rotary helpers (engine.py:175-180, 198-233):
    inv_freq = base ** (-2 i / D) in f64, cos/sin tables grown in f64 and cast
    to f32, interleaved (even, odd) pairs rotated with f32 products."""

    def __init__(self, head_dim: int, base: float = 10000.0):
        half = head_dim // 2
        self.inv_freq = base ** (-2.0 * np.arange(half, dtype=np.float64) / head_dim)  # engine.py:176-178
        self.cos = np.zeros((0, half), dtype=F32)
        self.sin = np.zeros((0, half), dtype=F32)

    def _trig(self, upto: int) -> None:  # engine.py:200-207
        if upto <= self.cos.shape[0]:
            return
        size = max(upto, 256, self.cos.shape[0] * 2)
        pos = np.arange(size, dtype=np.float64)[:, None]
        ang = pos * self.inv_freq
        self.cos = np.cos(ang).astype(F32)
        self.sin = np.sin(ang).astype(F32)

    def rotate_one(self, vec: np.ndarray, position: int) -> np.ndarray:  # engine.py:209-219
        self._trig(position + 1)
        cos, sin = self.cos[position], self.sin[position]
        even, odd = vec[:, 0::2], vec[:, 1::2]
        out = np.empty_like(vec)
        out[:, 0::2] = even * cos - odd * sin
        out[:, 1::2] = even * sin + odd * cos
        return out

    def rotate_many(self, block: np.ndarray, positions: np.ndarray) -> np.ndarray:  # engine.py:221-233
        if positions.size == 0:
            return block.copy()
        self._trig(int(positions.max()) + 1)
        cos, sin = self.cos[positions], self.sin[positions]
        even, odd = block[:, :, 0::2], block[:, :, 1::2]
        out = np.empty_like(block)
        out[:, :, 0::2] = even * cos - odd * sin
        out[:, :, 1::2] = even * sin + odd * cos
        return out


ROPE_MODES = (None, "cache_relative", "original")


# --------------------------------------------------------------------------
# composed streaming driver
# --------------------------------------------------------------------------


class StreamOracle:
    """S independent streams x L layers of the reference decode+evict path.

    Per decode step and layer (engine.py:264-273): append, attend over the
    cache including the new token, head-mean row, window push.  At an
    eviction (engine.py:310-337, called after a round's prompt
    engine.py:350-360): ``inf_mllm_decide`` -> ``gather_keep`` ->
    ``window.remap`` when the decision drops anything.

    ``window`` is the relevance-window row count W; the reference Session ties
    it to ``recent_len`` (engine.py:147) while the pure policy API takes it
    freely (policies.py:98), which is how BASELINE's W=32 is expressed.
    """

    def __init__(self, streams: int, layers: int, heads_q: int, heads_kv: int, head_dim: int,
                 cfg: PolicyConfig, window: Optional[int] = None, policy: str = "inf_mllm",
                 rope: Optional[str] = None, rope_base: float = 10000.0, rope_round=None):
        if heads_q % heads_kv:
            raise ValueError("heads_q must be a multiple of heads_kv")
        if policy not in POLICIES:
            raise ValueError(f"unknown policy {policy!r}")
        self.policy = policy
        if rope not in ROPE_MODES:
            raise ValueError(f"unknown rope mode {rope!r}")
        # Rotary positions: raw keys stay in the cache, rotated keys (the
        # Session's _rot store) are what attention reads.  rope_round models a
        # bf16 engine, whose rotated q / k are bf16 values (pass bf16_round).
        self.rope = rope
        self.rotary = Rotary(head_dim, rope_base) if rope else None
        self.rope_round = rope_round
        self.rot = [[np.zeros((heads_kv, 0, head_dim), dtype=F32) for _ in range(layers)] for _ in range(streams)]
        # heavy-hitter accumulators, one per (stream, layer) (engine.py:274)
        self.acc = [[np.zeros(0, dtype=F32) for _ in range(layers)] for _ in range(streams)]
        self.S, self.L, self.Hq, self.Hkv, self.D = streams, layers, heads_q, heads_kv, head_dim
        self.group = heads_q // heads_kv
        self.cfg = cfg
        self.W = window if window is not None else cfg.recent_len
        self.scale = F32(1.0 / np.sqrt(head_dim))  # engine.py:150
        self.kv = [[LayerKV(heads_kv, head_dim) for _ in range(layers)] for _ in range(streams)]
        self.win = [[RowWindow(self.W) for _ in range(layers)] for _ in range(streams)]
        self.pos = [0] * streams
        self.shadow = False

    def enable_shadow(self) -> None:
        """Session(oracle=True) (engine.py:142-151): a never-evicted shadow
        cache plus the last recent_len head-aggregated rows over it."""
        self.shadow = True
        S, L = self.S, self.L
        self.skv = [[LayerKV(self.Hkv, self.D) for _ in range(L)] for _ in range(S)]
        self.srows = [[RowWindow(self.cfg.recent_len) for _ in range(L)] for _ in range(S)]

    def shadow_metrics(self, s: int, layer: int, decision: "Decision"):
        """_evict_layer's oracle metrics (engine.py:314-331), before compaction:
        (retained mass, top-r overlap or None)."""
        orig = self.kv[s][layer].pos[: self.kv[s][layer].n]
        kept_ids, relevant_ids = orig[decision.kept], orig[decision.relevant]
        rows = self.srows[s][layer].rows
        mass = retained_mass_rows(rows, kept_ids)
        ns, l = self.skv[s][layer].n, self.cfg.recent_len
        overlap = None
        if ns > l and self.cfg.relevant_budget >= 1:
            cols = ns - l
            acc = np.zeros(cols, dtype=F32)
            for row in rows:
                m = min(row.size, cols)
                acc[:m] += row[:m]
            overlap = topk_overlap_ids(acc / F32(len(rows)), relevant_ids, self.cfg.relevant_budget)
        return mass, overlap

    def length(self, s: int, layer: int) -> int:
        return self.kv[s][layer].n

    def _expanded(self, s: int, layer: int):
        st = self.kv[s][layer]
        k, v = (st.keys() if not self.rope else self.rot[s][layer]), st.values()
        if self.group > 1:
            k = np.repeat(k, self.group, axis=0)
            v = np.repeat(v, self.group, axis=0)
        return k, v

    def step_layer(self, layer: int, q: np.ndarray, k: np.ndarray, v: np.ndarray,
                   streams: Optional[Sequence[int]] = None):
        """One decode step of one layer.  q: (S,Hq,D), k/v: (S,Hkv,D) f32.

        Returns out (S,Hq,D) f32 and the pushed rows (list of f32 vectors).
        """
        out = np.zeros((self.S, self.Hq, self.D), dtype=F32)
        rows = []
        for s in (range(self.S) if streams is None else streams):
            st = self.kv[s][layer]
            st.append(np.asarray(k[s], F32), np.asarray(v[s], F32), self.pos[s])
            qs = np.asarray(q[s], F32)
            if self.rope:  # engine.py:265-268: rotate the new key and the query at one position
                p = st.n - 1 if self.rope == "cache_relative" else self.pos[s]
                rk = self.rotary.rotate_one(np.asarray(k[s], F32), p)
                qs = self.rotary.rotate_one(qs, p)
                if self.rope_round is not None:
                    rk, qs = self.rope_round(rk), self.rope_round(qs)
                self.rot[s][layer] = np.concatenate([self.rot[s][layer], rk[:, None, :]], axis=1)
            keys, vals = self._expanded(s, layer)
            probs, o = attend_heads(keys, vals, qs, self.scale)
            row = head_mean(probs, self.cfg.head_agg)
            self.win[s][layer].push(row)
            self.acc[s][layer] = mass_accumulate(self.acc[s][layer], row)
            out[s] = o
            rows.append(row)
            if self.shadow:  # engine.py:275-284 (no RoPE in the shadow restatement)
                ss = self.skv[s][layer]
                ss.append(np.asarray(k[s], F32), np.asarray(v[s], F32), self.pos[s])
                sk, sv = ss.keys(), ss.values()
                if self.group > 1:
                    sk, sv = np.repeat(sk, self.group, axis=0), np.repeat(sv, self.group, axis=0)
                sprobs, _ = attend_heads(sk, sv, np.asarray(q[s], F32), self.scale)
                self.srows[s][layer].push(head_mean(sprobs, self.cfg.head_agg))
        return out, rows

    def advance(self, streams: Optional[Sequence[int]] = None) -> None:
        for s in (range(self.S) if streams is None else streams):
            self.pos[s] += 1

    def step(self, q, k, v):
        """All layers of one token: q (L,S,Hq,D), k/v (L,S,Hkv,D)."""
        outs = []
        for layer in range(self.L):
            o, _ = self.step_layer(layer, q[layer], k[layer], v[layer])
            outs.append(o)
        self.advance()
        return np.stack(outs)

    def decide(self, s: int, layer: int) -> Decision:
        """The Session's policy switch ``_decide`` (engine.py:293-307)."""
        n, cfg = self.kv[s][layer].n, self.cfg
        if self.policy == "none":
            return Decision.everything(n, min(cfg.recent_len, n))
        if self.policy == "window":
            return recent_only(n, cfg.budget)
        if self.policy == "sink_recent":
            return sinks_plus_recent(n, cfg.sink_count, cfg.budget)
        if self.policy == "heavy_hitter":
            return mass_decide(self.acc[s][layer], n, cfg.relevant_budget, cfg.recent_len)
        return saddle_decide(self.win[s][layer], n, cfg)

    def scores(self, s: int, layer: int) -> np.ndarray:
        return biased_scores(self.win[s][layer], self.kv[s][layer].n, self.cfg)

    def apply(self, s: int, layer: int, kept) -> None:
        """Compaction half of ``_evict_layer`` (engine.py:332-334)."""
        kept = np.asarray(kept, dtype=I64)
        if kept.size != self.kv[s][layer].n:
            self.kv[s][layer].gather_keep(kept)
            self.win[s][layer].remap(kept)
            self.acc[s][layer] = self.acc[s][layer][kept]  # engine.py:335
            if self.rope:  # _refresh_rotations, engine.py:339-342 (positions_for, cache.py:160-165)
                st = self.kv[s][layer]
                positions = np.arange(st.n, dtype=I64) if self.rope == "cache_relative" else st.pos[: st.n].copy()
                rot = self.rotary.rotate_many(st.keys(), positions)
                self.rot[s][layer] = self.rope_round(rot) if self.rope_round is not None else rot

    def evict(self):
        """Decide + apply for every (stream, layer); returns kept[s][l]."""
        kept = []
        for s in range(self.S):
            per = []
            for layer in range(self.L):
                d = self.decide(s, layer)
                self.apply(s, layer, d.kept)
                per.append(d.kept)
            kept.append(per)
        return kept


# --------------------------------------------------------------------------
# quality metrics (metrics.py:46-73)
# --------------------------------------------------------------------------


def retained_mass_rows(rows, kept_ids) -> float:
    """retained_mass (metrics.py:46-62): mean over rows of the f64 mass on kept ids."""
    if not rows:
        raise ValueError("retained_mass needs at least one scoring row")
    idx = np.asarray(kept_ids, dtype=I64)
    total = 0.0
    for row in rows:
        sel = idx[idx < row.size]
        total += float(row[sel].sum(dtype=np.float64)) if sel.size else 0.0
    return total / len(rows)


def topk_overlap_ids(oracle_scores, relevant_ids, r: int) -> float:
    """topk_overlap (metrics.py:65-73): |relevant & oracle top-r| / r."""
    top = set(int(i) for i in top_k_newer(np.asarray(oracle_scores, dtype=F32), r))
    return len(top & set(int(i) for i in np.asarray(relevant_ids, dtype=I64))) / r


# --------------------------------------------------------------------------
# near-tie-aware kept-set comparison (north-star parity rule)
# --------------------------------------------------------------------------


def kept_sets_match(cpu_biased: np.ndarray, cpu_kept: np.ndarray, gpu_kept: np.ndarray,
                    n: int, cfg: PolicyConfig, rel_tol: float = 1e-6) -> tuple:
    """Kept sets must be identical except where the CPU biased-score gap between
    a mismatched column and the CPU k-th score is below ``rel_tol`` relative.

    Returns (ok, n_mismatched, worst_gap).
    """
    a = set(np.asarray(cpu_kept).tolist())
    b = set(np.asarray(gpu_kept).tolist())
    diff = sorted(a ^ b)
    if not diff:
        return True, 0, 0.0
    if len(a) != len(b):
        return False, len(diff), float("inf")
    cols = n - cfg.recent_len
    if any(i >= cols for i in diff):  # the recent window must always agree
        return False, len(diff), float("inf")
    s = np.asarray(cpu_biased, dtype=np.float64)
    kth = np.sort(s)[::-1][cfg.relevant_budget - 1]
    worst = 0.0
    for i in diff:
        gap = abs(s[i] - kth) / max(abs(kth), abs(s[i]), 1e-30)
        worst = max(worst, gap)
    return worst <= rel_tol, len(diff), worst


# --------------------------------------------------------------------------
# seeded synthetic inputs (BASELINE.json configs; shapes only, no datasets)
# --------------------------------------------------------------------------


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(x, dtype=F32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) >> 16 << 16
    out = u.astype(np.uint32).view(F32).copy()
    nan = np.isnan(a)
    out[nan] = a[nan]
    return out


def synth_step(rng: np.random.Generator, streams: int, heads_q: int, heads_kv: int, head_dim: int,
               spike_prob: float, spike_gain: float, bf16: bool):
    """One token of q/k/v ~ N(0,1); a key spike multiplies all KV heads' key
    of that (stream, token) by ``spike_gain`` with probability ``spike_prob``."""
    q = rng.standard_normal((streams, heads_q, head_dim)).astype(F32)
    k = rng.standard_normal((streams, heads_kv, head_dim)).astype(F32)
    v = rng.standard_normal((streams, heads_kv, head_dim)).astype(F32)
    spikes = rng.random(streams) < spike_prob
    k[spikes] *= F32(spike_gain)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v
