"""B200-native (sm_100a) Inf-MLLM streaming-decode hot path.

Drop-in for the hot-path API of the reference ``streamkv`` package
(/root/reference/pkg/src/streamkv/__init__.py:3-32): ``KvCache``,
``AttentionWindow``, ``PolicyConfig``, ``EvictionDecision``,
``window_mean_scores``, ``bias_vector``, ``top_k_indices``, ``inf_mllm_decide``,
``aggregate_heads``, ``attend`` (Session._attend) and the tensorops
``softmax_row`` / ``attn_probs`` / ``weighted_sum`` / ``rope_apply``, the comparison baselines
``sliding_window_decide``, ``sink_recent_decide``, ``heavy_hitter_accumulate``
and ``heavy_hitter_decide``, plus the batched
``StreamEngine`` that runs decode + score + evict for many streams through
libstreamkv_b200.so.  No CPU fallback: everything computes on the GPU.
"""

from ._lib import LIB_PATH, load as load_library
from .cache import KvCache, PositionMode, TokenMeta
from .engine import EngineConfig, StreamEngine
from .policies import (
    AttentionWindow,
    EvictionDecision,
    PolicyConfig,
    aggregate_heads,
    bias_vector,
    heavy_hitter_accumulate,
    heavy_hitter_decide,
    inf_mllm_decide,
    sink_recent_decide,
    sliding_window_decide,
    top_k_indices,
    window_mean_scores,
)
from .metrics import MetricsRow, planted_recall, retained_mass, topk_overlap
from .replay import ReplayResult, replay_trace
from .tensorops import attend, attn_probs, rope_apply, softmax_row, weighted_sum
from .traceio import TraceFormatError, read_trace, read_trace_file

__version__ = "0.1.0"
