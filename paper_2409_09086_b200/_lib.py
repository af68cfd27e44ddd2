"""ctypes binding of libstreamkv_b200.so (the C ABI in include/streamkv_b200.h).

There is no fallback: if the library is missing or no CUDA device is present,
every compute entry point raises.  Domain errors (SKV_EINVAL) become
``ValueError`` exactly where the reference raises ``ValueError``; CUDA errors
become ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKV_LIB points the binding at another build of the same ABI (A/B timing of
# kernel variants with tools/; the product path uses the in-tree library)
LIB_PATH = os.environ.get("SKV_LIB") or os.path.join(_HERE, "libstreamkv_b200.so")

SKV_OK = 0
SKV_EINVAL = -1
SKV_ECUDA = -2
SKV_ENOMEM = -3
SKV_ESTATE = -4

DTYPE_F32 = 0
DTYPE_BF16 = 1
AGG_MEAN = 0
AGG_MAX = 1

# eviction policies (engine.py:296-307)
POLICIES = {"inf_mllm": 0, "window": 1, "sink_recent": 2, "heavy_hitter": 3, "none": 4}
# rotary position modes (PositionMode, cache.py:24-34); None: inputs arrive rotated
ROPE_MODES = {None: 0, "cache_relative": 1, "original": 2}


class SkvConfig(ctypes.Structure):
    _fields_ = [
        ("streams", ctypes.c_int32),
        ("layers", ctypes.c_int32),
        ("heads_q", ctypes.c_int32),
        ("heads_kv", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("recent_len", ctypes.c_int32),
        ("relevant_budget", ctypes.c_int32),
        ("bias", ctypes.c_float),
        ("window", ctypes.c_int32),
        ("capacity", ctypes.c_int32),
        ("head_agg", ctypes.c_int32),
        ("heads_q_total", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("sink_count", ctypes.c_int32),
        ("rope_mode", ctypes.c_int32),
        ("rope_base", ctypes.c_float),
    ]


# name -> (restype, argtypes); every symbol declared in include/streamkv_b200.h
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_F = ctypes.c_float
SIGNATURES = {
    "skv_last_error": (ctypes.c_char_p, []),
    "skv_version": (_I, []),
    "skv_create": (_I, [ctypes.POINTER(SkvConfig), ctypes.POINTER(_P)]),
    "skv_destroy": (_I, [_P]),
    "skv_device_bytes": (_I64, [_P]),
    "skv_decode_layer": (_I, [_P, _I, _P, _P, _P, _P, _P, _I, _P]),
    "skv_decode_step": (_I, [_P, _P, _P, _P, _P, _I, _P]),
    "skv_decode_step_host": (_I, [_P, _P, _P, _P, _P, _I, _P]),
    "skv_host_speculate": (_I, [_P, _I, _I]),
    "skv_host_speculate_stats": (_I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "skv_evict": (_I, [_P, _I, _P, _P]),
    "skv_evict_scores": (_I, [_P, _I, _P, _P]),
    "skv_evict_apply": (_I, [_P, _I, _P, _P, _P]),
    "skv_length": (_I, [_P, _I, _I]),
    "skv_kv_view": (_I, [_P, _I, _I, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "skv_positions": (_I, [_P, _I, _I, _P, _I]),
    "skv_window_rows": (_I, [_P, _I, _I, _P, _P]),
    "skv_last_scores": (_I, [_P, _I, _I, _P, _I]),
    "skv_state_inject": (_I, [_P, _I, _I, _I, _P, _P, _P, _I, _P, _P]),
    "skv_state_dump": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "skv_sync": (_I, [_P, _P]),
    "skv_slot_map": (_I, [_P, _I, _I, ctypes.POINTER(_P)]),
    "skv_moved_rows": (_I, [_P, _P]),
    "skv_capture_begin": (_I, [_P, _P]),
    "skv_capture_end": (_I, [_P, _P]),
    "skv_graph_launch": (_I, [_P, _P]),
    "skv_kernel_launches": (_I64, [_P]),
    "skv_timing": (_I, [_P, _I]),
    "skv_timing_read": (_I, [_P, _P, _I]),
    "skv_timing_cta": (_I, [_P, _I, _P]),
    "skv_layers_timeline": (_I, [_P, _P]),
    "skv_last_decode_kernel": (ctypes.c_char_p, [_P]),
    "skv_prefill_profile": (_I, [_P]),
    "skv_prefill_chunk": (_I, [_P, _I, _P, _P, _P, _I, _I, _P, _P]),
    "skv_prefill_attend": (_I, [_P, _I, _I, _I, _I, _P, _P, _I, _I, _I, _I, _P, _I, _P, _I64, _P, _P]),
    "skv_top_k": (_I, [_P, _I, _I, _P, _P]),
    "skv_decide": (_I, [_P, _I, _P, _I, _I, _I, _I, _F, _P, _P, _P]),
    "skv_policy_decide": (_I, [_I, _P, _I, _I, _I, _I, _P, _P, _P]),
    "skv_hh_accumulate": (_I, [_P, _I, _P, _I, _P, _P]),
    "skv_project_row": (_I, [_P, _I, _P, _I, _P, _P]),
    "skv_masked_row_sums": (_I, [_P, _I, _P, _I, _P, _I, _P, _P]),
    "skv_window_scores": (_I, [_P, _I, _P, _I, _I, _I, _F, _I, _P, _P]),
    "skv_gather_rows": (_I, [_P, _I64, _I, _I, _P, _I, _P]),
    "skv_attend": (_I, [_P, _P, _I, _I, _I, _I64, _P, _P, _P, _P]),
    "skv_softmax_row": (_I, [_P, _I, _P, _P]),
    "skv_attn_probs": (_I, [_P, _P, _I, _I, _F, _P, _P]),
    "skv_weighted_sum": (_I, [_P, _P, _I, _I, _P, _P]),
    "skv_rope_apply": (_I, [_P, _I, _I64, ctypes.c_double, _P, _P]),
    "skv_aggregate_heads": (_I, [_P, _I, _I, _I, _P, _P]),
    "skv_bias_vector": (_I, [_I, _I, _F, _P, _P]),
    "skv_window_view": (_I, [_P, _I, _I, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_I),
                             ctypes.POINTER(_I)]),
    "skv_positions_view": (_I, [_P, _I, _I, ctypes.POINTER(_P)]),
    "skv_round_metrics": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P]),
    "skv_replay_rows": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P]),
    "skv_replay_evict": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _F, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P, _I, _P, _P,
                              _P]),
}

_lib = None


def load():
    """Load the shared library (raises if it is absent: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing; build it with ./build.sh (or __graft_entry__.build()). "
                "There is no CPU fallback for the streamkv B200 path."
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> int:
    """Map a C status to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = load().skv_last_error().decode()
    if rc == SKV_EINVAL:
        raise ValueError(msg)
    if rc == SKV_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"streamkv_b200 error {rc}: {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("streamkv_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    load()
