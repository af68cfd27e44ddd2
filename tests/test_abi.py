"""CPU-side checks of the C ABI library: it loads without a GPU and exports
every symbol declared in include/streamkv_b200.h; host-side argument
validation maps to the reference's ValueError domain."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "streamkv_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(skv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    assert "skv_create" in names and "skv_decode_layer" in names and "skv_evict" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2409_09086_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_config_validation_without_gpu():
    """skv_create validates the config before touching the device."""
    from paper_2409_09086_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    bad = _lib.SkvConfig(streams=1, layers=1, heads_q=3, heads_kv=2, head_dim=128, dtype=1, recent_len=4,
                         relevant_budget=4, bias=0.1, window=4, capacity=64, head_agg=0)
    h = ctypes.c_void_p()
    assert lib.skv_create(ctypes.byref(bad), ctypes.byref(h)) == _lib.SKV_EINVAL
    assert b"multiple" in lib.skv_last_error()
    bad.heads_q = 4
    bad.head_dim = 96
    assert lib.skv_create(ctypes.byref(bad), ctypes.byref(h)) == _lib.SKV_EINVAL
    bad.head_dim = 128
    bad.recent_len = 0
    assert lib.skv_create(ctypes.byref(bad), ctypes.byref(h)) == _lib.SKV_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.SKV_EINVAL)
    assert lib.skv_top_k(None, 4, -1, None, None) == _lib.SKV_EINVAL


def test_policy_validation_without_gpu():
    """The Session's policy switch (engine.py:296-307) and sink_recent_decide's
    budget > sink_count >= 0 rule (policies.py:218-219) are checked host-side."""
    from paper_2409_09086_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    c = _lib.SkvConfig(streams=1, layers=1, heads_q=4, heads_kv=4, head_dim=128, dtype=1, recent_len=4,
                       relevant_budget=4, bias=0.1, window=4, capacity=64, head_agg=0, policy=9)
    h = ctypes.c_void_p()
    assert lib.skv_create(ctypes.byref(c), ctypes.byref(h)) == _lib.SKV_EINVAL
    assert b"policy" in lib.skv_last_error()
    c.policy = _lib.POLICIES["sink_recent"]
    c.sink_count = 8  # budget 8 is not > 8
    assert lib.skv_create(ctypes.byref(c), ctypes.byref(h)) == _lib.SKV_EINVAL
    assert b"sink_count" in lib.skv_last_error()
    # stand-alone decisions: argument checks precede any device work
    assert lib.skv_policy_decide(0, None, 4, 2, 2, 0, None, None, None) == _lib.SKV_EINVAL
    assert lib.skv_policy_decide(_lib.POLICIES["window"], None, 4, 0, 0, 0, None, None, None) == _lib.SKV_EINVAL
    assert lib.skv_policy_decide(_lib.POLICIES["heavy_hitter"], None, 9, 2, 2, 0, None, None, None) == _lib.SKV_EINVAL
    assert lib.skv_hh_accumulate(None, 5, None, 4, None, None) == _lib.SKV_EINVAL
    assert lib.skv_policy_decide(_lib.POLICIES["window"], None, 0, 4, 0, 0, None, None, None) == 0
