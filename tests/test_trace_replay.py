"""Trace replay: the .imtrace reader (CPU) and the
device replay of every policy against the reference's own replay_trace run
(tests/golden/ref_replay.npz, made by tests/golden/make_replay_golden.py)."""

import io
import os
import struct

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_replay.npz")
POLICIES = ["inf-mllm", "heavy-hitter", "window", "sink-recent", "none"]
CFG = dict(recent_len=16, relevant_budget=24, bias=0.05, sink_count=3)


def _trace_bytes():
    return np.load(GOLD)["trace"].tobytes()


def test_reader_parses_reference_trace():
    from paper_2409_09086_b200.traceio import AttnRow, RoundStart, SaddleTruth, Tokens, read_trace

    header, events = read_trace(io.BytesIO(_trace_bytes()))
    events = list(events)
    assert (header.layers, header.heads, header.version) == (2, 4, 1)
    rows = [e for e in events if isinstance(e, AttnRow)]
    assert len([e for e in events if isinstance(e, RoundStart)]) == 9
    assert len([e for e in events if isinstance(e, SaddleTruth)]) == 3
    assert all(isinstance(e, (AttnRow, RoundStart, SaddleTruth, Tokens)) for e in events)
    assert len(rows) == 2 * 9 * 44 and {r.layer for r in rows} == {0, 1}
    for r in rows:
        assert abs(float(r.probs.sum(dtype=np.float64)) - 1.0) <= 1e-3


def test_reader_errors_name_the_offset():
    from paper_2409_09086_b200.traceio import TraceFormatError, read_trace

    with pytest.raises(TraceFormatError, match="bad magic"):
        read_trace(io.BytesIO(b"XXXX" + bytes(16)))
    hdr = struct.pack("<4sIIII", b"IMT1", 1, 1, 1, 1)
    bad_row = struct.pack("<BII", 3, 0, 2) + np.array([0.2, 0.2], "<f4").tobytes()
    _, ev = read_trace(io.BytesIO(hdr + bad_row))
    with pytest.raises(TraceFormatError, match="byte offset 20"):
        list(ev)
    _, ev = read_trace(io.BytesIO(hdr + struct.pack("<BII", 3, 0, 4) + bytes(4)))
    with pytest.raises(TraceFormatError, match="truncated"):
        list(ev)
    _, ev = read_trace(io.BytesIO(hdr + bytes([9])))
    with pytest.raises(TraceFormatError, match="unknown event tag 9"):
        list(ev)


@pytest.mark.gpu
@pytest.mark.parametrize("fixture", ["ref_replay.npz", "ref_replay2.npz"])
@pytest.mark.parametrize("policy", POLICIES)
def test_device_replay_matches_reference(policy, fixture):
    """ref_replay2.npz: three layers, 8 heads, 40-token prompts, its own policy
    config (stored in the fixture) -- the reference replay_trace's output."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_09086_b200 import PolicyConfig
    from paper_2409_09086_b200.replay import replay_trace
    from paper_2409_09086_b200.traceio import read_trace

    ref = dict(np.load(os.path.join(os.path.dirname(GOLD), fixture)))
    l, r, sink, head_dim = (int(x) for x in ref["cfg"])
    cfg = PolicyConfig(recent_len=l, relevant_budget=r, bias=float(ref["bias"][0]), sink_count=sink)
    key = policy.replace("-", "_")
    header, events = read_trace(io.BytesIO(ref["trace"].tobytes()))
    res = replay_trace(header, list(events), policy, cfg, head_dim=head_dim)
    kept = [d.kept for rnd in res.decisions_per_round for d in rnd]
    off = ref[f"{key}_kept_off"]
    assert len(kept) == off.size - 1
    for i, k in enumerate(kept):
        k = k.cpu().numpy() if hasattr(k, "cpu") else np.asarray(k)
        np.testing.assert_array_equal(k, ref[f"{key}_kept"][off[i]: off[i + 1]], err_msg=f"decision {i}")
    m = ref[f"{key}_metrics"]
    assert len(res.rows) == m.shape[0]
    for row, want in zip(res.rows, m):
        assert row.round_id == int(want[0])
        np.testing.assert_allclose(row.retained_mass, want[1], rtol=1e-9)
        for got, w in ((row.topk_overlap, want[2]), (row.planted_recall, want[3])):
            if np.isnan(w):
                assert got is None
            else:
                assert got == pytest.approx(w, abs=1e-12)
        assert (row.cache_len, row.memory_bytes, row.flops_per_token) == (int(want[4]), int(want[5]), int(want[6]))
