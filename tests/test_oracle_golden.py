"""Pin the CPU oracle against the reference's own outputs and known answers.

The fixtures in tests/golden were produced by running the reference
``streamkv`` package (tests/golden/make_golden.py).  The oracle restates the
reference's float32 operation sequence, so agreement is required to be
bit-exact; see oracle/streamkv_oracle.py.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle.streamkv_oracle import (
    Decision,
    PolicyConfig,
    RowWindow,
    age_bias,
    attend_heads,
    biased_scores,
    head_mean,
    kept_sets_match,
    saddle_decide,
    top_k_newer,
    window_scores,
    LayerKV,
)
from tests.golden.cases import CASES, kat_instances
from tests.oracle_runner import run_oracle_case

F32 = np.float32
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return dict(np.load(os.path.join(GOLD, f"ref_{name}.npz")))


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_reference_run(name):
    ref = _load(name)
    got = run_oracle_case(name)
    np.testing.assert_array_equal(got["evict_steps"], ref["evict_steps"])
    np.testing.assert_array_equal(got["kept_off"], ref["kept_off"])
    np.testing.assert_array_equal(got["kept"], ref["kept"])
    np.testing.assert_array_equal(got["score_off"], ref["score_off"])
    # selection arithmetic is pinned bit-exactly
    np.testing.assert_array_equal(got["scores"].view(np.uint32), ref["scores"].view(np.uint32))
    np.testing.assert_array_equal(got["out_steps"], ref["out_steps"])
    # attention runs through the same BLAS calls on the same layout
    np.testing.assert_allclose(got["outs"], ref["outs"], rtol=0, atol=1e-6)
    np.testing.assert_array_equal(got["final_pos"], ref["final_pos"])
    np.testing.assert_array_equal(got["final_keys_sha"], ref["final_keys_sha"])
    if "shadow_mass" in ref and ref["shadow_mass"].size:  # Session(oracle=True) metrics
        np.testing.assert_allclose(got["shadow_mass"], ref["shadow_mass"], rtol=1e-12)
        np.testing.assert_array_equal(np.isnan(got["shadow_overlap"]), np.isnan(ref["shadow_overlap"]))
        np.testing.assert_array_equal(np.nan_to_num(got["shadow_overlap"]), np.nan_to_num(ref["shadow_overlap"]))


def test_algorithm1_kats_match_reference():
    ref = dict(np.load(os.path.join(GOLD, "ref_kat_algorithm1.npz")))
    for i, inst in enumerate(kat_instances()):
        w = RowWindow(len(inst["rows"]))
        for row in inst["rows"]:
            w.push(row)
        cfg = PolicyConfig(recent_len=inst["l"], relevant_budget=inst["r"], bias=inst["b"])
        kept = saddle_decide(w, inst["n"], cfg).kept
        want = ref["kept"][ref["kept_off"][i]: ref["kept_off"][i + 1]]
        np.testing.assert_array_equal(kept, want)
        if inst["n"] > inst["l"]:
            sc = biased_scores(w, inst["n"], cfg)
        else:
            sc = np.zeros(0, F32)
        sha = np.frombuffer(hashlib.sha256(sc.astype(F32).tobytes()).digest(), np.uint8)
        np.testing.assert_array_equal(sha, ref["score_sha"][i])


def test_topk_kats_match_reference():
    ref = dict(np.load(os.path.join(GOLD, "ref_kat_algorithm1.npz")))
    rng = np.random.default_rng(23)
    for i in range(200):
        size = int(rng.integers(1, 50))
        scores = rng.choice([0.1, 0.2, 0.3, 0.5], size=size).astype(F32)
        k = int(rng.integers(0, size + 1))
        want = ref["topk"][ref["topk_off"][i]: ref["topk_off"][i + 1]]
        np.testing.assert_array_equal(top_k_newer(scores, k), want)


# ---- worked examples written in the reference's unit tests -----------------


def _win(rows):
    w = RowWindow(len(rows))
    for r in rows:
        w.push(np.asarray(r, dtype=F32))
    return w


def test_window_mean_two_row_example():  # test_policies.py:44-46
    w = _win([[0.2, 0.4, 0.1, 0.3], [0.4, 0.2, 0.1, 0.3]])
    np.testing.assert_allclose(window_scores(w, 4, 2), [0.3, 0.3], atol=1e-7)


def test_bias_worked_example():  # test_policies.py:74-75
    np.testing.assert_allclose(age_bias(6, 2, 0.1), [-0.075, -0.05, -0.025, 0.0], atol=1e-7)
    np.testing.assert_array_equal(age_bias(5, 4, 2.5), [0.0])


def test_topk_tie_newer():  # test_policies.py:97-98
    np.testing.assert_array_equal(top_k_newer([0.5, 0.5, 0.2], 1), [1])
    assert top_k_newer([1.0, 2.0], 0).size == 0
    np.testing.assert_array_equal(top_k_newer([3.0, 1.0], 5), [0, 1])


def test_algorithm1_worked_example():  # test_policies.py:119-128
    w = _win([[0.30, 0.10, 0.20, 0.25, 0.15], [0.10, 0.30, 0.20, 0.15, 0.25]])
    d = saddle_decide(w, 5, PolicyConfig(recent_len=2, relevant_budget=1, bias=0.4))
    np.testing.assert_array_equal(d.relevant, [2])
    np.testing.assert_array_equal(d.recent, [3, 4])
    np.testing.assert_array_equal(d.kept, [2, 3, 4])


def test_uniform_scores_keep_newest():  # test_policies.py:135-139
    w = _win([np.full(10, 0.1, dtype=F32)])
    d = saddle_decide(w, 10, PolicyConfig(recent_len=2, relevant_budget=3, bias=0.0))
    np.testing.assert_array_equal(d.relevant, [5, 6, 7])


def test_under_budget_keeps_all():
    w = _win([np.full(5, 0.2)])
    d = saddle_decide(w, 5, PolicyConfig(recent_len=2, relevant_budget=3))
    np.testing.assert_array_equal(d.kept, np.arange(5))
    assert isinstance(d, Decision)


def test_domain_errors():
    with pytest.raises(ValueError):
        window_scores(RowWindow(4), 8, 2)
    with pytest.raises(ValueError):
        window_scores(_win([[0.5, 0.5]]), 2, 2)
    with pytest.raises(ValueError):
        age_bias(4, 4, 0.1)
    with pytest.raises(ValueError):
        top_k_newer([1.0], -1)
    with pytest.raises(ValueError):
        PolicyConfig(recent_len=0)
    st = LayerKV(1, 4)
    st.append(np.zeros((1, 4)), np.zeros((1, 4)), 0)
    st.append(np.zeros((1, 4)), np.zeros((1, 4)), 1)
    with pytest.raises(ValueError):
        st.append(np.zeros((1, 4)), np.zeros((1, 4)), 1)
    with pytest.raises(ValueError):
        st.gather_keep([1, 1])
    with pytest.raises(ValueError):
        st.gather_keep([0, 2])


def test_attend_first_token_unit_row():  # test_engine.py first-token row == [1.0]
    k = np.random.default_rng(0).standard_normal((2, 1, 8)).astype(F32)
    probs, out = attend_heads(k, k, k[:, 0], 1 / np.sqrt(8))
    np.testing.assert_allclose(head_mean(probs), [1.0], atol=1e-7)
    np.testing.assert_allclose(out, k[:, 0], atol=1e-7)


def test_near_tie_rule():
    cfg = PolicyConfig(recent_len=1, relevant_budget=1, bias=0.0)
    s = np.array([0.5, 0.5 * (1 + 1e-7), 0.1], dtype=F32)
    ok, nbad, _ = kept_sets_match(s, np.array([1, 3]), np.array([0, 3]), 4, cfg)
    assert ok and nbad == 2
    s2 = np.array([0.5, 0.6, 0.1], dtype=F32)
    ok, _, _ = kept_sets_match(s2, np.array([1, 3]), np.array([0, 3]), 4, cfg)
    assert not ok
