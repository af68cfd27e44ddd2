"""Live-session quality metrics (the reference Session's oracle mode,
engine.py:142-151, 275-284, 310-331, 391-451) on the device: OracleSession
against the reference's own metric values (tests/golden/ref_shadow_mini.npz,
made by make_golden.py with the reference's retained_mass / topk_overlap over
a never-evicted shadow cache)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.golden.cases import CASES, case_inputs  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_oracle_session_metrics_match_reference():
    from paper_2409_09086_b200 import EngineConfig
    from paper_2409_09086_b200.session import OracleSession

    name = "shadow_mini"
    c = CASES[name]
    ref = dict(np.load(os.path.join(GOLD, f"ref_{name}.npz")))
    cfg = EngineConfig(c["S"], c["L"], c["Hq"], c["Hkv"], c["D"], c["l"], c["r"], c["b"], c["W"],
                       c["l"] + c["r"] + c["E"], torch.float32)
    sess = OracleSession(cfg, max_tokens=c["T"] + 64)
    q_all, k_all, v_all = case_inputs(name)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    got_mass, got_ov = [], []
    deviations = []
    for t in range(c["T"]):
        sess.decode_step(dev(q_all[t]), dev(k_all[t]), dev(v_all[t]), record=True)
        if (t + 1) % c["E"] == 0:
            sess.evict()
            pl = sess.layer_metrics[-1]
            for s in range(c["S"]):
                for layer in range(c["L"]):
                    got_mass.append(pl[s, layer, 0])
                    got_ov.append(pl[s, layer, 1])
                    deviations.append(sess.attention_equivalence_check(s, layer, q_all[t, layer, s]))
    got_mass, got_ov = np.array(got_mass), np.array(got_ov)
    want_mass, want_ov = ref["shadow_mass"], ref["shadow_overlap"]
    assert got_mass.size == want_mass.size
    # rows come from the device attention (within ~1e-6 of the reference's)
    np.testing.assert_allclose(got_mass, want_mass, rtol=2e-5)
    np.testing.assert_array_equal(np.isnan(got_ov), np.isnan(want_ov))
    # the oracle's top-r may differ only by a near-tie swap of one member
    assert np.nanmax(np.abs(got_ov - want_ov)) <= 1.0 / c["r"] + 1e-12
    assert np.mean(np.nan_to_num(np.abs(got_ov - want_ov))) <= 0.25 / c["r"]
    # compressed-cache attention == masked full-cache attention (f32)
    assert max(deviations) <= 1e-5, max(deviations)
    rows = sess.metrics_rows[-1]
    assert len(rows) == c["S"] and all(r.cache_len == c["l"] + c["r"] for r in rows)
