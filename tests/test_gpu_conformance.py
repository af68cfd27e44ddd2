"""Boundary conformance: the reference's OWN unit tests for the hot-path API
(pkg/tests/test_policies.py, test_cache.py, test_tensorops.py) run against this
package through a `streamkv` shim that maps streamkv.policies / .cache /
.tensorops to the B200 drop-ins.

The tests are vendored (tools/vendor_ref_tests.py) into baseline/_ref/ref_tests,
which is git-ignored but ships to the GPU box; the test skips where that copy
is absent.  They run in a subprocess so their `oracles` module and the shim
never leak into this test session.
"""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "ref_tests")

SHIM = {
    "__init__.py": (
        "from paper_2409_09086_b200 import *  # noqa: F401,F403\n"
        "from paper_2409_09086_b200 import (KvCache, PositionMode, TokenMeta, AttentionWindow, EvictionDecision,\n"
        "    PolicyConfig, bias_vector, heavy_hitter_accumulate, heavy_hitter_decide, inf_mllm_decide,\n"
        "    sink_recent_decide, sliding_window_decide, top_k_indices, window_mean_scores, attn_probs,\n"
        "    rope_apply, softmax_row, weighted_sum)  # noqa: F401\n"
    ),
    "policies.py": "from paper_2409_09086_b200.policies import *  # noqa: F401,F403\n",
    "cache.py": "from paper_2409_09086_b200.cache import *  # noqa: F401,F403\n",
    "tensorops.py": "from paper_2409_09086_b200.tensorops import *  # noqa: F401,F403\n",
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("module", ["test_policies.py", "test_cache.py", "test_tensorops.py"])
def test_reference_unit_tests_pass_on_dropin(module, tmp_path):
    if not os.path.exists(os.path.join(REF_TESTS, module)):
        pytest.skip("reference tests not vendored (python tools/vendor_ref_tests.py)")
    shim = tmp_path / "shim" / "streamkv"
    shim.mkdir(parents=True)
    for name, body in SHIM.items():
        (shim / name).write_text(body)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(tmp_path / "shim"), REF_TESTS, ROOT])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REF_TESTS,
                        os.path.join(REF_TESTS, module)], env=env, cwd=str(tmp_path), capture_output=True,
                       text=True, timeout=1800)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
