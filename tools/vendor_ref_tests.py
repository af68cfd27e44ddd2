#!/usr/bin/env python
"""Copy the reference's own unit tests for the hot-path API into
baseline/_ref/ref_tests/ (git-ignored, NOT gpurun-ignored: it travels to the
GPU box, where /root/reference does not exist).  tests/test_gpu_conformance.py
runs them against this package through a `streamkv` shim.

Run in the dev container:  python tools/vendor_ref_tests.py
"""

import os
import shutil

REF = "/root/reference/pkg/tests"
FILES = ["test_policies.py", "test_cache.py", "test_tensorops.py", "oracles.py"]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "baseline", "_ref", "ref_tests")


def main():
    os.makedirs(DST, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(REF, f), os.path.join(DST, f))
    print(f"vendored {len(FILES)} files into {DST}")


if __name__ == "__main__":
    main()
