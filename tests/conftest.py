import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def _ensure_oracle():
    from oracle.oracle import PATHS
    if not os.path.exists(PATHS["restatement"]):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "restatement"])


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (test-only checker)."""
    _ensure_oracle()
    from oracle.oracle import Oracle
    return Oracle("restatement")


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library, when it was built here."""
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Oracle("reference")
