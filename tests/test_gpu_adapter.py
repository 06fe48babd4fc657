"""The reference-signature adapter (adapters/legend_reference_adapter.hpp):
legend_b200::run_epoch / evaluate with the reference's own types, built
against the reference headers by oracle/Makefile (target adapter, where the
reference sources exist) and run here: the reference's drop-in check
(test_pipeline.cpp:197-289, out-of-core epoch == in-memory restatement on the
unmodified reference primitives) with the B200 run_epoch in place of the
reference's, for DistMult / ComplEx / Dot, plus evaluate == legend::evaluate.
Runs on a B200 (-m gpu)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


def test_adapter_passes_the_reference_epoch_check():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/adapter_test not built (needs the reference sources)")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "adapter ok" in out.stdout
    assert out.stdout.count("adapter ") >= 4
