"""The checked build (liblegend_b200_checked.so: every hot-kernel gather /
scatter index and K4 segment invariant checked on the device, a violation
traps) runs the small workloads of profiles/sanitize_workload.py -- every
model, hub segments, the side-stream long-segment path, shared negatives on
tcgen05, evaluate -- without a trap, and prints the same losses and MRR as the
product build.  (compute-sanitizer is closed on this GPU pool: see
profiles/r02a/compute_sanitizer_refused.txt.)  Runs on a B200 (-m gpu)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2505_09258_b200", "liblegend_b200_checked.so")


def run(mode, lib=None):
    env = dict(os.environ)
    if lib:
        env["LGD_LIBRARY"] = lib
    out = subprocess.run([sys.executable, os.path.join(ROOT, "profiles", "sanitize_workload.py"),
                          mode], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    return out


@pytest.mark.parametrize("mode", ["exact", "shared"])
def test_checked_build_runs_clean_and_agrees(mode):
    if not os.path.exists(CHECKED):
        pytest.fail("liblegend_b200_checked.so missing: run `make -C paper_2505_09258_b200/csrc checked`")
    chk = run(mode, CHECKED)
    assert chk.returncode == 0, (chk.stdout[-2000:], chk.stderr[-2000:])
    assert "LGD_CHECKED" not in chk.stdout + chk.stderr
    plain = run(mode)
    assert plain.returncode == 0, plain.stderr[-2000:]
    assert chk.stdout.splitlines() == plain.stdout.splitlines()
