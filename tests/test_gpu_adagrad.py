"""The certified fast path of the FP64 Adagrad update (csrc/adagrad.cuh) is
bit-identical to the exact reference form (train.cpp:342-354) on 2^28 random
operands spanning first steps (S = 0), tiny and huge gradients and exact
zeros; builds and runs profiles/micro/adagrad_probe.cu (-m gpu)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1])  # 0: two Newton steps, 1: one (the K4 default)
def test_fast_adagrad_matches_exact_form(tmp_path, mode):
    exe = str(tmp_path / "adagrad_probe")
    src = os.path.join(ROOT, "profiles", "micro", "adagrad_probe.cu")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                    "-o", exe, src], check=True)
    out = subprocess.run([exe, str(1 << 28), str(mode)], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    fields = out.stdout.split()
    assert fields[fields.index("mismatches") + 1] == "0", out.stdout
    fast = float(fields[fields.index("fast") + 2].strip("(%)"))
    assert fast > 99.9, out.stdout  # the exact fallback stays rare
