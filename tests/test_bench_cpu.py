"""bench.py plumbing on the CPU: the N-rank self-launch, and the reference
arm's independence from the product library (it must time the unmodified
reference on the same workload, built by the host generator)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_launch_command_is_torchrun_per_gpu():
    cmd = bench.launch_command(["--gpus", "4", "--steps", "3"], 4, 29999)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-port=29999" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.dist_setup(4, init=False)


def test_gpus_2_self_launches_two_ranks_one_line(reference):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                          "reference", "--config", "fb15k", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 prints, rank 1 exits without work
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["batch_size"] == bench.BATCH == 100_000
    assert line["cpu_baseline"]["kind"] == "reference" and line["value"] > 0


def test_reference_arm_never_loads_the_product(reference):
    code = (
        "import sys, json; sys.path.insert(0, %r); import bench\n"
        "w = bench.ref_workload(bench.CONFIGS['fb15k'])\n"
        "r = bench.cpu_sample(bench.CONFIGS['fb15k'], 0, 1, w=w)\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'mods': 'paper_2505_09258_b200' in sys.modules,\n"
        "                  'so': 'liblegend_b200' in maps, 'ref': 'liblegend_ref' in maps,\n"
        "                  'edges': len(w['bucket'])}))\n" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    got = json.loads(out.stdout.strip().splitlines()[-1])
    assert got == {"mods": False, "so": False, "ref": True, "edges": 592_000}
