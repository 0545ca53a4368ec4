"""bench.py's host-side launch logic (CPU): --gpus N without torchrun re-executes under
torch.distributed.run with N ranks on 127.0.0.1; inside a rank (WORLD_SIZE set) or at N = 1 it
does not."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    d = dict(gpus=1, impl="ours")
    d.update(kw)
    return argparse.Namespace(**d)


def test_launch_cmd_shape():
    cmd = bench.launch_cmd(["--gpus", "8", "--steps", "3"], 8, 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "3"]
    assert os.path.samefile(cmd[-5], os.path.join(ROOT, "bench.py"))


def test_self_launch_only_outside_a_launcher(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.self_launch(_args(gpus=1)) is None
    assert bench.self_launch(_args(gpus=4, impl="reference")) is None   # rank 0 alone does the work
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.self_launch(_args(gpus=4)) is None                     # already a rank


def test_self_launch_spawns_n_ranks(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    class R:
        returncode = 0

    def fake_run(cmd, cwd=None):
        seen["cmd"] = cmd
        return R()

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "4"])
    assert bench.self_launch(_args(gpus=2)) == 0
    assert "--nproc-per-node=2" in seen["cmd"] and seen["cmd"][-4:] == ["--gpus", "2", "--steps", "4"]
