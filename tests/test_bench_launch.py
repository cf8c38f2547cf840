"""bench.py --gpus N launches N ranks by itself.

CPU tests: the launcher's command line, the refusal of N > visible GPUs,
and a real two-process run of the reference arm through the self-launch
(torchrun over 127.0.0.1; rank 0 prints the one JSON line, rank 1 exits 0).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_launch_command_shape():
    import bench
    cmd = bench.launch_command(4, ["--gpus", "4", "--steps", "3"], 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    assert Path(cmd[-5]).name == "bench.py"


def test_self_launch_refuses_more_gpus_than_visible(monkeypatch):
    import bench
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.delenv("LBM_B200_BACKEND", raising=False)
    args = bench.parse_args(["--gpus", "64"])
    with pytest.raises(SystemExit, match="CUDA device"):
        bench.self_launch(args, ["--gpus", "64"])


def test_self_launch_is_a_noop_under_a_launcher(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.self_launch(bench.parse_args(["--gpus", "2"]), []) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.self_launch(bench.parse_args(["--gpus", "1"]), []) is None


def test_two_rank_self_launch_reference_arm():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "2"
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "c0", "--steps", "2", "--warmup", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "torch.distributed.run" in res.stderr
