"""bench.py's driver contract on CPU: the entry points exist, and `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run (127.0.0.1 rendezvous)."""

import importlib.util
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", REPO / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_bench_defines_every_scenario_entry():
    b = _bench()
    for name in ("main_b200", "main_reference", "main_shift", "main_stack", "main_transport", "main_calibrate",
                 "self_launch", "setup_bench_layer", "measure_peer_copy", "measure_peer_latency", "cpu_threads",
                 "time_reference_package"):
        assert callable(getattr(b, name)), name


def test_self_launch_reexecs_under_torchrun(monkeypatch):
    b = _bench()
    seen = {}

    class Done:
        returncode = 0

    def fake_run(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return Done()

    monkeypatch.setattr(b.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    args = b.parse()
    assert b.self_launch(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")
