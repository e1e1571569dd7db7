"""Multi-GPU parity (G = 2 / 3 / 4 / 8): one torchrun process per GPU running tests/mgpu_worker.py.

A case runs only when the box has at least G GPUs: the layer kernels spin on flags their
peers' kernels raise, so two ranks must never share one GPU.  The 8-rank host logic
(layouts, route tables, migration rounds) is covered on CPU by tests/test_dist_gloo.py."""

import socket
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

REPO = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_multi_gpu_layer_matches_oracle(G):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs, have {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "tests" / "mgpu_worker.py")]
    res = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    sys.stdout.write(res.stdout[-4000:])
    sys.stderr.write(res.stderr[-8000:])
    assert res.returncode == 0
    assert f"mgpu ok: G={G}" in res.stdout


@pytest.mark.parametrize("G,config,steps", [(2, "toy", 4000), (4, "deepseek", 2000)])
def test_flag_protocol_soak(G, config, steps):
    """Thousands of back-to-back forwards at G > 1 (tools/soak.py): between chunks every rank's
    protocol state (mp_layer_sync_state) must show one epoch, all flags equal to it, arrival
    tickets and the router accumulator at zero and no timeout bits."""
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs, have {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "tools" / "soak.py"),
           "--gpus", str(G), "--config", config, "--steps", str(steps), "--warmup", "3", "--chunk=500"]
    res = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600)
    sys.stdout.write(res.stdout[-2000:])
    sys.stderr.write(res.stderr[-4000:])
    assert res.returncode == 0
    assert '"ok": true' in res.stdout


def test_multi_gpu_tail_split_plan_matches_oracle():
    """The opt-in tail split (MP_GEMM_TAILS: big groups' short CTA-pair tails on the side chain)
    through the same G = 2 cases, production split plans included."""
    G = 2
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs, have {torch.cuda.device_count()}")
    import os
    env = dict(os.environ, MP_GEMM_TAILS="128")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "tests" / "mgpu_worker.py")]
    res = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900, env=env)
    sys.stdout.write(res.stdout[-4000:])
    sys.stderr.write(res.stderr[-8000:])
    assert res.returncode == 0
    assert f"mgpu ok: G={G}" in res.stdout


def test_lost_peer_fails_loudly_without_trap():
    """A rank that stops calling forward: its peer's waits time out (bounded once per wait, no
    kernel trap), check() names the lost rank and the next forward refuses to launch."""
    G = 2
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs, have {torch.cuda.device_count()}")
    import os
    env = dict(os.environ, MP_PEER_TIMEOUT_MS="2000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "tests" / "mgpu_lost_peer.py")]
    res = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=300, env=env)
    sys.stdout.write(res.stdout[-2000:])
    sys.stderr.write(res.stderr[-4000:])
    assert res.returncode == 0
    assert "lost-peer ok" in res.stdout
