"""Multi-GPU parity (G = 2 / 3 / 4 / 8): one torchrun process per rank running tests/mgpu_worker.py.

G = 8 also runs on a 4-GPU box with two ranks per GPU (co-resident processes time-slice
the GPU): it checks the 8-rank flag protocol, layouts and migration, not speed."""

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
    need = 4 if G == 8 else G
    if torch.cuda.device_count() < need:
        pytest.skip(f"needs {need} GPUs, have {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(REPO / "tests" / "mgpu_worker.py")]
    res = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    sys.stdout.write(res.stdout[-4000:])
    sys.stderr.write(res.stderr[-8000:])
    assert res.returncode == 0
    assert f"mgpu ok: G={G}" in res.stdout
