"""The fused count + peer-memory exchange (paper_1911_02696_b200.exchange):
two and three ranks (torchrun, gloo for the handle exchange) on one GPU --
each rank's kernel stores its k-vector into every rank's gather slot; the rows
and their sum must equal the oracle.  No kernel waits on another rank, so
sharing one GPU is safe."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_peer_gather_matches_oracle(world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "exchange_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "exchange ok" in r.stdout
