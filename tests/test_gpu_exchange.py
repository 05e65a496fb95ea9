"""The fused count + device all-reduce over peer memory (paper_1911_02696_b200.exchange).

* Two and three ranks (torchrun, gloo for the handle exchange) on one GPU, a
  different seed every step and more steps than slots; every step's
  on-device total must equal the oracle.  The ranks share the GPU, so each
  phase is separated by a host barrier and no kernel waits on a rank that
  has not finished (B200_PROFILING.md: kernels of different processes that
  wait on one another raised Xid 109 on this driver).
* The unsynchronised protocol -- no host synchronisation at all, ranks
  pushed steps apart -- runs as n blocks of ONE cooperative launch
  (pospop_exchange_selftest), the safe way to run waiting ranks on one GPU."""
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


@pytest.mark.parametrize("n,slots", [(1, 1), (2, 2), (3, 2), (8, 2), (8, 3), (5, 1)])
def test_exchange_protocol_unsynchronised(n, slots):
    """The step-tag + credit protocol with no host synchronisation at all: n
    blocks of ONE cooperative launch play the n ranks (the only safe way to run
    ranks that wait on one another on one GPU), with the device functions of
    the counting kernel's producer and the reduce kernel.  Random device sleeps
    push ranks up to several steps apart; every rank's total of every step
    must equal the sum of that step's rows (a stale row, a row overwritten by a
    rank ahead, or a reduce that ran early would change it)."""
    import ctypes as C

    import numpy as np

    import paper_1911_02696_b200 as pp
    lib = pp._load()
    steps, k = 24, 16
    rng = np.random.default_rng(n * 10 + slots)
    inputs = rng.integers(0, 1 << 40, size=(steps, n, k), dtype=np.uint64)
    sleeps = np.where(rng.random((steps, n)) < 0.3, rng.integers(1_000, 300_000, size=(steps, n)), 0).astype(np.uint32)
    totals = np.zeros((n, steps, k), np.uint64)
    u64p = C.POINTER(C.c_uint64)
    lib.pospop_exchange_selftest.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, u64p, C.POINTER(C.c_uint32), u64p]
    rc = lib.pospop_exchange_selftest(k, n, slots, steps, inputs.ctypes.data_as(u64p),
                                      sleeps.ctypes.data_as(C.POINTER(C.c_uint32)), totals.ctypes.data_as(u64p))
    assert rc == 0, lib.pospop_last_error()
    want = inputs.sum(axis=1, dtype=np.uint64)
    for r in range(n):
        assert (totals[r] == want).all(), r


def test_exchange_single_rank_real_kernels():
    """One rank, the real kernels: count + publish, then the reduce kernel,
    for more steps than slots with a new input every step and no host
    synchronisation; the slot's credit is this rank's own reducer."""
    import numpy as np
    import torch

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import paper_1911_02696_b200 as pp
    import pyoracle
    orc = pyoracle.Oracle()
    torch.cuda.set_device(0)
    k, steps, n_words = 16, 7, 1_234_567
    ptr, _ = pp.ipc_alloc(pp.exchange_bytes(k, 1, 2))
    table = torch.tensor([ptr], dtype=torch.int64, device="cuda")
    data = [torch.empty(n_words * 2, dtype=torch.uint8, device="cuda") for _ in range(steps)]
    for st, d in enumerate(data):
        pp.generate(pp.GEN_CFG4, 50 + st, d)
    torch.cuda.synchronize()
    local = torch.zeros((steps, k), dtype=torch.int64, device="cuda")
    total = torch.full((steps, k), -1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    for st in range(steps):
        pp.count_allgather_async(data[st], local[st], k, table, 1, 0, st, 2, stream=s)
        pp.exchange_reduce_async(k, ptr, 1, st, total[st], 2, stream=s)
    s.synchronize()
    assert pp.exchange_status(ptr) == (steps, 0)
    for st in range(steps):
        want = orc.pospopcnt(orc.generate(pp.GEN_CFG4, 50 + st, n_words), 16, threads=4)
        assert (total[st].cpu().numpy().astype(np.uint64) == want).all(), st
        assert torch.equal(local[st], total[st])
    pp.ipc_free(ptr)
