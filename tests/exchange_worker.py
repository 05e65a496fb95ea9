"""Worker for tests/test_gpu_exchange.py (launched by torchrun, gloo backend):
every rank counts its shard with the fused count + peer-memory exchange and
checks the gathered rows and their sum against the oracle."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1911_02696_b200 as pp  # noqa: E402
from paper_1911_02696_b200.exchange import PeerGather  # noqa: E402
import pyoracle  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    orc = pyoracle.Oracle()
    for k, kind in ((16, 4), (64, 6), (8, 3)):
        n_total = 3_000_017
        lo, hi = n_total * rank // world, n_total * (rank + 1) // world
        host = orc.generate(kind, 5, n_total * k // 64 + 1).view(np.uint8)[: n_total * k // 8]
        want_all = orc.pospopcnt(host, k, threads=4)
        mine = host[lo * k // 8: hi * k // 8]
        d = torch.from_numpy(mine.copy()).cuda()
        pg, reason = PeerGather.create(k)
        assert pg is not None, reason
        out = torch.zeros(k, dtype=torch.int64, device="cuda")
        for step in range(3):  # slots 0, 1, 0: a slot is rewritten in place
            pg.count(d, out, step)
            torch.cuda.synchronize()
            dist.barrier()
            rows = pg.rows(step).cpu().numpy().astype(np.uint64)
            assert (rows[rank] == out.cpu().numpy().astype(np.uint64)).all()
            assert (rows[rank] == orc.pospopcnt(mine, k, threads=2)).all()
            assert (pg.result(step).cpu().numpy().astype(np.uint64) == want_all).all(), (k, step, rank)
            dist.barrier()
        pg.close()
    # A local failure on one rank (here: rank 1 cannot map a peer) must make
    # every rank fall back together, with no collective left waiting.
    import paper_1911_02696_b200.exchange as ex
    real_open = ex.ipc_open

    def failing_open(h):
        if rank == 1:
            raise RuntimeError("injected ipc_open failure")
        return real_open(h)
    ex.ipc_open = failing_open
    pg, reason = PeerGather.create(16)
    ex.ipc_open = real_open
    assert pg is None and reason, (rank, reason)
    pg, reason = PeerGather.create(16)  # and a clean retry still works
    assert pg is not None, reason
    pg.close()
    dist.barrier()
    if rank == 0:
        print("exchange ok", world)


if __name__ == "__main__":
    main()
