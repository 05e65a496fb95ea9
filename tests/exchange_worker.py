"""Worker for tests/test_gpu_exchange.py (launched by torchrun, gloo for the
handle exchange): every rank counts its shard with the fused count + device
all-reduce over peer memory (producer rows with step tags, a reduce kernel
that sums them, credit before a slot is reused), a different seed every step
and more steps than slots.  The ranks share ONE GPU, so no kernel may wait on
work another rank has not finished (B200_PROFILING.md): each phase is
separated by a host barrier, which leaves every device wait already
satisfied when its kernel starts.  (The unsynchronised protocol is exercised
by pospop_exchange_selftest: all ranks in one cooperative launch.)  Each
step's on-device total is checked against the oracle."""
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

STEPS = 9


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    orc = pyoracle.Oracle()
    s = torch.cuda.Stream()
    for k, kind in ((16, 4), (64, 6), (8, 3)):
        wb = k // 8
        n_total = 3_000_017 if k != 64 else 1_000_003
        lo, hi = n_total * rank // world, n_total * (rank + 1) // world
        # per-step inputs, generated up front (seed 1000 + step)
        shards = []
        for step in range(STEPS):
            d = torch.empty((hi - lo) * wb + 64, dtype=torch.uint8, device="cuda")
            pp.generate(kind, 1000 + step, d, base=lo, n=hi - lo)
            shards.append(d[: (hi - lo) * wb])
        torch.cuda.synchronize()
        pg, reason = PeerGather.create(k, slots=2)
        assert pg is not None, reason
        local = torch.zeros((STEPS, k), dtype=torch.int64, device="cuda")
        total = torch.full((STEPS, k), -1, dtype=torch.int64, device="cuda")
        dist.barrier()
        for step in range(STEPS):
            pg.count(shards[step], local[step], step, stream=s)  # credit already returned (barrier below)
            s.synchronize()
            dist.barrier()  # every rank's row of `step` is in every buffer
            pg.reduce(step, total[step], stream=s)
            s.synchronize()
            dist.barrier()  # every rank has consumed `step`
        consumed, err = pg.status()
        assert err == 0 and consumed == STEPS, (consumed, err)
        for step in range(STEPS):
            host = orc.generate(kind, 1000 + step, n_total).view(np.uint8)
            want_all = orc.pospopcnt(host, k, threads=4)
            mine = host[lo * wb: hi * wb]
            assert (local[step].cpu().numpy().astype(np.uint64) == orc.pospopcnt(mine, k, threads=2)).all(), \
                (k, step, rank)
            assert (total[step].cpu().numpy().astype(np.uint64) == want_all).all(), (k, step, rank)
        # the slot of the last step still holds every rank's row of that step
        last = STEPS - 1
        assert (pg.tags(last).cpu().numpy() == last + 1).all()
        assert torch.equal(pg.result(last), total[last])
        dist.barrier()
        pg.close()
    with pytest_raises(ValueError):  # steps must be consecutive
        pg2, _ = PeerGather.create(16)
        d = torch.zeros(64, dtype=torch.uint8, device="cuda")
        o = torch.zeros(16, dtype=torch.int64, device="cuda")
        try:
            pg2.count(d, o, 1)
        finally:
            pg2.close()
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


class pytest_raises:  # noqa: N801 -- tiny stand-in (no pytest inside torchrun workers)
    def __init__(self, exc):
        self.exc = exc

    def __enter__(self):
        return self

    def __exit__(self, tp, val, tb):
        assert tp is not None and issubclass(tp, self.exc), f"expected {self.exc.__name__}"
        return True


if __name__ == "__main__":
    main()
