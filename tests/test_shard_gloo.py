"""The N > 1 shard/reduce path, exercised with world_size 2 on CPU (gloo).

Each rank takes its contiguous shard (shard_range), counts it with an
injected counter (the oracle here; the GPU kernel in the product), and the
k-vector all-reduce must give exactly the single-process counts -- the
fork-join / merge_counts property of proj/tests/test_core.cpp:143-175."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, k, total, result_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch.distributed as dist

    import pyoracle
    from paper_1911_02696_b200.shard import shard_range, sharded_pospopcnt

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = pyoracle.Oracle()
    lo, hi = shard_range(total, rank, world)
    kind = {8: 3, 16: 4, 32: 5, 64: 6}[k]
    local = orc.generate(kind, 1, hi - lo, base=lo)  # in-place shard generation
    got = sharded_pospopcnt(local, k, counter=lambda a, kk: orc.pospopcnt(a, kk))
    result_q.put((rank, got.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("k,total", [(16, 1_000_003), (8, 777_777), (32, 100_001), (64, 54_321)])
def test_two_rank_shard_reduce_equals_whole(orc, k, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, k, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    kind = {8: 3, 16: 4, 32: 5, 64: 6}[k]
    whole = orc.naive(orc.generate(kind, 1, total), k)
    assert results[0] == results[1] == [int(x) for x in whole]


def test_shard_range_partitions():
    from paper_1911_02696_b200.shard import shard_range
    for total in (0, 1, 7, 2**32, 2**32 + 5):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
