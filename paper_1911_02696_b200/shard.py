"""Shard/reduce driver: one process per B200, contiguous shards, one k-vector all-reduce.

The reference's only parallel form is fork-join over contiguous chunks combined
with merge_counts (proj/tests/test_core.cpp:155-175); the
concatenation homomorphism pospopcnt(a ++ b) = merge_counts(pospopcnt(a),
pospopcnt(b)) makes every shard independent.  On an 8-GPU NVSwitch box that
becomes: rank r owns words [r*N/G, (r+1)*N/G) resident in its own HBM, counts
them with ONE kernel launch, and the k-entry u64 vector (128 B for k=16) is
summed with ONE all-reduce (NCCL over NVLink; integer sums are exact and
order-free, so every rank ends with the bit-exact total).

``counter`` is injectable (the analogue of the reference's KernelRunner,
proj/core/include/pospop/verify.hpp:47) so the host logic can be exercised with
the gloo backend on CPU; the product path leaves it as None, which counts on
the rank's GPU through the C ABI.
"""
from __future__ import annotations

from typing import Any, Callable, Optional

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, near-equal shard [lo, hi) of `total` words for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError(f"bad shard request total={total} rank={rank} world={world}")
    return total * rank // world, total * (rank + 1) // world


def sharded_pospopcnt(local: Any, k: int, *, group: Any = None,
                      counter: Optional[Callable[[Any, int], Any]] = None,
                      stream: Any = None):
    """Counts this rank's shard and sums the k-vector over the process group.

    Returns the global counts as a numpy uint64 array of length k on every rank.
    """
    import torch
    import torch.distributed as dist

    if counter is None:
        from . import count_async
        dev = local.device
        out = torch.zeros(k, dtype=torch.int64, device=dev)
        count_async(local, out, k, stream=stream)
    else:
        out = torch.as_tensor(np.asarray(counter(local, k), dtype=np.uint64).astype(np.int64))
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out.cpu().numpy().astype(np.uint64)
