"""Count fused with a device-side all-reduce over peer memory.

One process per GPU.  The reference's multi-chunk use is chunk-and-merge
(``merge_counts``, proj/core/src/pospop.cpp:33-37; proj/tests/test_core.cpp:155-175):
every shard's k-vector is added element-wise, and the sum is final only once
every partial is in.  Instead of a separate collective after the count:

* the producer is the counting kernel itself: its last CTA stores the rank's
  k counts as row ``rank`` of slot ``step % slots`` in EVERY rank's exchange
  buffer (mapped through CUDA IPC, so the stores travel over NVLink from
  inside the kernel) and release-stores the row's step tag;
* the consumer is a one-CTA reduce kernel on the same stream: it waits on the
  device until all n tags of the step have arrived, writes the row sum (the
  all-reduced counts) and returns the slot's credit;
* before rewriting a slot, a producer waits until every peer has consumed
  the slot's previous step, so a rank running ``slots`` steps ahead cannot
  overwrite rows a slower peer is still reading.

Both waits are bounded (20 s) and report a timeout through the buffer's error
word (``status()``).  Steps are consecutive integers from 0.

    pg, why = PeerGather.create(k=16)           # after torch.distributed init
    pg.allreduce(shard, local, total, step)     # count kernel + reduce kernel
    ...                                         # `total` is final on the device
"""
from __future__ import annotations

from typing import Any

from . import (count_allgather_async, exchange_bytes, exchange_reduce_async, exchange_status, ipc_alloc, ipc_close,
               ipc_free, ipc_open)

HEADER_WORDS = 8  # pospop_exchange.h kXHeader


class _DeviceView:
    """A raw device allocation as a torch tensor (CUDA array interface)."""

    def __init__(self, ptr: int, shape: tuple[int, ...]):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<i8", "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerGather:
    """This rank's exchange buffer, the mapped peer buffers and the device
    table of their pointers.  Build with :meth:`create` (collective-safe)."""

    k: int
    slots: int
    world: int
    rank: int

    @classmethod
    def create(cls, k: int, slots: int = 2, group: Any = None) -> "tuple[PeerGather | None, str]":
        """Collective-safe setup: every rank executes the same collectives
        whatever fails locally, and either all ranks get a PeerGather or all
        get (None, reason) -- a local failure never leaves peers blocked."""
        import torch
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self = cls.__new__(cls)
        self.k, self.slots, self.world, self.rank = int(k), int(slots), world, rank
        self._next_step = 0
        dev = torch.cuda.current_device()
        reason = ""
        self.ptr, handle = 0, None
        try:
            nbytes = exchange_bytes(self.k, world, self.slots)
            if nbytes == 0:
                raise ValueError(f"no exchange layout for k={k}, {world} ranks, {slots} slots")
            self.ptr, handle = ipc_alloc(nbytes)
        except Exception as e:  # noqa: BLE001
            reason = f"ipc_alloc: {e}"
        handles: list = [None] * world
        dist.all_gather_object(handles, handle, group=group)  # every rank, always
        opened: list[int] = []
        ok = all(h is not None for h in handles)
        if ok:
            try:
                for j in range(world):
                    opened.append(self.ptr if j == rank else ipc_open(handles[j]))
            except Exception as e:  # noqa: BLE001
                ok, reason = False, f"ipc_open: {e}"
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) != 1:
            for j, p in enumerate(opened):
                if j != rank:
                    ipc_close(p)
            if self.ptr:
                ipc_free(self.ptr)
            return None, reason or "a peer could not map the exchange buffers"
        self.peer_ptrs = opened
        self.table = torch.tensor(opened, dtype=torch.int64, device=f"cuda:{dev}")
        words = nbytes // 8
        self.buffer = torch.as_tensor(_DeviceView(self.ptr, (words,)), device=f"cuda:{dev}")
        return self, ""

    def _slot(self, step: int) -> int:
        return HEADER_WORDS + (step % self.slots) * (self.world + self.world * self.k)

    def count(self, data: Any, out: Any, step: int, *, stream: Any = None, len_words: int | None = None) -> None:
        """Producer: one kernel counts into `out` and publishes the row of `step` to every GPU."""
        if step != self._next_step:
            raise ValueError(f"exchange steps must be consecutive: expected {self._next_step}, got {step}")
        count_allgather_async(data, out, self.k, self.table, self.world, self.rank, step, self.slots,
                              stream=stream, len_words=len_words)
        self._next_step = step + 1

    def reduce(self, step: int, total: Any, *, stream: Any = None) -> None:
        """Consumer: waits on the device for every rank's row of `step`, total = their sum."""
        exchange_reduce_async(self.k, self.ptr, self.world, step, total, self.slots, stream=stream)

    def allreduce(self, data: Any, local: Any, total: Any, step: int, *, stream: Any = None,
                  len_words: int | None = None) -> None:
        """count + reduce: `local` = this rank's counts, `total` = merge_counts over the ranks."""
        self.count(data, local, step, stream=stream, len_words=len_words)
        self.reduce(step, total, stream=stream)

    def tags(self, step: int):
        o = self._slot(step)
        return self.buffer[o:o + self.world]

    def rows(self, step: int):
        """The n_ranks k-vectors in the slot of `step` (valid once its reduce has run)."""
        o = self._slot(step) + self.world
        return self.buffer[o:o + self.world * self.k].view(self.world, self.k)

    def result(self, step: int):
        """merge_counts over the slot's rows: int64[k] on this GPU."""
        return self.rows(step).sum(dim=0)

    def status(self) -> tuple[int, int]:
        """(steps consumed, error code); raises CudaError if a bounded wait timed out."""
        return exchange_status(self.ptr)

    def close(self) -> None:
        for j, p in enumerate(self.peer_ptrs):
            if j != self.rank:
                ipc_close(p)
        ipc_free(self.ptr)
        self.peer_ptrs = []
