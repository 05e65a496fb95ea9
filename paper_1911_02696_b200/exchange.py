"""Count fused with the cross-GPU exchange over peer memory.

One process per GPU.  The reference's multi-chunk use is chunk-and-merge
(``merge_counts``, proj/core/src/pospop.cpp:33-37; proj/tests/test_core.cpp:155-175):
every shard's k-vector is added element-wise.  Instead of a separate
collective after the count, every rank's counting kernel delivers its
k-vector itself: its last CTA stores the k counts into row ``rank`` of a gather
slot that lives in EVERY rank's memory (mapped through CUDA IPC, so the stores
travel over NVLink from inside the kernel).  Once all ranks' launches of a step
have completed, each GPU holds all n k-vectors of that step and the
all-reduced counts are the slot's row sum -- no NCCL kernel, no extra launch,
no kernel waiting on another rank.

    pg = PeerGather(k=16)                       # after torch.distributed init
    pg.count(shard, out, step)                  # one kernel: count + deliver
    ...                                         # (all ranks' launches complete)
    total = pg.result(step)                     # int64[k] on this GPU
"""
from __future__ import annotations

from typing import Any

from . import count_allgather_async, ipc_alloc, ipc_close, ipc_free, ipc_open


class _DeviceView:
    """A raw device allocation as a torch tensor (CUDA array interface)."""

    def __init__(self, ptr: int, shape: tuple[int, ...]):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<i8", "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerGather:
    """Gather slots in every rank's memory plus the per-slot device tables of
    peer pointers.  ``slots`` >= 2 lets step i+1 run while step i is read."""

    def __init__(self, k: int, slots: int = 2, group: Any = None):
        import torch
        import torch.distributed as dist

        self.k, self.slots = int(k), int(slots)
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        row_bytes = self.k * 8
        self._slot_bytes = self.world * row_bytes
        self.ptr, handle = ipc_alloc(self.slots * self._slot_bytes)
        handles: list = [None] * self.world
        dist.all_gather_object(handles, handle, group=group)
        self.peer_ptrs = [self.ptr if j == self.rank else ipc_open(handles[j]) for j in range(self.world)]
        dev = torch.cuda.current_device()
        self.tables = [torch.tensor([p + s * self._slot_bytes for p in self.peer_ptrs], dtype=torch.int64,
                                    device=f"cuda:{dev}") for s in range(self.slots)]
        self.buffer = torch.as_tensor(_DeviceView(self.ptr, (self.slots, self.world, self.k)), device=f"cuda:{dev}")

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
        self._slot_bytes = world * self.k * 8
        dev = torch.cuda.current_device()
        reason = ""
        try:
            self.ptr, handle = ipc_alloc(self.slots * self._slot_bytes)
        except Exception as e:  # noqa: BLE001
            self.ptr, handle, reason = 0, None, f"ipc_alloc: {e}"
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
            return None, reason or "a peer could not map the gather buffers"
        self.peer_ptrs = opened
        self.tables = [torch.tensor([p + s * self._slot_bytes for p in opened], dtype=torch.int64,
                                    device=f"cuda:{dev}") for s in range(self.slots)]
        self.buffer = torch.as_tensor(_DeviceView(self.ptr, (self.slots, world, self.k)), device=f"cuda:{dev}")
        return self, ""

    def count(self, data: Any, out: Any, step: int, *, stream: Any = None, len_words: int | None = None) -> None:
        """One kernel: this rank's counts into `out` and into row `rank` of slot step % slots on every GPU."""
        count_allgather_async(data, out, self.k, self.tables[step % self.slots], self.world, self.rank,
                              stream=stream, len_words=len_words)

    def rows(self, step: int):
        """The n_ranks k-vectors of a step (valid once every rank's launch completed)."""
        return self.buffer[step % self.slots]

    def result(self, step: int):
        """merge_counts over the ranks: int64[k] on this GPU."""
        return self.rows(step).sum(dim=0)

    def close(self) -> None:
        for j, p in enumerate(self.peer_ptrs):
            if j != self.rank:
                ipc_close(p)
        ipc_free(self.ptr)
        self.peer_ptrs = []
