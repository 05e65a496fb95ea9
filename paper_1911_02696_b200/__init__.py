"""B200-native positional population count (pospopcnt).

Host-side mirror of the reference's public API
(/root/reference/proj/core/include/pospop/types.hpp, pospop.hpp) over the
C ABI in include/pospopcnt_b200.h, implemented by the sm_100a CUDA library
``libpospopcnt_b200.so`` built in-tree from ``csrc/``.

Reference name              -> here
  pospop::pospopcnt            pospopcnt(words, config=None)       (pospop.hpp:34)
  pospop::PositionalCounts     PositionalCounts                    (types.hpp:35-46)
  pospop::merge_counts         merge_counts(a, b)                  (types.hpp:48-50)
  pospop::KernelKind           KernelKind                          (types.hpp:52-60)
  pospop::PospopcntConfig      PospopcntConfig                     (types.hpp:73-89)
  pospop::validate             validate(config)                    (pospop.cpp:63-70)
  pospop::KernelUnavailableError  KernelUnavailableError           (types.hpp:68-71)
  std::invalid_argument        InvalidArgument (a ValueError)
  supported_csa_widths / native_csa_width                          (cpu.cpp:39-55)

Extensions on the same path (BASELINE.json north_star): k = 8/16/32/64
(``pospopcnt_k``), the segmented/batched form (``pospopcnt_segmented``), a
device-resident asynchronous launch (``count_async``), CUDA-graph replay
(``CountGraph``), the fused FLAG statistics (``flagstats``), file/pipe
ingestion (``pospopcnt_file``), the multi-GPU shard/reduce driver
(``paper_1911_02696_b200.shard``) and the count fused with the cross-GPU
exchange over peer memory (``paper_1911_02696_b200.exchange``).

There is no CPU fallback: if the CUDA library or an sm_100 device is missing
every counting call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass
from typing import Any, Iterable, Sequence

import numpy as np

__all__ = [
    "KernelKind", "PospopcntConfig", "PositionalCounts", "InvalidArgument", "KernelUnavailableError",
    "CudaError", "validate", "merge_counts", "pospopcnt", "pospopcnt_k", "pospopcnt_u16_c32",
    "pospopcnt_segmented", "pospopcnt_segmented_split", "pospopcnt_sharded", "pospopcnt_split", "release_resources", "release_stream",
    "resource_stats", "count_async", "segmented_async", "count_allgather_async",
    "exchange_bytes", "exchange_reduce_async", "exchange_status",
    "ipc_alloc", "ipc_open", "ipc_close", "ipc_free", "generate", "digest",
    "supported_csa_widths", "native_csa_width", "device_available", "kernel_launches", "library_path",
    "FlagBucket", "FlagSummary", "InvalidFlagWordError", "flagstats", "pospopcnt_file",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libpospopcnt_b200.so"


BUILDS = {
    "release": "libpospopcnt_b200.so",         # production kernels only; reads no tuning knobs
    "tuning": "libpospopcnt_b200_tuning.so",   # every measured variant + the POSPOP_* tuning knobs
    "debug": "libpospopcnt_b200_debug.so",     # the tuning build with bounds-checked vector loads
}


def library_path(build: str | None = None) -> str:
    """The in-tree library.  `build` (or POSPOP_LIBRARY: a build name or a
    path) selects another build of it: "tuning" for tools/ sweeps and the
    tuning tests, "debug" for tests/test_gpu_bounds.py."""
    sel = build or os.environ.get("POSPOP_LIBRARY") or "release"
    if sel in BUILDS:
        return os.path.join(_HERE, BUILDS[sel])
    return sel


# -- errors (status codes of include/pospopcnt_b200.h) -----------------------

class InvalidArgument(ValueError):
    """std::invalid_argument from pospop::validate / the dispatcher (pospop.cpp:63-70, 110)."""


class KernelUnavailableError(RuntimeError):
    """pospop::KernelUnavailableError (types.hpp:68-71): kernel/width/device cannot run here."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the library."""


class InvalidFlagWordError(RuntimeError):
    """pospop::InvalidFlagWordError (flagstats.hpp:64-75): a FLAG word with bits 12-15 set."""

    def __init__(self, offset: int, word: int, msg: str = ""):
        super().__init__(msg or f"invalid FLAG word 0x{word:x} at offset {offset} (bits 12-15 must be clear)")
        self.offset = offset
        self.word = word


_OK, _EINVAL, _EUNAVAILABLE, _ECUDA, _ENOMEM, _EFLAG = range(6)

_u64p = C.POINTER(C.c_uint64)


_BUCKET_FIELDS = ("total", "secondary", "supplementary", "n_pair_good", "n_read1", "n_read2", "n_sgltn",
                  "pair_map", "mapped", "dup")


class _Bucket(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in _BUCKET_FIELDS]


class _Summary(C.Structure):
    _fields_ = [("pass_", _Bucket), ("fail", _Bucket)]


class _Config(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("register_width_bits", C.c_uint32),
                ("flush_threshold_blocks", C.c_uint32), ("auto_threshold_words", C.c_uint64)]


_lib = None


_libs: dict = {}


def _load():
    global _lib
    if _lib is None:
        _lib = load_library(library_path())
    return _lib


def load_library(path: str):
    """ctypes handle of one build of the library with every signature set
    (cached per path).  The package's functions call the handle in
    `paper_1911_02696_b200._lib` (the release build unless POSPOP_LIBRARY
    says otherwise; tests/conftest.py's `tuning` fixture swaps it)."""
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "or `make -C paper_1911_02696_b200/csrc` (there is no CPU fallback)")
    lib = C.CDLL(path)
    vp, sz = C.c_void_p, C.c_size_t
    sig = {
        "pospop_validate": ([C.POINTER(_Config)], C.c_int),
        "pospop_supported_widths": ([C.POINTER(C.c_uint32), C.c_int], C.c_int),
        "pospop_device_available": ([], C.c_int),
        "pospop_last_error": ([], C.c_char_p),
        "pospop_kernel_launches": ([], C.c_uint64),
        "pospopcnt_u8": ([vp, sz, _u64p], C.c_int),
        "pospopcnt_u16": ([vp, sz, _u64p], C.c_int),
        "pospopcnt_u32": ([vp, sz, _u64p], C.c_int),
        "pospopcnt_u64": ([vp, sz, _u64p], C.c_int),
        "pospopcnt_u16_config": ([vp, sz, C.POINTER(_Config), _u64p], C.c_int),
        "pospopcnt_k": ([C.c_int, vp, sz, C.c_uint32, _u64p], C.c_int),
        "pospopcnt_u16_c32": ([vp, C.c_uint32, C.POINTER(C.c_uint32)], C.c_int),
        "pospopcnt_segmented": ([C.c_int, vp, vp, sz, vp], C.c_int),
        "pospopcnt_sharded": ([C.c_int, C.POINTER(vp), C.POINTER(sz), C.POINTER(C.c_int), C.c_int, _u64p],
                              C.c_int),
        "pospopcnt_async": ([C.c_int, vp, sz, vp, C.c_int, C.c_uint32, C.c_int, C.c_int, vp], C.c_int),
        "pospopcnt_segmented_async": ([C.c_int, vp, vp, sz, vp, C.c_uint32, C.c_int, C.c_int, vp], C.c_int),
        "pospop_generate": ([C.c_int, C.c_uint64, C.c_uint64, sz, vp, vp], C.c_int),
        "pospop_digest": ([vp, sz, _u64p], C.c_int),
        "pospop_flagstats": ([vp, sz, C.POINTER(_Summary), _u64p, C.POINTER(C.c_uint16)], C.c_int),
        "pospopcnt_fd": ([C.c_int, C.c_int, _u64p, _u64p], C.c_int),
        "pospop_microop": ([C.c_int, C.c_int, vp, sz, vp, sz], C.c_int),
        "pospopcnt_graph_create": ([C.c_int, vp, sz, vp, C.POINTER(vp)], C.c_int),
        "pospopcnt_graph_launch": ([vp, vp], C.c_int),
        "pospopcnt_graph_destroy": ([vp], None),
        "pospopcnt_file": ([C.c_char_p, C.c_int, _u64p, _u64p], C.c_int),
        "pospop_ipc_alloc": ([sz, C.POINTER(vp), C.POINTER(C.c_ubyte)], C.c_int),
        "pospop_ipc_open": ([C.POINTER(C.c_ubyte), C.POINTER(vp)], C.c_int),
        "pospop_ipc_close": ([vp], C.c_int),
        "pospop_ipc_free": ([vp], C.c_int),
        "pospop_exchange_bytes": ([C.c_int, C.c_int, C.c_int], sz),
        "pospopcnt_allgather_async": ([C.c_int, vp, sz, vp, vp, C.c_int, C.c_int, C.c_uint64, C.c_int, vp], C.c_int),
        "pospop_exchange_reduce_async": ([C.c_int, vp, C.c_int, C.c_uint64, C.c_int, vp, vp], C.c_int),
        "pospop_exchange_status": ([vp, _u64p, _u64p], C.c_int),
        "pospopcnt_split": ([C.c_int, vp, sz, C.POINTER(C.c_int), C.c_int, _u64p], C.c_int),
        "pospopcnt_segmented_split": ([C.c_int, vp, vp, sz, C.POINTER(C.c_int), C.c_int, vp], C.c_int),
        "pospop_release_resources": ([], C.c_int),
        "pospop_release_stream": ([vp], C.c_int),
        "pospop_resource_stats": ([C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _libs[path] = lib
    return lib


def _check(status: int) -> None:
    if status == _OK:
        return
    msg = _load().pospop_last_error().decode(errors="replace")
    if status == _EINVAL:
        raise InvalidArgument(msg)
    if status == _EUNAVAILABLE:
        raise KernelUnavailableError(msg)
    if status == _ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg)


# -- reference types -----------------------------------------------------------

class KernelKind(enum.IntEnum):
    """pospop::KernelKind (types.hpp:52-60).  All kinds give identical counts."""
    ScalarBasic = 0
    Csa4 = 1
    Csa8 = 2
    Csa16 = 3
    Forest = 4
    ByteBlend = 5
    Auto = 6

    def __str__(self) -> str:  # to_string (pospop.cpp:39-50)
        return _KIND_NAMES[self]

    @classmethod
    def from_string(cls, name: str) -> "KernelKind | None":  # kernel_from_string (pospop.cpp:52-61)
        for k, v in _KIND_NAMES.items():
            if v == name:
                return k
        return None


_KIND_NAMES = {KernelKind.ScalarBasic: "scalar", KernelKind.Csa4: "csa4", KernelKind.Csa8: "csa8",
               KernelKind.Csa16: "csa16", KernelKind.Forest: "forest", KernelKind.ByteBlend: "byteblend",
               KernelKind.Auto: "auto"}


@dataclass
class PospopcntConfig:
    """pospop::PospopcntConfig (types.hpp:73-89), same defaults."""
    kernel: KernelKind = KernelKind.Auto
    register_width_bits: int = 0
    flush_threshold_blocks: int = 65535
    auto_threshold_words: int = 4096

    def _c(self) -> _Config:
        return _Config(int(self.kernel), int(self.register_width_bits) & 0xFFFFFFFF,
                       int(self.flush_threshold_blocks) & 0xFFFFFFFF, int(self.auto_threshold_words))


class PositionalCounts:
    """pospop::PositionalCounts (types.hpp:35-46): counts[p] = #words with bit p set."""

    __slots__ = ("counts",)

    def __init__(self, counts: Iterable[int] | None = None, k: int = 16):
        self.counts = np.zeros(k, np.uint64) if counts is None else np.asarray(counts, np.uint64).copy()

    def __getitem__(self, p: int) -> int:
        return int(self.counts[p])

    def __setitem__(self, p: int, v: int) -> None:
        self.counts[p] = v

    def __len__(self) -> int:
        return len(self.counts)

    def __iter__(self):
        return (int(x) for x in self.counts)

    def __eq__(self, other: Any) -> bool:
        other_counts = other.counts if isinstance(other, PositionalCounts) else np.asarray(other, np.uint64)
        return self.counts.shape == other_counts.shape and bool((self.counts == other_counts).all())

    def total(self) -> int:  # pospop.cpp:27-31
        return int(sum(int(x) for x in self.counts))

    def __repr__(self) -> str:
        return f"PositionalCounts({[int(x) for x in self.counts]})"


def merge_counts(a: PositionalCounts, b: PositionalCounts) -> PositionalCounts:
    """result[p] = a[p] + b[p] (pospop.cpp:33-37); associative and commutative."""
    return PositionalCounts(a.counts + b.counts)


def validate(config: PospopcntConfig) -> None:
    """Raises InvalidArgument for out-of-range fields (pospop.cpp:63-70)."""
    _check(_load().pospop_validate(C.byref(config._c())))


def supported_csa_widths() -> list[int]:
    buf = (C.c_uint32 * 16)()
    n = _load().pospop_supported_widths(buf, 16)
    return list(buf[:n])


def native_csa_width() -> int:
    return supported_csa_widths()[-1]


def device_available() -> bool:
    return bool(_load().pospop_device_available())


def kernel_launches() -> int:
    return int(_load().pospop_kernel_launches())


# -- buffers -------------------------------------------------------------------

def _addr_len(data: Any, k: int) -> tuple[int, int]:
    """(address, length in k-bit words) of a numpy array, torch tensor or (addr, len) pair."""
    if isinstance(data, tuple):
        return int(data[0]), int(data[1])
    if isinstance(data, np.ndarray):
        if not data.flags.c_contiguous:
            raise InvalidArgument("array must be C-contiguous")
        return (data.ctypes.data if data.size else 0), data.nbytes * 8 // k
    if hasattr(data, "data_ptr") and hasattr(data, "element_size"):  # torch.Tensor
        if not data.is_contiguous():
            raise InvalidArgument("tensor must be contiguous")
        nbytes = data.numel() * data.element_size()
        return (data.data_ptr() if nbytes else 0), nbytes * 8 // k
    if isinstance(data, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(data, np.uint8)
        return (arr.ctypes.data if arr.size else 0), arr.nbytes * 8 // k
    raise TypeError(f"unsupported buffer type {type(data)!r}")


def _stream_ptr(stream: Any) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(getattr(stream, "cuda_stream"))  # torch.cuda.Stream


# -- the hot path ----------------------------------------------------------------

def pospopcnt(words: Any, config: PospopcntConfig | None = None) -> PositionalCounts:
    """pospop::pospopcnt(Word16Span, PospopcntConfig) on the GPU (pospop.hpp:34)."""
    addr, n = _addr_len(words, 16)
    out = np.zeros(16, np.uint64)
    cfg = (config or PospopcntConfig())._c()
    _check(_load().pospopcnt_u16_config(addr or None, n, C.byref(cfg), out.ctypes.data_as(_u64p)))
    return PositionalCounts(out)


def pospopcnt_k(data: Any, k: int, flush_threshold_blocks: int = 65535, len_words: int | None = None
                ) -> PositionalCounts:
    """k in {8,16,32,64}: counts[p] = #k-bit words with bit p set."""
    addr, n = _addr_len(data, k)
    if len_words is not None:
        n = int(len_words)
    out = np.zeros(max(k, 1), np.uint64)
    _check(_load().pospopcnt_k(int(k), addr or None, n, int(flush_threshold_blocks), out.ctypes.data_as(_u64p)))
    return PositionalCounts(out)


def pospopcnt_u16_c32(words: Any, counters: np.ndarray) -> np.ndarray:
    """PAPER.md Fig. 6 signature: uint32 counters, accumulated in place."""
    addr, n = _addr_len(words, 16)
    if counters.dtype != np.uint32 or counters.size != 16:
        raise InvalidArgument("counters must be a uint32 array of 16")
    if n > 0xFFFFFFFF:
        raise InvalidArgument("len exceeds the uint32_t len of Fig. 6")
    _check(_load().pospopcnt_u16_c32(addr or None, n, counters.ctypes.data_as(C.POINTER(C.c_uint32))))
    return counters


def _offsets_addr(offsets: Any) -> tuple[int, int]:
    """(address, n_arrays) of an offsets array: int64/uint64, contiguous, >= 1 element."""
    if isinstance(offsets, np.ndarray):
        if offsets.dtype not in (np.dtype(np.uint64), np.dtype(np.int64)):
            raise InvalidArgument(f"offsets must be uint64 or int64, got {offsets.dtype}")
        if not offsets.flags.c_contiguous:
            raise InvalidArgument("offsets must be C-contiguous")
        n = offsets.size
    elif hasattr(offsets, "data_ptr") and hasattr(offsets, "element_size"):
        import torch
        if offsets.dtype not in (torch.int64, torch.uint64):
            raise InvalidArgument(f"offsets must be int64 or uint64, got {offsets.dtype}")
        if not offsets.is_contiguous():
            raise InvalidArgument("offsets must be contiguous")
        n = offsets.numel()
    else:
        raise TypeError(f"unsupported offsets type {type(offsets)!r}")
    if n < 1:
        raise InvalidArgument("offsets needs at least one element (n_arrays + 1)")
    return (_addr_len(offsets, 64)[0] if n else 0), n - 1


def _rows_addr(out: Any, n: int, k: int) -> int:
    """Address of a row buffer holding exactly n * k 8-byte elements."""
    if isinstance(out, np.ndarray):
        ok = out.dtype.itemsize == 8 and out.dtype.kind in "iu"
        size = out.size
    elif hasattr(out, "data_ptr") and hasattr(out, "element_size"):
        ok = out.element_size() == 8 and not out.is_floating_point()
        size = out.numel()
    else:
        raise TypeError(f"unsupported row buffer type {type(out)!r}")
    if not ok:
        raise InvalidArgument("rows must be an 8-byte integer array")
    if size != n * k:
        raise InvalidArgument(f"rows must hold n_arrays * k = {n * k} elements, got {size}")
    return _addr_len(out, 64)[0]


def pospopcnt_segmented(data: Any, offsets: Any, k: int, out: Any = None) -> Any:
    """Row a = counts of words [offsets[a], offsets[a+1]); returns (n_arrays, k) uint64."""
    addr, _ = _addr_len(data, k)
    if isinstance(offsets, np.ndarray) and offsets.dtype != np.uint64 and offsets.dtype.kind in "iu":
        offsets = np.ascontiguousarray(offsets, np.uint64)
    off_addr, n = _offsets_addr(offsets)
    if out is None:
        out = np.zeros((n, k), np.uint64)
    out_addr = _rows_addr(out, n, k)
    if n > 0:
        _check(_load().pospopcnt_segmented(int(k), addr or None, off_addr, n, out_addr))
    return out


def pospopcnt_segmented_split(data: Any, offsets: Any, k: int, devices: Sequence[int], out: Any = None) -> Any:
    """pospopcnt_segmented with the arrays cut into len(devices) contiguous
    groups of about equal bytes, group i counted on devices[i] (host data over
    each device's own link).  Returns (n_arrays, k) uint64."""
    addr, _ = _addr_len(data, k)
    if isinstance(offsets, np.ndarray) and offsets.dtype != np.uint64 and offsets.dtype.kind in "iu":
        offsets = np.ascontiguousarray(offsets, np.uint64)
    off_addr, n = _offsets_addr(offsets)
    if out is None:
        out = np.zeros((n, k), np.uint64)
    out_addr = _rows_addr(out, n, k)
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    _check(_load().pospopcnt_segmented_split(int(k), addr or None, off_addr, n, devs, len(devices), out_addr))
    return out


def pospopcnt_sharded(shards: Sequence[Any], devices: Sequence[int], k: int = 16) -> PositionalCounts:
    """One process, several devices: count every shard on its device, then merge_counts."""
    n = len(shards)
    ptrs = (C.c_void_p * n)()
    lens = (C.c_size_t * n)()
    devs = (C.c_int * n)(*[int(d) for d in devices])
    for i, s in enumerate(shards):
        a, l = _addr_len(s, k)
        ptrs[i], lens[i] = a or None, l
    out = np.zeros(k, np.uint64)
    _check(_load().pospopcnt_sharded(int(k), ptrs, lens, devs, n, out.ctypes.data_as(_u64p)))
    return PositionalCounts(out)


def pospopcnt_split(data: Any, devices: Sequence[int], k: int = 16) -> PositionalCounts:
    """Host-memory fork-join in one call (proj/tests/test_core.cpp:155-175): the
    words are split into len(devices) contiguous ranges, range i is streamed to
    devices[i] over that device's own host link, and the counts are merged."""
    addr, n = _addr_len(data, k)
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    out = np.zeros(k, np.uint64)
    _check(_load().pospopcnt_split(int(k), addr or None, n, devs, len(devices), out.ctypes.data_as(_u64p)))
    return PositionalCounts(out)


def release_resources() -> None:
    """Frees the library's idle per-device contexts and per-stream workspaces."""
    _check(_load().pospop_release_resources())


def release_stream(stream: Any) -> None:
    """Synchronises `stream` and frees the library's workspaces for it."""
    _check(_load().pospop_release_stream(_stream_ptr(stream)))


def resource_stats(device: int = 0) -> dict:
    """{contexts, idle_contexts, stream_workspaces} the library holds for `device`."""
    a, b, c = C.c_int(), C.c_int(), C.c_int()
    _check(_load().pospop_resource_stats(int(device), C.byref(a), C.byref(b), C.byref(c)))
    return {"contexts": a.value, "idle_contexts": b.value, "stream_workspaces": c.value}


def count_async(data: Any, out: Any, k: int, *, accumulate: bool = False, flush_threshold_blocks: int = 65535,
                grid: int = 0, block: int = 0, stream: Any = None, len_words: int | None = None) -> None:
    """Enqueues one device-resident count (no host sync); out: k uint64 on the device."""
    addr, n = _addr_len(data, k)
    if len_words is not None:
        n = int(len_words)
    out_addr, _ = _addr_len(out, 64)
    _check(_load().pospopcnt_async(int(k), addr or None, n, out_addr, int(accumulate), int(flush_threshold_blocks),
                                   int(grid), int(block), _stream_ptr(stream)))


def count_allgather_async(data: Any, out: Any, k: int, peers: Any, n_ranks: int, rank: int, step: int,
                          slots: int = 2, *, stream: Any = None, len_words: int | None = None) -> None:
    """Count fused with the producer half of the cross-GPU all-reduce
    (pospopcnt_allgather_async): out gets this rank's counts and the kernel's
    last CTA stores them as row `rank` of slot step % slots in every rank's
    exchange buffer (`peers`: device array of n_ranks buffer pointers, see
    paper_1911_02696_b200.exchange), tagged with the step."""
    addr, n = _addr_len(data, k)
    if len_words is not None:
        n = int(len_words)
    out_addr, _ = _addr_len(out, 64)
    peers_addr, _ = _addr_len(peers, 64)
    _check(_load().pospopcnt_allgather_async(int(k), addr or None, n, out_addr, peers_addr, int(n_ranks), int(rank),
                                             int(step), int(slots), _stream_ptr(stream)))


def exchange_bytes(k: int, n_ranks: int, slots: int = 2) -> int:
    return int(_load().pospop_exchange_bytes(int(k), int(n_ranks), int(slots)))


def exchange_reduce_async(k: int, own: int, n_ranks: int, step: int, total: Any, slots: int = 2, *,
                          stream: Any = None) -> None:
    """Consumer half: waits on the device for the n_ranks rows of `step` in this
    rank's buffer `own`, writes their sum to `total` (k int64 on the device)
    and returns the slot's credit to the producers."""
    total_addr, _ = _addr_len(total, 64)
    _check(_load().pospop_exchange_reduce_async(int(k), int(own), int(n_ranks), int(step), int(slots), total_addr,
                                                _stream_ptr(stream)))


def exchange_status(own: int) -> tuple[int, int]:
    """(steps consumed, error code) of an exchange buffer; raises CudaError on a device-reported timeout."""
    consumed, err = C.c_uint64(0), C.c_uint64(0)
    st = _load().pospop_exchange_status(int(own), C.byref(consumed), C.byref(err))
    if st != _OK and err.value == 0:
        _check(st)
    if err.value:
        raise CudaError(f"exchange error {int(err.value)}: {_load().pospop_last_error().decode()}")
    return int(consumed.value), int(err.value)


def ipc_alloc(nbytes: int) -> tuple[int, bytes]:
    """A zeroed device allocation exportable to other processes: (address, 64-byte handle)."""
    ptr = C.c_void_p()
    h = (C.c_ubyte * 64)()
    _check(_load().pospop_ipc_alloc(int(nbytes), C.byref(ptr), h))
    return int(ptr.value), bytes(h)


def ipc_open(handle: bytes) -> int:
    """Maps another process's pospop_ipc_alloc allocation into this one (peer access over NVLink)."""
    ptr = C.c_void_p()
    h = (C.c_ubyte * 64).from_buffer_copy(handle)
    _check(_load().pospop_ipc_open(h, C.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int) -> None:
    _check(_load().pospop_ipc_close(C.c_void_p(ptr)))


def ipc_free(ptr: int) -> None:
    _check(_load().pospop_ipc_free(C.c_void_p(ptr)))


def segmented_async(data: Any, offsets: Any, out: Any, k: int, *, flush_threshold_blocks: int = 65535,
                    grid: int = 0, block: int = 0, stream: Any = None) -> None:
    addr, _ = _addr_len(data, k)
    off_addr, n = _offsets_addr(offsets)
    out_addr = _rows_addr(out, n, k)
    _check(_load().pospopcnt_segmented_async(int(k), addr or None, off_addr, n, out_addr,
                                             int(flush_threshold_blocks), int(grid), int(block),
                                             _stream_ptr(stream)))


GEN_UNIFORM16, GEN_CFG2, GEN_CFG3, GEN_CFG4, GEN_U32, GEN_U64, GEN_FLAGS, GEN_FLAGMIX = 1, 2, 3, 4, 5, 6, 7, 8


def generate(kind: int, seed: int, out: Any, base: int = 0, n: int | None = None, stream: Any = None) -> None:
    """Fills a device buffer with synthetic input `kind` (Synthetic inputs)."""
    esize = {1: 2, 2: 2, 3: 1, 4: 2, 5: 4, 6: 8, 7: 2, 8: 2}[kind]
    addr, nbits = _addr_len(out, 8)
    count = nbits // esize if n is None else int(n)
    _check(_load().pospop_generate(int(kind), int(seed), int(base), count, addr or None, _stream_ptr(stream)))


def digest(data: Any) -> int:
    addr, nbytes = _addr_len(data, 8)
    out = C.c_uint64(0)
    _check(_load().pospop_digest(addr or None, nbytes, C.byref(out)))
    return int(out.value)


# -- FLAG statistics (the reference's application of the path) --------------------

@dataclass
class FlagBucket:
    """pospop::FlagBucket (flagstats.hpp:39-50)."""
    total: int = 0
    secondary: int = 0
    supplementary: int = 0
    n_pair_good: int = 0
    n_read1: int = 0
    n_read2: int = 0
    n_sgltn: int = 0
    pair_map: int = 0
    mapped: int = 0
    dup: int = 0

    def as_list(self) -> list[int]:
        return [getattr(self, f) for f in _BUCKET_FIELDS]


@dataclass
class FlagSummary:
    """pospop::FlagSummary (flagstats.hpp:54-62)."""
    pass_: FlagBucket
    fail: FlagBucket

    def total(self) -> int:
        return self.pass_.total + self.fail.total

    def as_list(self) -> list[int]:
        return self.pass_.as_list() + self.fail.as_list()


def flagstats(flags: Any) -> FlagSummary:
    """pospop::flagstats_pospopcnt (flagstats.hpp:100) fused into one GPU pass.

    Raises InvalidFlagWordError at the first word with bits 12-15 set."""
    addr, n = _addr_len(flags, 16)
    out = _Summary()
    off = C.c_uint64(0)
    word = C.c_uint16(0)
    st = _load().pospop_flagstats(addr or None, n, C.byref(out), C.byref(off), C.byref(word))
    if st == _EFLAG:
        raise InvalidFlagWordError(int(off.value), int(word.value))
    _check(st)
    conv = lambda b: FlagBucket(*[int(getattr(b, f)) for f in _BUCKET_FIELDS])  # noqa: E731
    return FlagSummary(conv(out.pass_), conv(out.fail))


# -- file / pipe ingestion (the reference CLI's input path) ------------------------

def pospopcnt_file(source: Any, k: int = 16) -> tuple[PositionalCounts, int]:
    """Counts a raw little-endian k-bit word stream from a path ("-" = stdin) or an
    open file descriptor; returns (counts, word count).  As the reference's
    read_word_stream (proj/tools/pospopcnt.cpp:52-75), a byte length that is not
    a multiple of k/8 raises InvalidArgument."""
    out = np.zeros(k, np.uint64)
    n = C.c_uint64(0)
    if isinstance(source, int):
        st = _load().pospopcnt_fd(source, int(k), out.ctypes.data_as(_u64p), C.byref(n))
    else:
        st = _load().pospopcnt_file(os.fsencode(source), int(k), out.ctypes.data_as(_u64p), C.byref(n))
    _check(st)
    return PositionalCounts(out), int(n.value)


def microop(op: int, depth: int, inputs: Sequence[int], n_out: int) -> np.ndarray:
    """Diagnostics: runs a device primitive (0 csa, 1 tree, 2 extract, 3 drain,
    4 warp totals) on 32-bit registers; see pospop_microop in the C ABI."""
    a = np.ascontiguousarray(np.asarray(inputs, dtype=np.uint64).astype(np.uint32))
    out = np.zeros(max(n_out, 1), np.uint32)
    _check(_load().pospop_microop(int(op), int(depth), a.ctypes.data, a.size, out.ctypes.data, n_out))
    return out[:n_out]


class CountGraph:
    """CUDA-graph replay of one device-resident count (launch-latency path).

    Bound to (data, out); every replay() recounts the buffer's current
    contents into `out` (k uint64 on the device)."""

    def __init__(self, data: Any, out: Any, k: int, len_words: int | None = None):
        addr, n = _addr_len(data, k)
        if len_words is not None:
            n = int(len_words)
        out_addr, _ = _addr_len(out, 64)
        h = C.c_void_p()
        _check(_load().pospopcnt_graph_create(int(k), addr or None, n, out_addr, C.byref(h)))
        self._h = h
        self._keep = (data, out)  # the graph holds raw pointers to these buffers

    def replay(self, stream: Any = None) -> None:
        _check(_load().pospopcnt_graph_launch(self._h, _stream_ptr(stream)))

    def close(self) -> None:
        if self._h:
            _load().pospopcnt_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass
