"""ctypes bindings for the CHECKER libraries -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product package
(paper_1911_02696_b200) never does.

* ``Oracle``    -> oracle/liboracle.so, the plain-C restatement
                   (oracle/pospop_oracle.c).
* ``Reference`` -> oracle/_ref/libpospop_ref.so, the unmodified reference
                   core library compiled from /root/reference by
                   oracle/Makefile, behind oracle/ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpospop_ref.so")

_u64p = C.POINTER(C.c_uint64)

# KernelKind order: proj/core/include/pospop/types.hpp:52-60
KERNELS = {"scalar": 0, "csa4": 1, "csa8": 2, "csa16": 3, "forest": 4, "byteblend": 5, "auto": 6}

DTYPES = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}


def build(force: bool = False) -> None:
    """Builds liboracle.so (and the reference library when /root/reference exists)."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if os.path.isdir("/root/reference/proj/core") and (force or not os.path.exists(REF_SO)):
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref"])


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data if a.size else 0)


class Oracle:
    """The C restatement of the reference algorithm."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.orc_naive.argtypes = [C.c_void_p, C.c_size_t, C.c_int, _u64p]
        lib.orc_csa.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _u64p]
        lib.orc_csa_tree.argtypes = [C.c_int, _u64p, _u64p, _u64p]
        lib.orc_csa_tree.restype = C.c_uint64
        lib.orc_extract_top.argtypes = [C.c_uint64, _u64p, C.POINTER(C.c_uint32)]
        lib.orc_flush_bank.argtypes = [_u64p, C.POINTER(C.c_uint32), _u64p, C.c_uint32]
        lib.orc_finalize_carries.argtypes = [_u64p, C.c_int, _u64p]
        lib.orc_run_csa64.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_uint32, _u64p]
        lib.orc_run_csa64.restype = C.c_int
        lib.orc_pospopcnt.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, _u64p]
        lib.orc_pospopcnt.restype = C.c_int
        lib.orc_segmented.argtypes = [C.c_void_p, _u64p, C.c_size_t, C.c_int, C.c_int, _u64p]
        lib.orc_segmented.restype = C.c_int
        lib.orc_mt_generate_stream.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        lib.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_size_t, C.c_void_p, C.c_int]
        lib.orc_generate.restype = C.c_int
        lib.orc_digest.argtypes = [C.c_void_p, C.c_size_t]
        lib.orc_digest.restype = C.c_uint64
        for fn in (lib.orc_flagstats_reference, lib.orc_flagstats_pospopcnt):
            fn.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p]
            fn.restype = C.c_int
        lib.orc_flag_transform.argtypes = [C.c_uint16, C.POINTER(C.c_uint16), C.POINTER(C.c_uint16)]
        lib.orc_mt64_draws.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        self.lib = lib

    # -- counting -----------------------------------------------------------
    def naive(self, words: np.ndarray, k: int | None = None) -> np.ndarray:
        k = k or words.dtype.itemsize * 8
        out = np.zeros(k, np.uint64)
        self.lib.orc_naive(_ptr(words), words.size * words.dtype.itemsize * 8 // k, k,
                           out.ctypes.data_as(_u64p))
        return out

    def run_csa64(self, words: np.ndarray, block_log2: int = 4, flush: int = 65535) -> np.ndarray:
        out = np.zeros(16, np.uint64)
        rc = self.lib.orc_run_csa64(_ptr(words), words.size, block_log2, flush,
                                    out.ctypes.data_as(_u64p))
        if rc:
            raise ValueError("orc_run_csa64: invalid argument")
        return out

    def pospopcnt(self, data, k: int, len_words: int | None = None, threads: int = 1) -> np.ndarray:
        """Counts k-bit words starting at `data` (ndarray, or an int address + len_words)."""
        if isinstance(data, np.ndarray):
            addr = data.ctypes.data if data.size else 0
            n = data.nbytes * 8 // k if len_words is None else len_words
        else:
            addr, n = int(data), int(len_words)
        out = np.zeros(k, np.uint64)
        if self.lib.orc_pospopcnt(C.c_void_p(addr), n, k, threads, out.ctypes.data_as(_u64p)):
            raise ValueError("orc_pospopcnt: invalid argument")
        return out

    def segmented(self, data: np.ndarray, offsets: np.ndarray, k: int, threads: int = 1) -> np.ndarray:
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        out = np.zeros((n, k), np.uint64)
        if self.lib.orc_segmented(_ptr(data), offsets.ctypes.data_as(_u64p), n, k, threads,
                                  out.ctypes.data_as(_u64p)):
            raise ValueError("orc_segmented: invalid argument")
        return out

    # -- micro-ops ------------------------------------------------------------
    def csa(self, a: int, b: int, c: int) -> tuple[int, int]:
        h, l = C.c_uint64(), C.c_uint64()
        self.lib.orc_csa(a, b, c, C.byref(h), C.byref(l))
        return h.value, l.value

    def csa_tree(self, depth: int, carries: np.ndarray, inputs: np.ndarray) -> tuple[int, int]:
        calls = C.c_uint64(0)
        top = self.lib.orc_csa_tree(depth, carries.ctypes.data_as(_u64p),
                                    inputs.ctypes.data_as(_u64p), C.byref(calls))
        return top, calls.value

    def extract_top(self, top: int, counter: np.ndarray, blocks: int) -> int:
        b = C.c_uint32(blocks)
        self.lib.orc_extract_top(top, counter.ctypes.data_as(_u64p), C.byref(b))
        return b.value

    def flush_bank(self, counter: np.ndarray, blocks: int, counts: np.ndarray, weight: int) -> int:
        b = C.c_uint32(blocks)
        self.lib.orc_flush_bank(counter.ctypes.data_as(_u64p), C.byref(b),
                                counts.ctypes.data_as(_u64p), weight)
        return b.value

    def finalize_carries(self, carries: np.ndarray, depth: int, counts: np.ndarray) -> None:
        self.lib.orc_finalize_carries(carries.ctypes.data_as(_u64p), depth, counts.ctypes.data_as(_u64p))

    # -- generators -----------------------------------------------------------
    def mt64_draws(self, seed: int, n: int) -> np.ndarray:
        """The first n draws of std::mt19937_64(seed)."""
        out = np.empty(n, np.uint64)
        self.lib.orc_mt64_draws(seed, n, _ptr(out))
        return out

    def acceptance_flag_streams(self, count: int = 100, n: int = 100000):
        """acceptance.cpp:277-285: mt19937_64(0xF1A6), word = rng() & 0x0FFF, `count` streams of n."""
        draws = self.mt64_draws(0xF1A6, count * n)
        return (draws & np.uint64(0x0FFF)).astype(np.uint16).reshape(count, n)

    def mt_generate_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint16)
        self.lib.orc_mt_generate_stream(seed, n, _ptr(out))
        return out

    GEN_DTYPE = {1: np.uint16, 2: np.uint16, 3: np.uint8, 4: np.uint16, 5: np.uint32, 6: np.uint64, 7: np.uint16,
                 8: np.uint16}

    # -- FLAG statistics -----------------------------------------------------
    def flagstats(self, flags: np.ndarray, route: str = "reference"):
        """(rc, out20, bad_offset); rc 1 = invalid FLAG word at bad_offset."""
        out = np.zeros(20, np.uint64)
        bad = C.c_uint64(0)
        fn = self.lib.orc_flagstats_reference if route == "reference" else self.lib.orc_flagstats_pospopcnt
        rc = fn(_ptr(flags), flags.size, out.ctypes.data_as(_u64p), C.byref(bad))
        return rc, out, bad.value

    def flag_transform(self, word: int) -> tuple[int, int]:
        p, f = C.c_uint16(), C.c_uint16()
        self.lib.orc_flag_transform(word, C.byref(p), C.byref(f))
        return p.value, f.value

    def generate(self, kind: int, seed: int, n: int, base: int = 0, threads: int = 1,
                 out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(n, self.GEN_DTYPE[kind])
        if self.lib.orc_generate(kind, seed, base, n, _ptr(out), threads):
            raise ValueError(f"unknown generator kind {kind}")
        return out

    def digest(self, buf: np.ndarray) -> int:
        return int(self.lib.orc_digest(_ptr(buf), buf.nbytes))


class Reference:
    """The unmodified reference library (compiled from /root/reference)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        lib = C.CDLL(path)
        lib.ref_pospopcnt_u16.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_uint32, C.c_uint32,
                                          C.c_uint64, _u64p]
        lib.ref_validate.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64]
        lib.ref_oracle_u16.argtypes = [C.c_void_p, C.c_size_t, _u64p]
        lib.ref_pospopcnt_u16_mt.argtypes = [C.c_void_p, C.c_size_t, C.c_int, _u64p]
        lib.ref_generate_stream.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        lib.ref_supported_widths.argtypes = [C.POINTER(C.c_uint32), C.c_int]
        lib.ref_csa.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _u64p]
        lib.ref_csa_block.argtypes = [C.c_int, _u64p, _u64p, C.c_size_t, _u64p, _u64p]
        lib.ref_extract_top.argtypes = [C.c_uint64, _u64p, C.POINTER(C.c_uint32)]
        lib.ref_flush_bank.argtypes = [_u64p, C.POINTER(C.c_uint32), _u64p, C.c_uint32]
        lib.ref_finalize_carries.argtypes = [_u64p, C.c_int, _u64p]
        lib.ref_flagstats.argtypes = [C.c_void_p, C.c_size_t, C.c_int, _u64p, _u64p]
        lib.ref_segmented.argtypes = [C.c_int, C.c_void_p, _u64p, C.c_size_t, C.c_int, _u64p]
        lib.ref_segmented.restype = C.c_int
        self.lib = lib

    def pospopcnt(self, words: np.ndarray, kernel: str = "auto", width: int = 0,
                  flush: int = 65535, auto_threshold: int = 4096) -> tuple[int, np.ndarray]:
        out = np.zeros(16, np.uint64)
        rc = self.lib.ref_pospopcnt_u16(_ptr(words), words.size, KERNELS[kernel], width, flush,
                                        auto_threshold, out.ctypes.data_as(_u64p))
        return rc, out

    def validate(self, kernel: str = "auto", width: int = 0, flush: int = 65535,
                 auto_threshold: int = 4096) -> int:
        return self.lib.ref_validate(KERNELS[kernel], width, flush, auto_threshold)

    def oracle(self, words: np.ndarray) -> np.ndarray:
        out = np.zeros(16, np.uint64)
        self.lib.ref_oracle_u16(_ptr(words), words.size, out.ctypes.data_as(_u64p))
        return out

    def segmented(self, data: np.ndarray, offsets: np.ndarray, k: int, threads: int = 1) -> np.ndarray:
        """cfg5 on the reference's 16-bit API (ref_segmented, SURVEY 8c restatement)."""
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        out = np.zeros((n, k), np.uint64)
        rc = self.lib.ref_segmented(k, _ptr(data), offsets.ctypes.data_as(_u64p), n, threads,
                                    out.ctypes.data_as(_u64p))
        if rc:
            raise RuntimeError(f"ref_segmented failed ({rc})")
        return out

    def pospopcnt_mt(self, words: np.ndarray, threads: int) -> np.ndarray:
        out = np.zeros(16, np.uint64)
        if self.lib.ref_pospopcnt_u16_mt(_ptr(words), words.size, threads, out.ctypes.data_as(_u64p)):
            raise RuntimeError("reference fork-join failed")
        return out

    def generate_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint16)
        self.lib.ref_generate_stream(seed, n, _ptr(out))
        return out

    def supported_widths(self) -> list[int]:
        buf = (C.c_uint32 * 8)()
        n = self.lib.ref_supported_widths(buf, 8)
        return list(buf[:n])

    def csa(self, a: int, b: int, c: int) -> tuple[int, int]:
        h, l = C.c_uint64(), C.c_uint64()
        self.lib.ref_csa(a, b, c, C.byref(h), C.byref(l))
        return h.value, l.value

    def csa_block(self, depth: int, regs4: np.ndarray, inputs: np.ndarray) -> tuple[int, int, int]:
        top, calls = C.c_uint64(), C.c_uint64()
        rc = self.lib.ref_csa_block(depth, regs4.ctypes.data_as(_u64p), inputs.ctypes.data_as(_u64p),
                                    inputs.size, C.byref(top), C.byref(calls))
        return rc, top.value, calls.value

    def flagstats(self, words: np.ndarray, use_pospopcnt: bool = True):
        out = np.zeros(20, np.uint64)
        bad = C.c_uint64(0)
        rc = self.lib.ref_flagstats(_ptr(words), words.size, int(use_pospopcnt),
                                    out.ctypes.data_as(_u64p), C.byref(bad))
        return rc, out, bad.value
