#!/usr/bin/env python
"""cfg5 back-to-back segmented launches under different row-buffer
allocations (measurement tool; DESIGN.md 3.2 "allocation effect").

    python tools/alloc_effect.py > gpurun_out/alloc_effect.txt
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402

K, WORDS, ARRAYS = 32, 4096, 65536
ROW_BYTES = ARRAYS * K * 8


def timed(data, offs, rows, s, steps=100):
    for _ in range(5):
        pp.segmented_async(data, offs, rows, K, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        pp.segmented_async(data, offs, rows, K, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    data = torch.empty(ARRAYS * WORDS * 4, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_U32, 1, data, stream=s)
    offs = torch.arange(ARRAYS + 1, dtype=torch.int64, device="cuda") * WORDS
    cudart = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            cudart = C.CDLL(name)
            break
        except OSError:
            pass
    keep = []

    def exact():
        return torch.empty((ARRAYS, K), dtype=torch.int64, device="cuda")

    def exact_zeroed():
        return torch.zeros((ARRAYS, K), dtype=torch.int64, device="cuda")

    def carved(total_mib, off_mib, zero):
        big = (torch.zeros if zero else torch.empty)(total_mib << 20, dtype=torch.uint8, device="cuda")
        keep.append(big)
        return big[off_mib << 20:(off_mib << 20) + ROW_BYTES].view(torch.int64).view(ARRAYS, K)

    def raw_cudamalloc(nbytes):
        p = C.c_void_p()
        assert cudart.cudaMalloc(C.byref(p), C.c_size_t(nbytes)) == 0
        return (p.value, ARRAYS * K)

    cases = [
        ("exact", exact),
        ("exact zeroed", exact_zeroed),
        ("carved 64 MiB @0 unwritten", lambda: carved(64, 0, False)),
        ("carved 64 MiB @0 zeroed", lambda: carved(64, 0, True)),
        ("carved 64 MiB @32 zeroed", lambda: carved(64, 32, True)),
        ("carved 18 MiB @0 zeroed", lambda: carved(18, 0, True)),
        ("carved 32 MiB @16 unwritten", lambda: carved(32, 16, False)),
    ]
    for rep in range(2):
        for name, mk in cases:
            rows = mk()
            ms = timed(data, offs, rows, s)
            print(f"{name:32s} {ms * 1e3:8.2f} us  {ARRAYS * WORDS * 4 / (ms * 1e-3) / 1e9:8.1f} GB/s", flush=True)
            del rows
        if cudart is not None:
            p, n = raw_cudamalloc(ROW_BYTES)
            out = torch.empty(0)
            # raw pointer: wrap as a tuple-addressed buffer through the C ABI directly
            lib = pp._load()
            st = s.cuda_stream
            for _ in range(5):
                lib.pospopcnt_segmented_async(K, data.data_ptr(), offs.data_ptr(), ARRAYS, p, 65535, 0, 0, st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(100):
                lib.pospopcnt_segmented_async(K, data.data_ptr(), offs.data_ptr(), ARRAYS, p, 65535, 0, 0, st)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 100
            print(f"{'cudaMalloc exact':32s} {ms * 1e3:8.2f} us  {ARRAYS * WORDS * 4 / (ms * 1e-3) / 1e9:8.1f} GB/s", flush=True)
            cudart.cudaFree(C.c_void_p(p))


if __name__ == "__main__":
    main()
