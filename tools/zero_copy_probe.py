#!/usr/bin/env python
"""Pinned host input: the counting kernel reading host memory directly
(zero-copy through UVA) vs the staged path of the C ABI (measurement tool).

    python tools/zero_copy_probe.py > gpurun_out/zero_copy.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    maxb = 1 << 33
    host = torch.empty(maxb, dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    hv[: 1 << 24] = np.random.default_rng(1).integers(0, 256, size=1 << 24, dtype=np.uint8)
    for off in range(1 << 24, maxb, 1 << 24):
        hv[off:off + (1 << 24)] = hv[: 1 << 24]
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    print("bytes,staged_sync_us,zero_copy_async_us,staged_gbs,zero_copy_gbs,equal")
    for nb in [1 << 16, 1 << 18, 1 << 20, 1 << 21, 1 << 22, 1 << 23, 1 << 24, 1 << 26, 1 << 28, 1 << 30, 1 << 33]:
        reps = 20 if nb <= (1 << 26) else (5 if nb <= (1 << 30) else 2)
        view = (host.data_ptr(), nb // 2)
        want = pp.pospopcnt_k(view, 16)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            got = pp.pospopcnt_k(view, 16)
            ts.append(time.perf_counter() - t0)
        staged = sorted(ts)[len(ts) // 2]
        tz = []
        for _ in range(reps):
            t0 = time.perf_counter()
            pp.count_async(view, out, 16, stream=s)
            s.synchronize()
            tz.append(time.perf_counter() - t0)
        zc = sorted(tz)[len(tz) // 2]
        eq = [int(x) for x in out.cpu().numpy()] == [int(x) for x in want]
        print(f"{nb},{staged * 1e6:.1f},{zc * 1e6:.1f},{nb / staged / 1e9:.1f},{nb / zc / 1e9:.1f},{eq}", flush=True)


if __name__ == "__main__":
    main()
