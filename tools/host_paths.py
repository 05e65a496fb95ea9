#!/usr/bin/env python
"""Host-input throughput of the C ABI (measurement tool): the same words from
pinned memory, pageable memory and a file, through pospopcnt_k / pospopcnt_file.

    python tools/host_paths.py [--gib 2] [--reps 3]
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=2.0)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1911_02696_b200 as pp

    torch.cuda.set_device(0)
    n = int(args.gib * (1 << 30)) // 2
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, d)
    want = pp.pospopcnt(d)
    pinned = torch.empty(n, dtype=torch.int16, pin_memory=True)
    pinned.copy_(d)
    pageable = d.cpu().numpy().copy()
    cases = {"pinned": pinned.numpy(), "pageable": pageable}
    for name, arr in cases.items():
        assert pp.pospopcnt(arr) == want
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            pp.pospopcnt(arr)
            ts.append(time.perf_counter() - t0)
        print(json.dumps({"path": name, "bytes": 2 * n, "gbs_best": round(2 * n / min(ts) / 1e9, 2)}), flush=True)
    with tempfile.NamedTemporaryFile(dir="/tmp", delete=False) as f:
        pageable.tofile(f)
        path = f.name
    try:
        c, nw = pp.pospopcnt_file(path, 16)
        assert nw == n and c == want
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            pp.pospopcnt_file(path, 16)
            ts.append(time.perf_counter() - t0)
        print(json.dumps({"path": "file (page cache)", "bytes": 2 * n, "gbs_best": round(2 * n / min(ts) / 1e9, 2)}),
              flush=True)
    finally:
        os.unlink(path)


if __name__ == "__main__":
    main()
