#!/usr/bin/env python
"""Back-to-back count throughput versus input size (measurement tool): K
launches per size on the same stream (programmatic dependent launch, no events
between launches), GB/s = K x bytes / elapsed.

    python tools/size_curve.py [--k 16] [--reps 50]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--min-lg", type=int, default=20)
    ap.add_argument("--max-lg", type=int, default=33)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    data = torch.empty(1 << 33, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, data, n=1 << 32, stream=s)
    outs = [torch.zeros(64, dtype=torch.int64, device="cuda") for _ in range(2)]
    wb = args.k // 8
    for lg in range(args.min_lg, args.max_lg + 1):
        nbytes = 1 << lg
        reps = args.reps if lg >= 26 else args.reps * 4
        for i in range(3):
            pp.count_async(data, outs[i % 2], args.k, stream=s, len_words=nbytes // wb)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        for i in range(reps):
            pp.count_async(data, outs[i % 2], args.k, stream=s, len_words=nbytes // wb)
        b.record(s)
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        print(json.dumps({"bytes": nbytes, "us_per_launch": round(ms * 1e3, 2),
                          "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
