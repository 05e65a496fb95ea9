#!/usr/bin/env python
"""Launches one workload a few times (for ncu captures; measurement tool).

    python tools/one_shot.py --what stream|seg32|seg64|flag [--reps 3]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="stream")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    if args.what == "stream":
        d = torch.empty(1 << 33, dtype=torch.uint8, device="cuda")
        pp.generate(pp.GEN_CFG4, 1, d, stream=s)
        out = torch.zeros(16, dtype=torch.int64, device="cuda")
        for _ in range(args.reps):
            pp.count_async(d, out, 16, stream=s)
    elif args.what in ("seg32", "seg64"):
        k = 32 if args.what == "seg32" else 64
        arrays, words = 65536, 4096
        d = torch.empty(arrays * words * k // 8, dtype=torch.uint8, device="cuda")
        pp.generate(pp.GEN_U32 if k == 32 else pp.GEN_U64, 1, d, stream=s)
        offs = torch.arange(0, arrays + 1, dtype=torch.int64, device="cuda") * words
        out = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
        for _ in range(args.reps):
            pp.segmented_async(d, offs, out, k, stream=s)
    elif args.what == "flag":
        d = torch.empty(1 << 32, dtype=torch.int16, device="cuda")
        pp.generate(pp.GEN_FLAGS, 1, d, stream=s)
        torch.cuda.synchronize()
        lib = pp._load()
        summ = pp._Summary()
        for _ in range(args.reps):
            assert lib.pospop_flagstats(d.data_ptr(), d.numel(), C.byref(summ), None, None) == 0
    torch.cuda.synchronize()
    print("ok", args.what)


if __name__ == "__main__":
    main()
