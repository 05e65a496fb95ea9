#!/usr/bin/env python
"""Segmented kernels vs the stream kernel on the same 1 GiB of u32 (measurement
tool): back-to-back launches (PDL) and isolated launches, GB/s of input.

    python tools/seg_vs_stream.py [--reps 50] [--variants "7,32,13,1;6,32,13,2"]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def timed(fn, reps, s):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    b2b = a.elapsed_time(b) / reps
    iso = []
    for _ in range(7):
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        iso.append(a.elapsed_time(b))
    return b2b, statistics.median(iso)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--variants", default=";7,32,13,1;6,32,13,2;6,32,11,2")
    ap.add_argument("--words", default="4096,16384")
    ap.add_argument("--k", type=int, default=32, choices=[32, 64])
    ap.add_argument("--rounds", type=int, default=1, help="alternate the variants this many times")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    k, total = args.k, 1 << 30
    data = torch.empty(total, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_U32 if k == 32 else pp.GEN_U64, 1, data, stream=s)
    cnt = torch.zeros(k, dtype=torch.int64, device="cuda")
    b2b, iso = timed(lambda: pp.count_async(data, cnt, k, stream=s), args.reps, s)
    print(json.dumps({"kernel": f"stream k={k}", "b2b_gbs": round(total / b2b / 1e6, 1),
                      "iso_gbs": round(total / iso / 1e6, 1), "b2b_us": round(b2b * 1e3, 2)}), flush=True)
    for words in [int(w) for w in args.words.split(",")]:
        arrays = total // (k // 8) // words
        offs = torch.arange(arrays + 1, dtype=torch.int64, device="cuda") * words
        out = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
        for var in args.variants.split(";") * args.rounds:
            if var:
                os.environ["POSPOP_SEG_VARIANT"] = var
            else:
                os.environ.pop("POSPOP_SEG_VARIANT", None)
            b2b, iso = timed(lambda: pp.segmented_async(data, offs, out, k, stream=s), args.reps, s)
            rows = out.sum(dim=1)
            ok = bool(torch.equal(rows.sum(), cnt.sum()))
            print(json.dumps({"kernel": f"segmented {var or 'default'}", "words": words, "b2b_gbs":
                              round(total / b2b / 1e6, 1), "iso_gbs": round(total / iso / 1e6, 1),
                              "b2b_us": round(b2b * 1e3, 2), "total_ok": ok}), flush=True)


if __name__ == "__main__":
    main()
