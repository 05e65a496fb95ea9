#!/usr/bin/env python
"""Segmented kernels vs the stream kernel on the same 1 GiB of u32 (measurement
tool): back-to-back launches (PDL) and isolated launches, GB/s of input.

    python tools/seg_vs_stream.py [--reps 50] [--variants "7,32,13,1;6,32,13,2"]
"""
import argparse
import json
import os
os.environ.setdefault("POSPOP_LIBRARY", "tuning")  # POSPOP_* knobs: the tuning build
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
    ap.add_argument("--total-mib", type=int, default=1024, help="input size")
    ap.add_argument("--rounds", type=int, default=1, help="alternate the variants this many times")
    ap.add_argument("--rows-in", type=int, default=0, help="carve the rows from a buffer of this many MiB")
    ap.add_argument("--data-extra", type=int, default=0,
                    help="allocate the 1 GiB input inside a buffer this many MiB larger (negative: leave the extra unwritten)")
    ap.add_argument("--rows-init", default="empty", choices=["empty", "zeros", "ones"])
    ap.add_argument("--rows-at", type=int, default=0, help="MiB offset of the rows inside the --rows-in buffer")
    ap.add_argument("--zero-mib", default="", help="lo,hi: zero only this MiB range of the --rows-in buffer")
    ap.add_argument("--prealloc", type=int, default=0,
                    help="allocate (and zero, if negative: leave unwritten) then free this many MiB before the rows")
    ap.add_argument("--offs-in", type=int, default=0, help="carve the offsets from a buffer of this many MiB")
    ap.add_argument("--giant-frac", type=float, default=0.0,
                    help="replace this fraction of the arrays (in the middle) by ONE giant array")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    k, total = args.k, args.total_mib << 20
    if args.data_extra:
        big = torch.empty(total + (abs(args.data_extra) << 20), dtype=torch.uint8, device="cuda")
        if args.data_extra > 0:
            big.zero_()
        data = big[:total]
    else:
        data = torch.empty(total, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_U32 if k == 32 else pp.GEN_U64, 1, data, stream=s)
    cnt = torch.zeros(k, dtype=torch.int64, device="cuda")
    b2b, iso = timed(lambda: pp.count_async(data, cnt, k, stream=s), args.reps, s)
    print(json.dumps({"kernel": f"stream k={k}", "b2b_gbs": round(total / b2b / 1e6, 1),
                      "iso_gbs": round(total / iso / 1e6, 1), "b2b_us": round(b2b * 1e3, 2)}), flush=True)
    for words in [int(w) for w in args.words.split(",")]:
        arrays = total // (k // 8) // words
        offs = torch.arange(arrays + 1, dtype=torch.int64, device="cuda") * words
        if args.giant_frac > 0:  # arrays [g0, g1) merged into one
            g0 = int(arrays * (0.5 - args.giant_frac / 2))
            g1 = int(arrays * (0.5 + args.giant_frac / 2))
            offs = torch.cat([offs[:g0 + 1], offs[g1:]])
            arrays = offs.numel() - 1
        if args.offs_in:
            ob = torch.empty(args.offs_in << 17, dtype=torch.int64, device="cuda")
            ob[:offs.numel()].copy_(offs)
            offs = ob[:offs.numel()]
        if args.prealloc:
            tmp = torch.empty(abs(args.prealloc) << 20, dtype=torch.uint8, device="cuda")
            if args.prealloc > 0:
                tmp.zero_()
            torch.cuda.synchronize()
            del tmp
        if args.rows_in:
            rb = torch.empty(args.rows_in << 17, dtype=torch.int64, device="cuda")
            if args.rows_init == "zeros":
                rb.zero_()
            if args.zero_mib:
                zlo, zhi = (int(x) for x in args.zero_mib.split(","))
                rb[zlo << 17:zhi << 17].zero_()
            out = rb[(args.rows_at << 17):(args.rows_at << 17) + arrays * k].view(arrays, k)
        else:
            out = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
        if args.rows_init != "empty" and not args.rows_in:
            out.fill_(0 if args.rows_init == "zeros" else -1)
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
