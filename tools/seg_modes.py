#!/usr/bin/env python
"""Segmented throughput by array length for each schedule (measurement tool):
the pipelined bit-plane kernel (sched 6), grouped G=4 (sched 5) and the
adaptive kernel (sched 8) in its forced lane / grouped / pipelined modes and
with its default thresholds.  1 GiB of u32 (k = 32) per shape.

    python tools/seg_modes.py [--reps 20]
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

CASES = [("sched6", {"POSPOP_SEG_VARIANT": "5,16,6"}),
         ("cpasync-d5-s3", {"POSPOP_SEG_VARIANT": "5,16,10,3"}),
         ("cpasync-d5-s2", {"POSPOP_SEG_VARIANT": "5,16,10,2"}),
         ("cpasync-d5-s4", {"POSPOP_SEG_VARIANT": "5,16,10,4"}),
         ("cpasync-d4-s4", {"POSPOP_SEG_VARIANT": "4,16,10,4"}),
         ("grouped4", {"POSPOP_SEG_VARIANT": "6,16,5,4"}),
         ("auto", {"POSPOP_SEG_VARIANT": "5,16,8"}),
         ("auto:lane", {"POSPOP_SEG_VARIANT": "5,16,8", "POSPOP_SEG_LANE_MEAN_BYTES": "1048576"}),
         ("auto:grouped", {"POSPOP_SEG_VARIANT": "5,16,8", "POSPOP_SEG_LANE_MEAN_BYTES": "0",
                           "POSPOP_SEG_GROUP_MEAN_BYTES": "1048576"}),
         ("auto:pipelined", {"POSPOP_SEG_VARIANT": "5,16,8", "POSPOP_SEG_LANE_MEAN_BYTES": "0",
                             "POSPOP_SEG_GROUP_MEAN_BYTES": "0"})]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    k = 32
    total = 1 << 30
    data = torch.empty(total, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_U32, 1, data, stream=s)
    for words in (16, 64, 256, 1024, 4096, 65536, 262144):
        arrays = total // 4 // words
        offs = torch.arange(arrays + 1, dtype=torch.int64, device="cuda") * words
        out = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
        want = None
        for name, env in CASES:
            for key in ("POSPOP_SEG_VARIANT", "POSPOP_SEG_LANE_MEAN_BYTES", "POSPOP_SEG_GROUP_MEAN_BYTES"):
                os.environ.pop(key, None)
            os.environ.update(env)
            for _ in range(2):
                pp.segmented_async(data, offs, out, k, stream=s)
            torch.cuda.synchronize()
            if want is None:
                want = out.clone()
            ok = bool(torch.equal(out, want))
            ts = []
            for _ in range(args.reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                pp.segmented_async(data, offs, out, k, stream=s)
                b.record(s)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            print(json.dumps({"words": words, "arrays": arrays, "schedule": name, "ok": ok,
                              "gbs": round(total / (statistics.median(ts) * 1e-3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
