#!/usr/bin/env python
"""Per-warp timeline of the segmented tile mode in back-to-back launches
(measurement tool; tuning build: pospop_tuning_seg_trace).  cfg5 shapes.

For the LAST of a run of back-to-back launches, per warp: entry, first array
counted (the warp now wants to store its row and waits for the previous
launch), wait done, exit.  The earliest wait-done time is the previous
launch's completion; the spread of the rest shows how much of the previous
launch's tail the early start covers.

    python tools/seg_trace.py > gpurun_out/seg_trace.jsonl
"""
import ctypes as C
import json
import os
import statistics
import sys

os.environ.setdefault("POSPOP_LIBRARY", "tuning")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))]


def main():
    lib = pp._load()
    lib.pospop_tuning_seg_trace.argtypes = [C.c_void_p]
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nw = sms * 2 * 8
    trace = torch.zeros(nw * 5, dtype=torch.int64, device="cuda")
    for k, kind in ((32, pp.GEN_U32), (64, pp.GEN_U64)):
        arrays, words = 65536, 4096
        d = torch.empty(arrays * words * k // 8, dtype=torch.uint8, device="cuda")
        pp.generate(kind, 1, d, stream=s)
        offs = torch.arange(arrays + 1, dtype=torch.int64, device="cuda") * words
        rows = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
        for mode, reps in (("isolated", 1), ("back_to_back", 20)):
            for _ in range(3):
                pp.segmented_async(d, offs, rows, k, stream=s)
            torch.cuda.synchronize()
            trace.zero_()
            assert lib.pospop_tuning_seg_trace(trace.data_ptr()) == 0
            if mode == "isolated":
                torch.cuda._sleep(2_000_000)
            for _ in range(reps):
                pp.segmented_async(d, offs, rows, k, stream=s)
            torch.cuda.synchronize()
            assert lib.pospop_tuning_seg_trace(None) == 0
            t = trace.view(nw, 5).cpu().tolist()
            t = [r for r in t if r[0] and r[3]]
            base = min(r[0] for r in t)
            entry = [(r[0] - base) / 1e3 for r in t]
            first = [(r[1] - base) / 1e3 for r in t if r[1]]
            waited = [(r[2] - base) / 1e3 for r in t if r[2]]
            exit_ = [(r[3] - base) / 1e3 for r in t]
            idle = [(r[2] - r[1]) / 1e3 for r in t if r[1] and r[2]]
            print(json.dumps({
                "k": k, "mode": mode, "warps": len(t),
                "entry_us_p0_p50_p100": [round(min(entry), 2), round(statistics.median(entry), 2), round(max(entry), 2)],
                "first_array_done_us_p0_p50_p100": [round(min(first), 2), round(statistics.median(first), 2),
                                                    round(max(first), 2)],
                "wait_done_us_p0_p50_p100": [round(min(waited), 2), round(statistics.median(waited), 2),
                                             round(max(waited), 2)],
                "idle_waiting_us_p50_p90_max": [round(statistics.median(idle), 2), round(pct(idle, 0.9), 2),
                                                round(max(idle), 2)],
                "exit_us_p0_p50_p100": [round(min(exit_), 2), round(statistics.median(exit_), 2), round(max(exit_), 2)],
            }), flush=True)


if __name__ == "__main__":
    main()
