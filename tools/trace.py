#!/usr/bin/env python
"""Per-CTA timeline of the stream kernel (measurement tool, not product).

Uses pospopcnt_trace_async (per-CTA %globaltimer stamps) to split a launch's
device time into launch latency, CTA start skew, main-loop imbalance (tail)
and epilogue, for several sizes.  Prints one JSON line per (size, rep).

    python tools/trace.py > gpurun_out/trace.jsonl
"""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 or os.environ.get("POSPOP_STREAM_VARIANT"):
    os.environ.setdefault("POSPOP_LIBRARY", "tuning")  # variant strings: the tuning build
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def main():
    lib = pp._load()
    lib.pospopcnt_trace_async.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t,
                                          C.POINTER(C.c_int), C.c_void_p]
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    n = 1 << 32
    data = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, data, n=n, stream=s)
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    cap = 148 * 64
    trace = torch.zeros(cap * 5, dtype=torch.int64, device="cuda")
    grid = C.c_int(0)
    variants = [os.environ.get("POSPOP_STREAM_VARIANT", "")] + sys.argv[1:]
    for var in variants:
        if var:
            os.environ["POSPOP_STREAM_VARIANT"] = var
        sizes = [int(x) for x in os.environ.get("TRACE_BYTES", "").split(",") if x] or [1 << 29, 1 << 30, 1 << 33]
        for nbytes in sizes:
            for rep in range(4):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                rc = lib.pospopcnt_trace_async(16, data.data_ptr(), nbytes // 2, out.data_ptr(), trace.data_ptr(),
                                               cap, C.byref(grid), s.cuda_stream)
                e1.record(s)
                assert rc == 0, lib.pospop_last_error()
                torch.cuda.synchronize()
                if rep == 0:
                    continue  # warm-up
                g = grid.value
                t = trace[:g * 5].view(g, 5).cpu().tolist()
                wt = trace[g * 5:g * 5 + g * 8 * 3].view(g * 8, 3).cpu().tolist()
                t0 = [r[0] for r in t]
                t1 = [r[1] for r in t]
                t2 = [r[2] for r in t]
                t3 = [r[3] for r in t]
                base = min(t0)
                loop = [b - a for a, b in zip(t0, t1)]
                print(json.dumps({
                    "variant": var or "default", "bytes": nbytes, "grid": g, "event_us": round(e0.elapsed_time(e1) * 1e3, 2),
                    "span_us": round((max(t3) - base) / 1e3, 2),
                    "start_skew_us": round((max(t0) - base) / 1e3, 2),
                    "loop_us_min_med_max": [round(min(loop) / 1e3, 2), round(statistics.median(loop) / 1e3, 2),
                                            round(max(loop) / 1e3, 2)],
                    "loop_end_spread_us": round((max(t1) - min(t1)) / 1e3, 2),
                    "flush_us_max": round(max(b - a for a, b in zip(t1, t2)) / 1e3, 2),
                    "last_cta_us": round((max(t3) - max(t2)) / 1e3, 2),
                    "warp_range_end_us_min_med_max": [round((f(x[0] for x in wt) - base) / 1e3, 2)
                                                      for f in (min, lambda v: statistics.median(list(v)), max)],
                    "warp_pool_end_us_min_med_max": [round((f(x[1] for x in wt) - base) / 1e3, 2)
                                                     for f in (min, lambda v: statistics.median(list(v)), max)],
                    "pool_tiles_min_max_sum": [min(x[2] for x in wt), max(x[2] for x in wt), sum(x[2] for x in wt)],
                    "gbs_event": round(nbytes / (e0.elapsed_time(e1) * 1e6), 1),
                    "gbs_span": round(nbytes / (max(t3) - base), 1),
                }), flush=True)
        os.environ.pop("POSPOP_STREAM_VARIANT", None)


if __name__ == "__main__":
    main()
