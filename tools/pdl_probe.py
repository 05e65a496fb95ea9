#!/usr/bin/env python
"""Back-to-back launch throughput with/without programmatic dependent launch
(measurement tool, not product).  One JSON line per (size, pdl, events)."""
import json
import os
os.environ.setdefault("POSPOP_LIBRARY", "tuning")  # POSPOP_* knobs: the tuning build
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    n = 1 << 32
    data = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, data, n=n, stream=s)
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    ref = {}
    reps = 50
    for nb in (1 << 29, 1 << 30, 1 << 31, 1 << 33):
        for pdl in ("0", "1"):
            os.environ["POSPOP_PDL"] = pdl
            for per_step_events in (False, True):
                for _ in range(5):
                    pp.count_async(data, out, 16, stream=s, len_words=nb // 2)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                t0.record(s)
                for i in range(reps):
                    if per_step_events:
                        ev[2 * i].record(s)
                    pp.count_async(data, out, 16, stream=s, len_words=nb // 2)
                    if per_step_events:
                        ev[2 * i + 1].record(s)
                t1.record(s)
                torch.cuda.synchronize()
                ms = t0.elapsed_time(t1) / reps
                c = out.cpu().tolist()
                ref.setdefault(nb, c)
                line = {"bytes": nb, "pdl": pdl, "per_step_events": per_step_events, "ms_per_launch": round(ms, 5),
                        "gbs": round(nb / ms / 1e6, 1), "counts_equal": c == ref[nb]}
                if per_step_events:
                    k = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps)) / reps
                    line["kernel_ms_events"] = round(k, 5)
                print(json.dumps(line), flush=True)
    os.environ.pop("POSPOP_PDL", None)


if __name__ == "__main__":
    main()
