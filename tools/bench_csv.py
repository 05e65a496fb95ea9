#!/usr/bin/env python
"""Size sweep in the reference's CSV schema (measurement tool).

The reference's bench::sweep / write_csv (proj/core/src/bench.cpp:132-173,
header proj/core/include/pospop/bench.hpp:74-75) emit
    kernel,len_words,reps,wall_ns,gbps,cycles_per_word,instructions_per_word,stderr_pct
This tool emits the same columns for the GPU path -- `gpu_device` (device-
resident, CUDA-event time of one async launch), `gpu_graph` (the same count
replayed from a CUDA graph) and `gpu_host` (the synchronous
C-ABI call on a pinned host buffer, wall time incl. H2D + D2H) -- extended
with gpus,dev_ns,bytes,pct_hbm_peak,words_per_s.  Like the reference, every
cell is gated on correctness first (bench.cpp:64-68: a mismatch produces an
error cell) and keeps the best of `reps`.  CPU counters are not applicable
(columns left empty, as the reference does when perf counters are
unavailable).

    python tools/bench_csv.py [--sizes 4k,256k,8m,128m] [--reps 20] > gpurun_out/sweep.csv
"""
import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

HEADER = "kernel,len_words,reps,wall_ns,gbps,cycles_per_word,instructions_per_word,stderr_pct"
EXTRA = "gpus,dev_ns,bytes,pct_hbm_peak,words_per_s"


def parse_sizes(csv):  # proj/tools/pospopcnt.cpp:97-125 (k = x1024, m = x1048576)
    out = []
    for tok in csv.split(","):
        mult = {"k": 1024, "m": 1048576}.get(tok[-1].lower(), 1)
        out.append(int(tok[:-1] if mult > 1 else tok) * mult)
    return out


def stderr_pct(samples):  # bench.cpp:34-51
    if len(samples) < 2:
        return 0.0
    mean = statistics.fmean(samples)
    return 100.0 * math.sqrt(statistics.variance(samples) / len(samples)) / mean if mean > 0 else 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4k,256k,8m,128m,1024m")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_1911_02696_b200 as pp
    import pyoracle

    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    orc = pyoracle.Oracle()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    print(HEADER + "," + EXTRA)
    for n in parse_sizes(args.sizes):
        host = orc.generate(1, args.seed, n, threads=8)  # uniform u16 (the reference sweeps uniform data)
        expected = orc.pospopcnt(host, 16, threads=8)
        pinned = torch.empty(n, dtype=torch.int16).pin_memory()
        pinned.numpy().view(np.uint16)[:] = host
        dev = pinned.cuda()
        out = torch.zeros(16, dtype=torch.int64, device="cuda")
        graph = pp.CountGraph(dev, out, 16)
        for kernel in ("gpu_device", "gpu_graph", "gpu_host"):
            try:
                if kernel == "gpu_device":
                    pp.count_async(dev, out, 16, stream=s)
                    torch.cuda.synchronize()
                    if not (out.cpu().numpy().astype(np.uint64) == expected).all():
                        raise RuntimeError("correctness gate: gpu_device disagrees with the oracle")
                    times = []
                    for _ in range(args.reps):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(s)
                        pp.count_async(dev, out, 16, stream=s)
                        b.record(s)
                        b.synchronize()
                        times.append(a.elapsed_time(b) * 1e6)
                elif kernel == "gpu_graph":  # CUDA-graph replay (latency path)
                    graph.replay(s)
                    torch.cuda.synchronize()
                    if not (out.cpu().numpy().astype(np.uint64) == expected).all():
                        raise RuntimeError("correctness gate: gpu_graph disagrees with the oracle")
                    times = []
                    for _ in range(args.reps):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(s)
                        graph.replay(s)
                        b.record(s)
                        b.synchronize()
                        times.append(a.elapsed_time(b) * 1e6)
                else:
                    got = pp.pospopcnt(pinned)
                    if got != expected:
                        raise RuntimeError("correctness gate: gpu_host disagrees with the oracle")
                    times = []
                    for _ in range(args.reps):
                        t0 = time.perf_counter_ns()
                        pp.pospopcnt(pinned)
                        times.append(time.perf_counter_ns() - t0)
                best = max(1, int(min(times)))
                gbps = 2.0 * n / best
                print(f"{kernel},{n},{args.reps},{best},{gbps:.4f},,,{stderr_pct(times):.3f},"
                      f"1,{best},{2 * n},{100 * gbps / peak:.2f},{n / best * 1e9:.4g}", flush=True)
            except Exception as e:  # noqa: BLE001 -- a failed cell keeps the sweep going (bench.cpp:143-152)
                print(f"{kernel},{n},{args.reps},,,,,,1,,{2 * n},,", flush=True)
                print(f"# {kernel} n={n}: {e}", file=sys.stderr)


if __name__ == "__main__":
    main()
