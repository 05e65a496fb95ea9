#!/usr/bin/env python
"""Single-GPU proxy for the cfg4 strong-scaling curve (measurement tool).

For G in 1, 2, 4, 8 it times, back to back on ONE B200, what one rank of a
G-GPU run executes per step: the count of its 2^32/G-word shard through the
fused exchange path (count kernel publishing its row with a step tag, then
the device reduce kernel) with the rank's own buffer as the only peer, and
the same shard with the plain count.  Output: per-rank GB/s and the
projected aggregate G x shard / step.  What the proxy does not contain: the
other ranks (their rows arrive over NVLink; 128 B per rank per step) and the
system-scope fence / acquire latency to remote GPUs, so it bounds the
per-GPU fixed costs from below.  The driver's 2/4/8-GPU runs are the
measurement.

    python tools/scale_proxy.py > gpurun_out/scale_proxy.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402

N = 1 << 32
K = 16


def per_step_ms(fn, s, steps):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(steps):
        fn(5 + i)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    data = torch.empty(N, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, data, stream=s)
    local = torch.zeros(K, dtype=torch.int64, device="cuda")
    total = torch.zeros(K, dtype=torch.int64, device="cuda")
    own, _ = pp.ipc_alloc(pp.exchange_bytes(K, 1, 2))
    peers = torch.tensor([own], dtype=torch.int64, device="cuda")
    step_no = [0]
    full_rate = None
    for g in (1, 2, 4, 8):
        shard = data[: N // g]
        steps = 50 * g

        def plain(i):
            pp.count_async(shard, local, K, stream=s)

        def fused(i):
            pp.count_allgather_async(shard, local, K, peers, 1, 0, step_no[0], stream=s)
            pp.exchange_reduce_async(K, own, 1, step_no[0], total, stream=s)
            step_no[0] += 1

        ms_plain = per_step_ms(plain, s, steps)
        ms_fused = per_step_ms(fused, s, steps)
        pp.exchange_status(own)
        nbytes = shard.numel() * 2
        if g == 1:
            full_rate = nbytes / ms_fused
        agg = g * nbytes / (ms_fused * 1e-3) / 1e9
        print(json.dumps({
            "gpus": g, "shard_bytes": nbytes, "ms_per_step_count": round(ms_plain, 5),
            "ms_per_step_count_plus_exchange": round(ms_fused, 5),
            "exchange_overhead_us": round((ms_fused - ms_plain) * 1e3, 2),
            "per_gpu_gbs": round(nbytes / (ms_fused * 1e-3) / 1e9, 1),
            "projected_aggregate_gbs": round(agg, 1),
            "projected_efficiency": round((nbytes / ms_fused) / full_rate, 4),
            "total_ok": int(total.sum().item()) == int(local.sum().item()),
        }), flush=True)
    pp.ipc_free(own)


if __name__ == "__main__":
    main()
