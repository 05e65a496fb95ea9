#!/usr/bin/env python
"""Benchmark: pospopcnt_u16 input GB/s and % of HBM peak at 1/2/4/8 B200 vs host CPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg4]

One rank per GPU (torchrun for N > 1, NCCL).  A *step* is one pass of the hot
path over the workload: for the default cfg4 (BASELINE.json configs[3]) every
rank counts its contiguous shard of 2^32 u16 words (Bernoulli(0.1) bits,
generated in place in HBM) with ONE kernel launch; for N > 1 that kernel's
last CTA also stores the rank's 16-entry u64 k-vector into every GPU's gather
slot through peer memory (paper_1911_02696_b200.exchange; two alternating
slots), so every GPU holds the summable rows when the step's launches
complete -- proven at setup against an NCCL all-reduce, which is the fallback
(double-buffered, on a high-priority communication stream) when peer mapping
is unavailable.  Every exchange completes inside the timed region.  Other
workloads (--workload): cfg2, cfg3, cfg5 / cfg5_u64 (segmented), flag /
flagmix (fused FLAG statistics).
Device-timed with CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  The input (8 GiB) is far larger
than the 126 MB L2, so no L2 flush is needed between steps.

Rank 0 prints ONE JSON line.  Extra keys: roofline (dominant kernel vs the
measured HBM peak), cpu_baseline (the reference library on the host cores,
N=1 only), e2e (the C-ABI call on pinned HOST buffers, H2D + D2H inside the
timed region), gpu_launches, clocks (NVML sampled during the timed region).

``--gpus N`` without torchrun re-launches itself under torch.distributed.run
with N local ranks (one GPU each); the ranks check that their GPUs are
distinct (by UUID) and refuse to print a headline if two share one.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref/libpospop_ref.so: pospop::pospopcnt, fork-join + merge_counts
over all host threads) on the SAME workload as our arm (all 2^32 words of
cfg4 per step), correctness gate first (proj/core/src/bench.cpp:55-107);
rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pospopcnt_u16 input GB/s and % of HBM peak at 1/2/4/8 B200 vs host CPU"
CFG4_WORDS = 1 << 32
FALLBACK_HBM = 6650.0

WORKLOADS = {
    # name: (k, generator kind, total words, description)
    "cfg4": (16, 4, 1 << 32, "cfg4: 2^32 u16 words, each bit Bernoulli(6554/65536), contiguous shards "
                             "over the N GPUs, k=16 u64 counters summed across GPUs (delivered to every GPU "
                             "by the counting kernel through peer memory; NCCL all-reduce as the fallback)"),
    "cfg2": (16, 2, 1 << 28, "cfg2: 2^28 u16 one-hot words, position Zipf(1.1), k=16 u64 counters"),
    "cfg3": (8, 3, (1 << 30) - 7, "cfg3: 2^30-7 u8 words at a +3 byte offset, 4 KiB runs one-hot/uniform, "
                                  "k=8 u64 counters"),
    # segmented / batched (BASELINE cfg5): one row of k counts per array
    "cfg5": (32, 5, 65536 * 4096, "cfg5: 65,536 arrays x 4096 uniform u32 words (1 GiB), one k=32 row per array "
                                  "(16 MiB of rows); arrays split over the N GPUs, no exchange"),
    "cfg5_u64": (64, 6, 65536 * 4096, "cfg5 (u64): 65,536 arrays x 4096 u64 words (2 GiB), one k=64 row per array "
                                      "(32 MiB of rows); arrays split over the N GPUs, no exchange"),
    # SURVEY 8f row f1 (not the headline metric): flagstats_pospopcnt over SAM FLAG words
    "flag": (16, 7, 1 << 32, "flag: 2^32 SAM FLAG words, uniform over the 4096 valid values (every flag combination equally likely, half QC-fail), "
                             "flagstats_pospopcnt pass/fail buckets in one fused pass; contiguous shards, "
                             "20-counter summary summed across GPUs"),
}
WORKLOADS["flagmix"] = (16, 8, 1 << 32, "flagmix: 2^32 SAM FLAG words, a paired-end-like mix (proper pairs 86%, "
                                        "duplicates 1/8, secondary/supplementary 1/128, QC-fail 2^-16), "
                                        "flagstats_pospopcnt pass/fail buckets in one fused pass")
FLAG_METRIC = "flagstats_pospopcnt input GB/s (SAM FLAG words) vs host CPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the workload's total words split over N (BASELINE cfg4); weak: per GPU")
    ap.add_argument("--clock-interval-ms", type=float, default=20.0,
                    help="NVML clock/throttle sampling period during the timed region (0 = off)")
    ap.add_argument("--collective", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 cfg4: p2p = the k-vector delivered to every GPU by the counting kernel itself "
                         "(peer-memory stores, paper_1911_02696_b200.exchange); nccl = a separate all-reduce")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-words", type=int, default=0,
                    help="reference arm only: cap the words per step (CPU-only tests; 0 = the whole workload)")
    return ap.parse_args()


def measured_peak() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str, n_gpus: int):
    """dram bytes (read+write) per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        e = t.get(f"{workload}:n{n_gpus}")
        return None if e is None else int(e["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """NVML clocks + throttle reasons sampled periodically while active.  The
    samples are taken from a side thread; at a 5 ms period the polling cost
    the launch thread ~2% of throughput, so the default period is 20 ms (a
    cfg4 timed region of 200 steps lasts ~230 ms, >= 10 samples)."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, interval_s: float = 0.02):
        self.interval_s = interval_s
        self.samples: list[int] = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        if interval_s <= 0:
            return
        try:
            import pynvml
            self._nv = pynvml
            self._h = nvml_handle(device_index)  # by UUID: NVML indices ignore CUDA_VISIBLE_DEVICES
            if self._h is None:
                return
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(self.interval_s)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self._ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for n, bit in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def h2d_link_gbs(host, dev, nbytes: int = 1 << 30, reps: int = 3):
    """The host->device link ceiling: a plain pinned cudaMemcpy of `nbytes`
    (no counting), best of `reps`, CUDA events on a side stream."""
    import torch
    n = min(nbytes, host.numel())
    if n < (64 << 20):
        return None
    dst = torch.empty(n, dtype=torch.uint8, device=dev)
    src = host.view(torch.uint8)[:n]
    s = torch.cuda.Stream(dev)
    best = None
    with torch.cuda.stream(s):
        for _ in range(reps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            dst.copy_(src, non_blocking=True)
            b.record(s)
            b.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None or ms < best else best
    del dst
    return round(n / (best * 1e-3) / 1e9, 2)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


def spawn(args) -> int:
    """--gpus N > 1 without torchrun: re-launch under torch.distributed.run
    with N local ranks (the driver's own launch form); rank 0 prints the line."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def nvml_handle(dev_index: int):
    """NVML handle of torch device `dev_index`, matched by UUID (NVML indices
    ignore CUDA_VISIBLE_DEVICES); None if NVML is unavailable."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(dev_index).uuid).lower()
        for i in range(pynvml.nvmlDeviceGetCount()):
            h = pynvml.nvmlDeviceGetHandleByIndex(i)
            u = pynvml.nvmlDeviceGetUUID(h)
            u = (u.decode() if isinstance(u, bytes) else u).lower()
            if u.endswith(uuid) or uuid.endswith(u.replace("gpu-", "")):
                return h
        return pynvml.nvmlDeviceGetHandleByIndex(dev_index)
    except Exception:  # noqa: BLE001
        return None


def pin_numa(dev_index: int) -> str:
    """Restricts this rank's host threads to the CPUs NVML reports as close to
    its GPU, so the pinned host buffers it then first-touches (and the staging
    threads of the e2e path) sit on the GPU's NUMA node.  Used for N > 1 only."""
    h = nvml_handle(dev_index)
    if h is None:
        return "nvml unavailable"
    try:
        import pynvml
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (int(m) >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return "no NUMA-local CPUs in this process's affinity"
        os.sched_setaffinity(0, cpus)
        return f"{len(cpus)} NUMA-local CPUs"
    except Exception as e:  # noqa: BLE001
        return f"affinity unavailable ({e})"


def init_rank(args):
    """One process per GPU: device, process group (NCCL INIT lines on), and the
    check that every rank owns a distinct GPU.  Returns
    (world, rank, local device index, torch.device, shared-GPU reason or "", numa note)."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1 and world != args.gpus:
        raise SystemExit(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}")
    # POSPOP_BENCH_DIST_BACKEND=gloo runs the N > 1 host path with fewer GPUs
    # than ranks (tests only; the shared-GPU guard below then trips).
    backend = os.environ.get("POSPOP_BENCH_DIST_BACKEND", "nccl")
    ndev = max(torch.cuda.device_count(), 1)
    if backend == "nccl" and local >= ndev:
        raise SystemExit(f"[bench] rank {rank}: local rank {local} but only {ndev} visible GPUs")
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa = pin_numa(local) if world > 1 else "n/a (one rank)"
    shared = ""
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # INIT lines name every rank's device
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        uuid = str(torch.cuda.get_device_properties(local).uuid)
        uuids: list = [None] * world
        dist.all_gather_object(uuids, uuid)
        if len(set(uuids)) != world:
            shared = f"ranks share a GPU ({world} ranks on {len(set(uuids))} distinct GPUs: {uuids})"
    return world, rank, local, dev, shared, numa


def reject_shared(args, metric, world, rank, shared) -> bool:
    """True if the run must stop: ranks time-slicing one GPU would report
    total bytes / max rank time above any single GPU's ceiling.  Rank 0 prints
    a line with no value.  POSPOP_BENCH_ALLOW_SHARED_GPU=1 (tests) runs on,
    marking the line."""
    if not shared or os.environ.get("POSPOP_BENCH_ALLOW_SHARED_GPU") == "1":
        return False
    import torch.distributed as dist
    if rank == 0:
        print(json.dumps({"metric": metric, "value": None, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "rejected": shared, "workload": args.workload}), flush=True)
    print(f"[bench] rank {rank}: {shared}; no headline", file=sys.stderr, flush=True)
    dist.destroy_process_group()
    return True


def isolated_ms(launch, stream, reps: int = 5) -> float:
    """Device time of ONE launch, free of host launch latency: a device sleep
    is queued first, so the start event, the launch and the end event are all
    enqueued before the GPU reaches them.  Median of `reps`."""
    import torch
    out = []
    with torch.cuda.stream(stream):
        for _ in range(reps):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)  # ~1 ms of device time
            a0.record(stream)
            launch()
            a1.record(stream)
            a1.synchronize()
            out.append(a0.elapsed_time(a1))
    return statistics.median(out)


# ---------------------------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation
# ---------------------------------------------------------------------------------------------

def _ref_libs():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    orc = pyoracle.Oracle()
    try:
        return orc, pyoracle.Reference(), "reference"
    except Exception:  # noqa: BLE001
        return orc, None, "port"


def ref_count_fn(orc, ref, k: int, threads: int):
    """fn(data) -> k counts: pospop::pospopcnt fork-join + merge_counts over
    `threads` contiguous chunks (proj/tests/test_core.cpp:155-175).  k = 8 runs
    the reference's 16-bit API per chunk with the SURVEY 8c fold (odd head /
    tail bytes counted directly); the oracle port when the reference is absent."""
    import numpy as np
    if ref is None:
        return lambda data: np.asarray(orc.pospopcnt(data, k, threads=threads), np.uint64)
    if k == 16:
        return lambda data: np.asarray(ref.pospopcnt_mt(data.view(np.uint16), threads), np.uint64)

    def run(data):
        n = data.nbytes * 8 // k
        cuts = np.array([n * i // (4 * threads) for i in range(4 * threads + 1)], np.uint64)
        return ref.segmented(data, cuts, k, threads).sum(axis=0, dtype=np.uint64)
    return run


def ref_flagstats_mt(words, threads):
    """The reference's flagstats_pospopcnt (flagstats.cpp:127-145) fork-joined
    over `threads` contiguous chunks (ctypes releases the GIL); the 20-counter
    summaries add.  Returns the summed out20."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    ref = pyoracle.Reference()
    n = words.size
    cuts = [n * i // threads for i in range(threads + 1)]

    def one(i):
        rc, out, _ = ref.flagstats(words[cuts[i]:cuts[i + 1]])
        assert rc == 0
        return out
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(one, range(threads)))
    return np.sum(parts, axis=0, dtype=np.uint64)


def oracle_flagstats_mt(orc, words, threads):
    """The oracle's flagstats (per-word restatement) over `threads` chunks, summed: the gate."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    n = words.size
    cuts = [n * i // threads for i in range(threads + 1)]

    def one(i):
        rc, out, _ = orc.flagstats(words[cuts[i]:cuts[i + 1]])
        assert rc == 0
        return out
    with ThreadPoolExecutor(threads) as ex:
        return np.sum(list(ex.map(one, range(threads))), axis=0, dtype=np.uint64)


SEG_WORDS = 4096  # words per array in cfg5


def host_workload(orc, workload: str, words: int, threads: int):
    """The workload's first `words` words generated on the host (same counter-
    based generator as the device: bit-identical data).  cfg3 sits at +3 bytes
    of a 16-byte-aligned buffer, like the device run."""
    import numpy as np
    k, gen_kind, _, _ = WORKLOADS[workload]
    wb = k // 8
    if workload == "cfg3":
        raw = np.empty(words * wb + 64, np.uint8)
        base = (-raw.ctypes.data) % 16
        view = raw[base + 3: base + 3 + words * wb]
        orc.generate(gen_kind, 1, words, threads=threads, out=view)
        return view
    return orc.generate(gen_kind, 1, words, threads=threads)


def time_steps(fn, steps: int, warmup: int, budget_s: float = 240.0):
    for _ in range(max(warmup, 1)):
        fn()
    times = []
    t_all = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:  # keep the arm within a few minutes
            break
    return times


def run_reference(args):
    """The reference arm: the whole workload per step, correctness gate first
    (proj/core/src/bench.cpp:55-107: a result that disagrees with the oracle
    produces no record), then `steps` timed passes (mean reported, best too)."""
    import numpy as np
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    threads = host_threads()
    orc, ref, kind = _ref_libs()
    k, gen_kind, total, desc = WORKLOADS[args.workload]
    wb = k // 8
    metric = FLAG_METRIC if args.workload in ("flag", "flagmix") else METRIC
    t_gen = time.perf_counter()
    if args.workload.startswith("cfg5"):
        arrays = total // SEG_WORDS
        if args.ref_words:
            arrays = max(1, min(arrays, args.ref_words // SEG_WORDS))
        words = arrays * SEG_WORDS
        data = orc.generate(gen_kind, 1, words, threads=threads)
        offs = np.arange(arrays + 1, dtype=np.uint64) * SEG_WORDS
        if ref is None:
            run = lambda: orc.segmented(data, offs, k, threads=threads)  # noqa: E731
        else:
            run = lambda: ref.segmented(data, offs, k, threads)  # noqa: E731
        want = orc.segmented(data, offs, k, threads=threads)
        gate = lambda got: bool((got == want).all())  # noqa: E731
        what = (f"all {arrays} arrays x {SEG_WORDS} words per step; per array the reference's 16-bit "
                f"pospop::pospopcnt after the SURVEY 8c deinterleave (k/16 streams), arrays fork-joined over "
                f"{threads} threads")
    elif args.workload in ("flag", "flagmix"):
        words = min(total, args.ref_words) if args.ref_words else total
        data = orc.generate(gen_kind, 1, words, threads=threads)
        run = lambda: ref_flagstats_mt(data, threads)  # noqa: E731
        want20 = oracle_flagstats_mt(orc, data, threads)
        gate = lambda got: [int(x) for x in got] == [int(x) for x in want20]  # noqa: E731
        what = (f"all {words} words of the {args.workload} stream per step; pospop::flagstats_pospopcnt "
                f"fork-joined over {threads} chunks, summaries summed")
    else:
        words = min(total, args.ref_words) if args.ref_words else total
        data = host_workload(orc, args.workload, words, threads)
        fn = ref_count_fn(orc, ref, k, threads)
        run = lambda: fn(data)  # noqa: E731
        want = np.asarray(orc.pospopcnt(data, k, threads=threads), np.uint64)
        gate = lambda got: bool((np.asarray(got, np.uint64) == want).all())  # noqa: E731
        what = (f"all {words} words of the {args.workload} stream per step"
                + (" (at +3 bytes)" if args.workload == "cfg3" else "")
                + f"; pospop::pospopcnt (Auto->Csa16 at native width) fork-join over {threads} threads "
                  f"+ merge_counts" + ("; k = 8 via the SURVEY 8c fold" if k == 8 else ""))
    t_gen = time.perf_counter() - t_gen
    if not gate(run()):  # correctness gate, doubles as warm-up
        raise SystemExit("[bench] correctness gate: the reference disagrees with the oracle")
    times = time_steps(run, args.steps, args.warmup)
    nbytes = words * wb
    mean = sum(times) / len(times)
    gbs = nbytes / mean / 1e9
    same = words == total if not args.workload.startswith("cfg5") else words == total
    line = {
        "impl": "reference", "metric": metric, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": round(mean * 1e3, 4), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": f"u{k}", "data": "synthetic",
        "config": {"workload": desc, "words_per_step": words, "bytes_per_step": nbytes, "host_threads": threads,
                   "same_config_as_ours": same, "generate_s": round(t_gen, 2)},
        "best_gbs": round(nbytes / min(times) / 1e9, 3),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": what + f"; correctness gate vs the oracle passed; mean of {len(times)} steps "
                                          f"(best {nbytes / min(times) / 1e9:.2f} GB/s)"},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_full(host, k: int, workload: str, gpu_counts, words: int):
    """Our arm's cpu_baseline leg (rank 0, N = 1): the reference on the SAME
    host copy of the whole workload the e2e leg just counted, best of 3, with
    the GPU's counts as the gate."""
    import numpy as np
    threads = host_threads()
    orc, ref, kind = _ref_libs()
    fn = ref_count_fn(orc, ref, k, threads)
    got = fn(host)
    assert (np.asarray(got, np.uint64) == np.asarray(gpu_counts, np.uint64)).all(), \
        "correctness gate: GPU and reference disagree"
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        fn(host)
        dt = time.perf_counter() - t0
        best = dt if best is None or dt < best else best
    t0 = time.perf_counter()
    ref_count_fn(orc, ref, k, 1)(host[: min(host.nbytes, 1 << 28)])
    single = min(host.nbytes, 1 << 28) / (time.perf_counter() - t0) / 1e9
    return {"value": round(host.nbytes / best / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"all {words} words ({host.nbytes >> 20} MiB) of the {workload} stream (the e2e leg's host "
                      f"copy), pospop::pospopcnt fork-join over {threads} threads + merge_counts, best of 3 "
                      f"(1 thread on 256 MiB: {single:.2f} GB/s); counts equal the GPU's"}


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------

def run_ours_seg(args):
    """cfg5: one segmented launch per step over this rank's arrays (contiguous
    array ranges; rows are per array, so there is no exchange)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_02696_b200 as pp

    world, rank, local, dev, shared, numa = init_rank(args)
    if reject_shared(args, METRIC, world, rank, shared):
        return 3
    k, gen_kind, total, desc = WORKLOADS[args.workload]
    wb = k // 8
    n_arrays_total = total // SEG_WORDS
    if args.scaling == "weak":
        a_lo, a_hi = rank * n_arrays_total, (rank + 1) * n_arrays_total
    else:
        a_lo, a_hi = n_arrays_total * rank // world, n_arrays_total * (rank + 1) // world
    arrays = a_hi - a_lo
    words = arrays * SEG_WORDS
    data = torch.empty(words * wb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    pp.generate(gen_kind, 1, data, base=a_lo * SEG_WORDS, n=words, stream=stream)
    offs = torch.arange(arrays + 1, dtype=torch.int64, device=dev) * SEG_WORDS
    rows = torch.empty((arrays, k), dtype=torch.int64, device=dev)
    torch.cuda.synchronize(dev)

    def step():
        pp.segmented_async(data, offs, rows, k, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = pp.kernel_launches()
    sampler = ClockSampler(local, args.clock_interval_ms / 1e3)
    with sampler:
        t_begin.record(stream)
        for _ in range(args.steps):
            step()  # no events between launches: programmatic dependent launch overlaps them
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = pp.kernel_launches() - launches0
    elapsed_ms = t_begin.elapsed_time(t_end)
    iso_ms = isolated_ms(step, stream)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t[0])
    ms_per_step = elapsed_ms / args.steps
    total_bytes = n_arrays_total * SEG_WORDS * wb * (world if args.scaling == "weak" else 1)
    value = total_bytes / (ms_per_step * 1e-3) / 1e9
    kern_ms = elapsed_ms / args.steps
    per_launch_bytes = words * wb + arrays * k * 8  # input read + rows written
    achieved = per_launch_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # correctness gate: every row of this rank against the oracle
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    host_data = data.cpu().numpy()
    host_offs = np.arange(arrays + 1, dtype=np.uint64) * SEG_WORDS
    want = pyoracle.Oracle().segmented(host_data, host_offs, k, threads=host_threads())
    assert (rows.cpu().numpy().view(np.uint64) == want).all(), "segmented rows disagree with the oracle"

    e2e = None
    if not args.no_e2e:
        host = torch.empty(words * wb, dtype=torch.uint8, pin_memory=True)
        host.copy_(data)
        host_rows = np.empty((arrays, k), np.uint64)
        host_arr = host.numpy()
        pp.pospopcnt_segmented(host_arr, host_offs, k, out=host_rows)
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        step_ms = []
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            pp.pospopcnt_segmented(host_arr, host_offs, k, out=host_rows)
            step_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_s = sum(step_ms) / len(step_ms) / 1e3
        assert (host_rows == want).all()
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": round(total_bytes / float(tt[0]) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": words * wb + (arrays + 1) * 8, "d2h_bytes_per_step": arrays * k * 8,
               "steps": e2e_steps, "step_ms": [round(x, 2) for x in step_ms],
               "path": "pospopcnt_segmented C ABI: pinned host data + pageable host offsets and rows; <= 32 MiB units cut "
                       "at array boundaries through a 3-slot device staging ring, unit H2D / segmented launch / "
                       "row D2H overlapped on three streams"}
        link = h2d_link_gbs(host, dev)
        if link:
            e2e["h2d_link_gbs"] = link
            e2e["frac_of_h2d_link"] = round(e2e["value"] / world / link, 4)
        del host

    cpu = None
    if world == 1 and not args.no_cpu:
        threads = host_threads()
        orc, ref, kind = _ref_libs()
        seg = (lambda: ref.segmented(host_data, host_offs, k, threads)) if ref is not None else \
            (lambda: orc.segmented(host_data, host_offs, k, threads=threads))
        assert (seg() == want).all(), "correctness gate: reference rows disagree"
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            seg()
            dt = time.perf_counter() - t0
            best = dt if best is None or dt < best else best
        cpu = {"value": round(host_data.nbytes / best / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": kind,
               "sample": f"all {arrays} arrays ({host_data.nbytes >> 20} MiB); per array the reference's 16-bit "
                         f"pospop::pospopcnt after the SURVEY 8c deinterleave, arrays fork-joined over {threads} "
                         f"threads, best of 3; rows equal the GPU's"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": f"u{k}",
        "data": "synthetic (counter-based generator, generated in place in HBM)",
        "config": {"workload": desc, "arrays_total": n_arrays_total, "words_per_array": SEG_WORDS, "k": k,
                   "bytes_per_step": total_bytes, "parallelism": f"shard{world}",
                   "l2_policy": "input >> 126 MB L2; no flush needed", "numa": numa,
                   "kernel": "segmented_auto_kernel (adaptive: tile mode for 16/32 KiB arrays); one launch per step"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.workload, world),
                     "peak_source": peak_src, "kernel_ms": round(kern_ms, 5),
                     "kernel_ms_single_launch": round(iso_ms, 5),
                     "achieved_single_launch": round(per_launch_bytes / (iso_ms * 1e-3) / 1e9, 2),
                     "timing": "back-to-back launches with programmatic dependent launch, CUDA events around the "
                               "timed region; single launch = events around one launch queued behind a device "
                               "sleep (no host launch latency), median of 5",
                     "bytes_per_launch": per_launch_bytes,
                     "frac_of_theoretical_8180": round(achieved / 8180.0, 4)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if shared:
        line["rejected"] = shared
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ours_flag(args):
    """Row f1: one pospop_flagstats C-ABI call per step over this rank's shard of
    device-resident FLAG words (one fused kernel launch + the 33-counter D2H);
    N > 1 sums the 20-counter summaries with one all-reduce."""
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_02696_b200 as pp

    world, rank, local, dev, shared, numa = init_rank(args)
    if reject_shared(args, FLAG_METRIC, world, rank, shared):
        return 3
    k, gen_kind, total, desc = WORKLOADS[args.workload]
    lo, hi = (rank * total, (rank + 1) * total) if args.scaling == "weak" else \
        (total * rank // world, total * (rank + 1) // world)
    words = hi - lo
    data = torch.empty(words, dtype=torch.int16, device=dev)
    stream = torch.cuda.current_stream(dev)
    pp.generate(gen_kind, 1, data, base=lo, n=words, stream=stream)
    torch.cuda.synchronize(dev)
    lib = pp._load()
    summ = pp._Summary()
    fields = pp._BUCKET_FIELDS
    red = torch.zeros(2 * len(fields), dtype=torch.int64, device=dev)

    def call():
        assert lib.pospop_flagstats(data.data_ptr(), words, C.byref(summ), None, None) == 0

    def step():
        call()
        if world > 1:
            vals = [getattr(summ.pass_, f) for f in fields] + [getattr(summ.fail, f) for f in fields]
            red.copy_(torch.tensor(vals, dtype=torch.int64))
            dist.all_reduce(red)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = pp.kernel_launches()
    sampler = ClockSampler(local, args.clock_interval_ms / 1e3)
    with sampler:
        t_begin.record(stream)
        for _ in range(args.steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    launches = pp.kernel_launches() - launches0
    elapsed_ms = t_begin.elapsed_time(t_end)
    # the kernel alone: async launches of the same kernel, back to back
    out33 = torch.zeros(33, dtype=torch.int64, device=dev)
    iso_ms = isolated_ms(call, stream)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t[0])
    ms_per_step = elapsed_ms / args.steps
    total_bytes = total * (world if args.scaling == "weak" else 1) * 2
    value = total_bytes / (ms_per_step * 1e-3) / 1e9
    kern_ms = elapsed_ms / args.steps if world == 1 else iso_ms
    per_launch_bytes = words * 2
    achieved = per_launch_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    del out33
    gpu_summary = pp.flagstats(data).as_list()

    host_arr = None
    e2e = None
    if not args.no_e2e:
        host = torch.empty(words, dtype=torch.int16, pin_memory=True)
        host.copy_(data)
        host_arr = host.numpy().view(np.uint16)
        assert pp.flagstats(host_arr).as_list() == gpu_summary
        e2e_steps = max(1, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            got = pp.flagstats(host_arr)
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        assert got.as_list() == gpu_summary
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": round(total_bytes / float(tt[0]) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": words * 2, "d2h_bytes_per_step": 33 * 8, "steps": e2e_steps,
               "path": "pospop_flagstats C ABI on a pinned host buffer (staged H2D ring overlapped with the kernel)"}
        link = h2d_link_gbs(host, dev)
        if link:
            e2e["h2d_link_gbs"] = link
            e2e["frac_of_h2d_link"] = round(e2e["value"] / world / link, 4)

    cpu = None
    if world == 1 and not args.no_cpu:
        threads = host_threads()
        hs = host_arr if host_arr is not None else data.cpu().numpy().view(np.uint16)
        ref_out = ref_flagstats_mt(hs, threads)
        assert [int(x) for x in ref_out] == gpu_summary, "correctness gate: GPU and reference flagstats disagree"
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            ref_flagstats_mt(hs, threads)
            dt = time.perf_counter() - t0
            best = dt if best is None or dt < best else best
        cpu = {"value": round(hs.nbytes / best / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
               "sample": f"all {words} words ({hs.nbytes >> 20} MiB) of the {args.workload} stream; "
                         f"pospop::flagstats_pospopcnt fork-joined over {threads} chunks, best of 3; "
                         f"summary equals the GPU's"}

    line = {
        "metric": FLAG_METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u16",
        "data": "synthetic (counter-based FLAG generator, generated in place in HBM)",
        "config": {"workload": desc, "words_total": total, "bytes_per_step": total_bytes,
                   "parallelism": f"shard{world}", "l2_policy": "input >> 126 MB L2; no flush needed",
                   "numa": numa,
                   "kernel": "stream_ring_kernel<3,5,MODE=2,16 warps,1 slot>: per-warp cp.async.bulk ring, "
                             "byte-frame FLAG transform + Harley-Seal trees; one launch + 33-counter D2H per step"},
        "words_per_s": round(total_bytes / 2 / (ms_per_step * 1e-3), 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.workload, world),
                     "peak_source": peak_src, "kernel_ms": round(kern_ms, 5),
                     "kernel_ms_single_launch": round(iso_ms, 5),
                     "timing": "CUDA events around K synchronous C-ABI calls (kernel + 264-byte D2H each); single "
                               "launch = one call queued behind a device sleep, median of 5",
                     "bytes_per_launch": per_launch_bytes,
                     "frac_of_theoretical_8180": round(achieved / 8180.0, 4)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if shared:
        line["rejected"] = shared
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_02696_b200 as pp

    world, rank, local, dev, shared, numa = init_rank(args)
    if reject_shared(args, METRIC, world, rank, shared):
        return 3
    k, gen_kind, total, desc = WORKLOADS[args.workload]
    wb = k // 8
    if args.scaling == "weak":
        lo, hi = rank * total, (rank + 1) * total
    else:
        lo, hi = total * rank // world, total * (rank + 1) // world
    words = hi - lo
    offset = 3 if args.workload == "cfg3" else 0
    buf = torch.empty(words * wb + offset + 64, dtype=torch.uint8, device=dev)
    data = buf[offset:offset + words * wb]
    stream = torch.cuda.current_stream(dev)
    pp.generate(gen_kind, 1, data, base=lo, n=words, stream=stream)
    torch.cuda.synchronize(dev)

    # Per step, N = 1: one count launch.  N > 1: the count kernel publishes the
    # rank's k-vector (step-tagged rows in every GPU's exchange buffer over
    # peer memory) and a one-CTA reduce kernel waits for all rows and writes
    # the all-reduced counts on the device (paper_1911_02696_b200.exchange);
    # fallback: an NCCL all-reduce on a communication stream, double-buffered.
    local_out = [torch.zeros(k, dtype=torch.int64, device=dev) for _ in range(2)]
    totals = [torch.zeros(k, dtype=torch.int64, device=dev) for _ in range(2)]
    comm = torch.cuda.Stream(dev, priority=-1) if world > 1 else None
    counted = [torch.cuda.Event() for _ in range(2)]
    reduced = [torch.cuda.Event() for _ in range(2)]
    issued = [False, False]
    xs = [0]  # the exchange's next step number (steps are consecutive)

    # Fused exchange: set it up and prove it on this machine (every rank's
    # device total equals the NCCL all-reduce of the local counts), else fall
    # back to NCCL.  Every rank runs the same collectives in the same order
    # whatever fails locally, so one rank's failure cannot hang the others.
    pg, collective = None, ("nccl" if world > 1 else "none")
    if world > 1 and args.collective == "p2p" and not shared:
        from paper_1911_02696_b200.exchange import PeerGather
        pg, reason = PeerGather.create(k)
        if pg is not None:
            probe_l = torch.zeros(k, dtype=torch.int64, device=dev)
            probe_t = torch.zeros(k, dtype=torch.int64, device=dev)
            local_ok = 1
            try:
                pg.allreduce(data, probe_l, probe_t, xs[0], stream=stream, len_words=min(words, 1 << 20))
                xs[0] += 1
                torch.cuda.synchronize(dev)
                pg.status()
            except Exception as e:  # noqa: BLE001
                local_ok, reason = 0, f"fused count: {e}"
            ref = probe_l.clone()
            dist.all_reduce(ref)  # every rank, always
            ok = torch.tensor([local_ok * int(torch.equal(probe_t, ref))], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) != 1:
                pg, reason = None, reason or "exchange totals disagree with the NCCL all-reduce"
        if pg is not None:
            collective = "p2p"
        else:
            print(f"[bench] p2p exchange unavailable ({reason}); using NCCL all-reduce", file=sys.stderr)
            collective = f"nccl (p2p unavailable: {str(reason)[:120]})"

    def step(i):
        o, tot = local_out[i % 2], totals[i % 2]
        if pg is not None:  # count + publish, then the device-side reduce
            pg.allreduce(data, o, tot, xs[0], stream=stream, len_words=words)
            xs[0] += 1
            return
        if world > 1 and issued[i % 2]:
            stream.wait_event(reduced[i % 2])
        pp.count_async(data, o, k, stream=stream, len_words=words)
        if world > 1:
            counted[i % 2].record(stream)
            with torch.cuda.stream(comm):
                comm.wait_event(counted[i % 2])
                tot.copy_(o)
                dist.all_reduce(tot)
                reduced[i % 2].record(comm)
            issued[i % 2] = True

    def join():
        if world > 1 and pg is None:
            stream.wait_stream(comm)

    for i in range(max(args.warmup, 3)):
        step(i)
    join()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    # No events inside the step loop: consecutive launches overlap through
    # programmatic dependent launch (the next count's CTAs start on SMs freed by
    # the previous one's tail) and any stream operation in between would
    # serialise them.  The average step duration is then region / K.
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = pp.kernel_launches()
    sampler = ClockSampler(local, args.clock_interval_ms / 1e3)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    with sampler:
        t_begin.record(stream)
        for i in range(args.steps):
            step(i)
        join()  # every step's reduction is inside the timed region
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = pp.kernel_launches() - launches0
    elapsed_ms = t_begin.elapsed_time(t_end)
    last = (args.steps - 1) % 2
    if pg is not None:
        pg.status()  # raises if a bounded device wait timed out
    if world == 1:
        kern_ms = elapsed_ms / args.steps  # the step is exactly one launch
    else:  # the count kernel alone: a launch-only loop on the same stream
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kreps = max(5, min(args.steps, 50))
        k0.record(stream)
        for _ in range(kreps):
            pp.count_async(data, local_out[0], k, stream=stream, len_words=words)
        k1.record(stream)
        torch.cuda.synchronize(dev)
        kern_ms = k0.elapsed_time(k1) / kreps
    iso_ms = isolated_ms(lambda: pp.count_async(data, local_out[0], k, stream=stream, len_words=words), stream)
    t = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, kern_ms_max = float(t[0]), float(t[1])
    ms_per_step = elapsed_ms / args.steps
    total_bytes = (total * (world if args.scaling == "weak" else 1)) * wb
    value = total_bytes / (ms_per_step * 1e-3) / 1e9

    # the last step's device total vs an NCCL all-reduce of this step's local counts
    pp.count_async(data, local_out[0], k, stream=stream, len_words=words)
    torch.cuda.synchronize(dev)
    mine = local_out[0].cpu().numpy().astype(np.uint64)
    counts = mine
    if world > 1:
        ref = local_out[0].clone()
        dist.all_reduce(ref)
        counts = ref.cpu().numpy().astype(np.uint64)
        assert (totals[last].cpu().numpy().astype(np.uint64) == counts).all(), \
            f"{collective} exchange disagrees with an NCCL all-reduce"
    if args.workload == "cfg2":
        assert int(counts.sum()) == total, "one-hot invariant violated"

    peak, peak_src = measured_peak()
    per_launch_bytes = words * wb + k * 8
    achieved = per_launch_bytes / (kern_ms * 1e-3) / 1e9

    # ---- e2e: the C-ABI call on pinned HOST memory (H2D + D2H inside the timed region) ----
    e2e = None
    host_arr = None
    if not args.no_e2e:
        hbuf = torch.empty(words * wb + offset + 64, dtype=torch.uint8, pin_memory=True)
        host = hbuf[offset:offset + words * wb]
        host.copy_(data)
        torch.cuda.synchronize(dev)
        host_arr = host.numpy()
        got = pp.pospopcnt_k(host_arr, k)  # warm-up: staging buffers, pinned result
        assert (np.asarray(got.counts, np.uint64) == mine).all(), "e2e counts disagree with the device count"
        e2e_steps = max(1, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        red = torch.zeros(k, dtype=torch.int64, device=dev)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            c = pp.pospopcnt_k(host_arr, k)
            if world > 1:
                red.copy_(torch.from_numpy(c.counts.astype(np.int64)))
                dist.all_reduce(red)
                red.cpu()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
        e2e = {"value": round(total_bytes / e2e_s / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": words * wb, "d2h_bytes_per_step": k * 8, "steps": e2e_steps,
               "path": "pospopcnt_k C ABI on a pinned host buffer: chunked H2D (64 MiB x3 ring) overlapped "
                       "with the kernel, k-vector D2H" + ("; one rank per GPU on its own host link, k-vectors "
                                                         "all-reduced" if world > 1 else "")}
        link = h2d_link_gbs(host, dev)
        if link:
            e2e["h2d_link_gbs"] = link
            e2e["frac_of_h2d_link"] = round(e2e["value"] / world / link, 4)

    # ---- CPU baseline on the host (rank 0, N = 1 only): the whole workload ----
    cpu = None
    if world == 1 and not args.no_cpu:
        if host_arr is None:
            hb = np.empty(words * wb + 64, np.uint8)
            o16 = (-hb.ctypes.data) % 16 + offset
            host_arr = hb[o16:o16 + words * wb]
            host_arr[:] = data.cpu().numpy()
        cpu = cpu_baseline_full(host_arr, k, args.workload, mine, words)

    traffic = ncu_traffic(args.workload, world)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u16" if k == 16 else f"u{k}",
        "data": "synthetic (counter-based generator, generated in place in HBM)",
        "config": {"workload": desc, "words_total": total, "k": k, "bytes_per_step": total_bytes,
                   "parallelism": f"shard{world}", "l2_policy": "input >> 126 MB L2; no flush needed",
                   "collective": collective, "numa": numa,
                   "kernel": "stream_kernel<NBANK=1,L=7,VB=32,BLOCK=256,SCHED=2>: LDG.E.NA.256 + LOP3 Harley-Seal depth 7, CTA ranges + shared-counter warp tiles + global tail pool; one launch per step"
                             + ("; its last CTA also publishes the step-tagged k-vector to every GPU (peer memory) "
                                "and a one-CTA reduce kernel waits for all rows and sums them on the device"
                                if collective == "p2p" else "")},
        "words_per_s": round(total_bytes / wb / (ms_per_step * 1e-3), 1),
        "pct_hbm_peak": round(100 * value / world / peak, 2),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "kernel_ms": round(kern_ms, 5), "kernel_ms_max_over_ranks": round(kern_ms_max, 5),
                     "kernel_ms_single_launch": round(iso_ms, 5),
                     "achieved_single_launch": round(per_launch_bytes / (iso_ms * 1e-3) / 1e9, 2),
                     "timing": "back-to-back launches with programmatic dependent launch, CUDA events "
                               "around the timed region (no events between launches); single launch = events "
                               "around one launch queued behind a device sleep (no host launch latency), "
                               "median of 5",
                     "bytes_per_launch": per_launch_bytes,
                     "frac_of_theoretical_8180": round(achieved / 8180.0, 4)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if shared:
        line["rejected"] = shared
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.workload in ("flag", "flagmix"):
        return run_ours_flag(args)
    if args.workload.startswith("cfg5"):
        return run_ours_seg(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
