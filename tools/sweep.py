#!/usr/bin/env python
"""Tuning sweep (measurement tool, not product): kernel variants on the BASELINE
configs, device-timed with CUDA events (median of reps), plus the pure-read
probe (tools/probe) for the achievable read-only HBM bandwidth.

    python tools/sweep.py [--what probe,stream,seg] [--reps 20] > gpurun_out/sweep.jsonl
"""
import argparse
import ctypes as C
import json
import os
os.environ.setdefault("POSPOP_LIBRARY", "tuning")  # POSPOP_* knobs: the tuning build
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402


def timed(fn, reps, stream):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    return statistics.median(ms), min(ms)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="probe,stream,seg")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    what = set(args.what.split(","))
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    sp = s.cuda_stream
    n = 1 << 32
    buf = torch.empty(2 * n + 4096, dtype=torch.uint8, device="cuda")
    data = buf[:2 * n]
    pp.generate(pp.GEN_CFG4, 1, data, n=n, stream=s)
    torch.cuda.synchronize()
    nbytes = 2 * n

    if "probe" in what:
        lib = C.CDLL(os.path.join(ROOT, "tools", "probe", "libpospop_probe.so"))
        lib.probe_read.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p]
        sink = torch.zeros(1, dtype=torch.int64, device="cuda")
        for vb, hint, vpt in [(16, 0, 4), (16, 0, 8), (16, 0, 16), (16, 2, 8), (16, 2, 16), (32, 0, 2), (32, 0, 4),
                              (32, 0, 8), (32, 1, 4), (32, 1, 8)]:
            for block, per_sm in [(256, 0), (256, 2), (256, 4), (512, 2), (1024, 1), (128, 8)]:
                def fn():
                    rc = lib.probe_read(data.data_ptr(), nbytes, vb, hint, vpt, block, per_sm, sp, sink.data_ptr())
                    assert rc == 0, rc
                try:
                    med, best = timed(fn, args.reps, s)
                except AssertionError as e:
                    emit(kind="probe", vb=vb, hint=hint, vpt=vpt, block=block, per_sm=per_sm, error=str(e))
                    continue
                emit(kind="probe", vb=vb, hint=hint, vpt=vpt, block=block, per_sm=per_sm,
                     gbs_med=round(nbytes / med / 1e6, 1), gbs_best=round(nbytes / best / 1e6, 1))

    if "stream" in what:
        out = torch.zeros(16, dtype=torch.int64, device="cuda")
        for key in ("POSPOP_STREAM_VARIANT", "POSPOP_BLOCKS_PER_SM", "POSPOP_CHUNK_A", "POSPOP_CHUNK_B",
                    "POSPOP_TAIL_TILES_PER_WARP", "POSPOP_POOL_TILES_PER_WARP"):
            os.environ.pop(key, None)
        pp.count_async(data, out, 16, stream=s)
        torch.cuda.synchronize()
        want = out.clone()
        cases = [  # (variant, per_sm, CA, CB, tail or pool tiles per warp)
            ("7,32,0,256,0", "", "", "", ""),
            ("7,32,0,256,1", "", "64", "", "32"), ("7,32,0,256,1", "", "32", "", "64"),
            ("7,32,0,256,2", "", "", "", ""),
            ("7,32,0,256,2", "", "", "", "0"), ("7,32,0,256,2", "", "", "", "1"), ("7,32,0,256,2", "", "", "", "2"),
            ("7,32,0,256,2", "", "", "", "8"), ("7,32,0,256,2", "", "", "", "16"),
            ("7,32,0,256,2", "", "", "1", ""), ("7,32,0,256,2", "", "", "4", ""), ("7,32,0,256,2", "", "", "8", "16"),
            ("7,32,0,256,2", "2", "", "", ""),
            ("6,32,0,256,2", "", "", "", ""), ("7,16,0,256,2", "", "", "", ""),
        ]
        for var, per_sm, ca, cb, tail in cases:
            env = {"POSPOP_STREAM_VARIANT": var, "POSPOP_BLOCKS_PER_SM": per_sm, "POSPOP_CHUNK_A": ca,
                   "POSPOP_CHUNK_B": cb, "POSPOP_TAIL_TILES_PER_WARP": tail if var.endswith(",1") else "",
                   "POSPOP_POOL_TILES_PER_WARP": tail if var.endswith(",2") else ""}
            for kk, vv in env.items():
                if vv:
                    os.environ[kk] = vv
                else:
                    os.environ.pop(kk, None)
            for nb in (1 << 29, 1 << 30, 1 << 33):
                try:
                    med, best = timed(lambda: pp.count_async(data, out, 16, stream=s, len_words=nb // 2), args.reps, s)
                    ok = nb != (1 << 33) or bool(torch.equal(out, want))
                    emit(kind="stream16", bytes=nb, variant=var, per_sm=per_sm or "occ", CA=ca or "16", CB=cb or "2",
                         tail=tail or "8", gbs_med=round(nb / med / 1e6, 1), gbs_best=round(nb / best / 1e6, 1), ok=ok)
                except Exception as e:  # noqa: BLE001
                    emit(kind="stream16", variant=var, error=repr(e))
        for key in ("POSPOP_STREAM_VARIANT", "POSPOP_BLOCKS_PER_SM", "POSPOP_CHUNK_A", "POSPOP_CHUNK_B",
                    "POSPOP_TAIL_TILES_PER_WARP", "POSPOP_POOL_TILES_PER_WARP"):
            os.environ.pop(key, None)
        # other k on the same bytes
        for k, var in [(8, "7,32,0,256,2"), (32, "7,32,0,256,2"), (64, "6,32,0,256,2"), (64, "6,32,0,256,0")]:
            os.environ["POSPOP_STREAM_VARIANT"] = var
            o = torch.zeros(k, dtype=torch.int64, device="cuda")
            for nb in (1 << 30, 1 << 33):
                med, best = timed(lambda: pp.count_async(data, o, k, stream=s, len_words=nb * 8 // k), args.reps, s)
                emit(kind=f"stream{k}", bytes=nb, variant=var, gbs_med=round(nb / med / 1e6, 1),
                     gbs_best=round(nb / best / 1e6, 1))
        os.environ.pop("POSPOP_STREAM_VARIANT", None)
        # cfg3 (u8 at +3, 2^30-7) and cfg2 (2^28 one-hot), default variant
        b3 = torch.empty((1 << 30) + 64, dtype=torch.uint8, device="cuda")
        n3 = (1 << 30) - 7
        pp.generate(pp.GEN_CFG3, 1, b3[3:3 + n3], stream=s)
        o8 = torch.zeros(8, dtype=torch.int64, device="cuda")
        b2 = torch.empty(1 << 29, dtype=torch.uint8, device="cuda")
        pp.generate(pp.GEN_CFG2, 1, b2, stream=s)
        med, best = timed(lambda: pp.count_async(b3[3:3 + n3], o8, 8, stream=s), args.reps, s)
        emit(kind="cfg3", gbs_med=round(n3 / med / 1e6, 1), gbs_best=round(n3 / best / 1e6, 1))
        med, best = timed(lambda: pp.count_async(b2, out, 16, stream=s), args.reps, s)
        emit(kind="cfg2", gbs_med=round((1 << 29) / med / 1e6, 1), gbs_best=round((1 << 29) / best / 1e6, 1))
        del b3, b2

    if "tma" in what:  # TMA-staged (SCHED 3) vs LDG (SCHED 2) on the same bytes
        out = torch.zeros(16, dtype=torch.int64, device="cuda")
        cases = [("7,32,0,256,2", ""), ("5,32,0,256,3", "8,6"), ("6,32,0,256,3", "8,3"), ("5,32,0,256,3", "8,4"),
                 ("4,32,0,256,3", "8,6"), ("5,32,0,256,3", "4,6")]
        for var, tma in cases:
            os.environ["POSPOP_STREAM_VARIANT"] = var
            if tma:
                os.environ["POSPOP_TMA"] = tma
            else:
                os.environ.pop("POSPOP_TMA", None)
            for nb in (1 << 30, 1 << 33):
                med, best = timed(lambda: pp.count_async(data, out, 16, stream=s, len_words=nb // 2), args.reps, s)
                emit(kind="tma16", variant=var, tma=tma, bytes=nb, gbs_med=round(nb / med / 1e6, 1),
                     gbs_best=round(nb / best / 1e6, 1))
        for var, tma in [("6,32,0,256,2", ""), ("4,32,0,256,3", "8,6"), ("5,32,0,256,3", "8,3")]:
            os.environ["POSPOP_STREAM_VARIANT"] = var
            if tma:
                os.environ["POSPOP_TMA"] = tma
            else:
                os.environ.pop("POSPOP_TMA", None)
            o = torch.zeros(64, dtype=torch.int64, device="cuda")
            med, best = timed(lambda: pp.count_async(data, o, 64, stream=s), args.reps, s)
            emit(kind="tma64", variant=var, tma=tma, bytes=1 << 33, gbs_med=round((1 << 33) / med / 1e6, 1))
        os.environ.pop("POSPOP_STREAM_VARIANT", None)
        os.environ.pop("POSPOP_TMA", None)

    if "flag" in what or "flagmix" in what:
        lib = pp._load()
        nf = 1 << 32  # 8 GiB of FLAG words
        pp.generate(pp.GEN_FLAGMIX if "flagmix" in what else pp.GEN_FLAGS, 1, data, n=nf, stream=s)
        torch.cuda.synchronize()
        import ctypes as CC
        summ = pp._Summary()
        for var in ["5,32,0,512,2,2", "5,16,0,512,2,2", "4,32,0,512,2,2", "6,32,0,256,2,2", "6,32,0,512,2"]:
            var, _, tma = var.partition("/")
            os.environ["POSPOP_FLAG_VARIANT"] = var
            if tma:
                os.environ["POSPOP_TMA"] = tma
            else:
                os.environ.pop("POSPOP_TMA", None)
            for nb in (1 << 30, 1 << 33):
                med, best = timed(lambda: lib.pospop_flagstats(data.data_ptr(), nb // 2, CC.byref(summ), None, None),
                                  max(3, args.reps // 4), s)
                emit(kind="flagstats", bytes=nb, variant=var, tma=tma, gbs_med=round(nb / med / 1e6, 1),
                     gbs_best=round(nb / best / 1e6, 1), note="sync C-ABI call incl. D2H of 33 u64")
        os.environ.pop("POSPOP_FLAG_VARIANT", None)
        os.environ.pop("POSPOP_TMA", None)

    if "seg" in what:
        seg_cases = {
            32: ["5,16,6", "5,32,6", "6,16,5,4", "6,16,5,8", "5,16,3", "4,16,7", "4,32,7", "6,16,5,16"],
            64: ["5,16,1", "4,16,6", "4,32,6", "3,32,6", "3,16,7", "4,16,5,8"],
        }
        for k, kind in [(32, pp.GEN_U32), (64, pp.GEN_U64)]:
            shapes = [(65536, 4096)] + ([(262144, 1024), (1048576, 256), (4194304, 64), (4096, 65536),
                                         (1024, 262144)] if k == 32 else [])
            for arrays, words in shapes:
                d = data[:arrays * words * k // 8]
                pp.generate(kind, 1, d, stream=s)
                offs = torch.arange(0, arrays + 1, dtype=torch.int64, device="cuda") * words
                o = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
                want = None
                variants = seg_cases[k] if (arrays, words) == (65536, 4096) else seg_cases[k][:4]
                for var in variants:
                    os.environ["POSPOP_SEG_VARIANT"] = var
                    med, best = timed(lambda: pp.segmented_async(d, offs, o, k, stream=s), args.reps, s)
                    if want is None:
                        want = o.clone()
                    emit(kind=f"seg{k}", arrays=arrays, words=words, variant=var, ok=bool(torch.equal(o, want)),
                         gbs_med=round(d.numel() / med / 1e6, 1), gbs_best=round(d.numel() / best / 1e6, 1))
                os.environ.pop("POSPOP_SEG_VARIANT", None)


if __name__ == "__main__":
    main()
