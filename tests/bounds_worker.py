"""Worker for tests/test_gpu_bounds.py: every kernel family on edge-case
inputs, run against the bounds-checked library (POSPOP_LIBRARY =
libpospopcnt_b200_debug.so, every vector load asserts its index).  Any
out-of-range load traps the kernel and the process exits non-zero."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_02696_b200 as pp  # noqa: E402
import pyoracle  # noqa: E402


def run(name, var_env, fn):
    for key, val in var_env.items():
        os.environ[key] = val
    try:
        fn()
    finally:
        for key in var_env:
            os.environ.pop(key, None)
    torch.cuda.synchronize()
    print("ok", name, var_env, flush=True)


def main():
    assert "debug" in pp.library_path(), pp.library_path()
    torch.cuda.set_device(0)
    orc = pyoracle.Oracle()
    raw = orc.generate(6, 4, (6 << 20) // 8).view(np.uint8)
    pool = torch.from_numpy(raw.copy()).cuda()

    def counts():
        for k in (8, 16, 32, 64):
            wb = k // 8
            for off in sorted({0, wb, 3 * wb, 8, 16 - wb, 32 - wb}):
                for n in (0, 1, 7, 31, 33, 1000, 4097, 40_000, 300_001, (1 << 20) // wb + 5, (5 << 20) // wb):
                    view = pool[off:off + n * wb]  # data placed at the very start/end of the allocation region
                    assert pp.pospopcnt_k(view, k) == orc.pospopcnt(raw[off:off + n * wb], k, threads=4), (k, off, n)
    run("counts (small / cluster / stream kernels)", {}, counts)
    run("counts, stream kernel only", {"POSPOP_SMALL_BYTES": "0", "POSPOP_CLUSTER_BYTES": "0"}, counts)
    for var, tma in (("4,32,0,256,3", "8,6"),):  # a TMA variant instantiated for both bank counts
        run("counts, TMA", {"POSPOP_STREAM_VARIANT": var, "POSPOP_TMA": tma, "POSPOP_SMALL_BYTES": "0",
                            "POSPOP_CLUSTER_BYTES": "0"}, counts)

    flags = orc.generate(7, 9, (3 << 20) + 5)
    rc, want, _ = orc.flagstats(flags)
    fdev = torch.from_numpy(flags.view(np.uint8).copy()).cuda()

    def flag():
        for off in (0, 2, 6, 30):
            n = flags.size - off // 2 - 3
            got = pp.flagstats((fdev.data_ptr() + off, n)).as_list()
            assert got == list(orc.flagstats(flags[off // 2: off // 2 + n])[1])
    for v in ("", "6,32,0,512,2", "5,32,0,512,5,2", "4,32,0,512,4,2"):
        run("flagstats", {"POSPOP_FLAG_VARIANT": v} if v else {}, flag)
    # paired-end-like mix: rare QC-fail reads -> the fail-free fast path and its reload fix-up
    flags = orc.generate(8, 2, (3 << 20) + 5)
    flags[[0, 4097, 3 << 19]] |= 0x200
    fdev = torch.from_numpy(flags.view(np.uint8).copy()).cuda()
    run("flagstats, QC-fail prediction", {}, flag)

    rng = np.random.default_rng(5)
    for k in (8, 16, 32, 64):
        dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[k]
        data = raw.view(dt)
        lens = rng.integers(0, 3000, size=700)
        lens[[3, 50]] = [200_000, 0]
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        offs = offs[offs <= data.size]
        want_rows = orc.segmented(data, offs, k, threads=4)
        d = torch.from_numpy(data.view(np.uint8).copy()).cuda()
        o = torch.from_numpy(offs.view(np.int64)).cuda()
        variants = ["5,16,0", "5,16,1", "5,16,3", "5,16,6", "6,16,5,4", "6,16,5,8", "5,16,10,2"] if k < 64 else \
                   ["5,16,0", "5,16,1", "4,16,6", "4,16,5,8", "3,16,10,4"]
        auto = "4,16,8" if k == 64 else "5,16,8"

        def seg():
            out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
            pp.segmented_async(d, o, out, k)
            torch.cuda.synchronize()
            assert (out.cpu().numpy().view(np.uint64) == want_rows).all()
        for v in variants:
            run(f"segmented k={k}", {"POSPOP_SEG_VARIANT": v, "POSPOP_SEG_BIG_KIB": "64"}, seg)
        for lane, group, tile, rounds in ((1 << 20,) * 3 + (0,), (0, 1 << 20, 1 << 20, 0), (0, 0, 0, 0),
                                          (0, 0, 0, 255)):
            # adaptive: lane / grouped / tile / range modes
            for giant in ("1024", "16"):  # a 16 KiB giant bound: the queue carries the longer arrays
                run(f"segmented adaptive k={k}", {"POSPOP_SEG_VARIANT": auto, "POSPOP_SEG_LANE_MEAN_BYTES": str(lane),
                                                  "POSPOP_SEG_GROUP_MEAN_BYTES": str(group),
                                                  "POSPOP_SEG_TILE_MEAN_BYTES": str(tile),
                                                  "POSPOP_SEG_RANGE": str(rounds),
                                                  "POSPOP_SEG_GIANT_KIB": giant}, seg)
    print("bounds ok")


if __name__ == "__main__":
    main()
