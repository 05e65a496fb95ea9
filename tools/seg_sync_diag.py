import sys, time, os
os.environ.setdefault("POSPOP_LIBRARY", "tuning")  # POSPOP_* knobs: the tuning build
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1911_02696_b200 as pp
torch.cuda.set_device(0)
arrays, words = 65536, 4096
for k, kind in ((32, 5), (64, 6)):
    d = torch.empty(arrays * words * k // 8, dtype=torch.uint8, device='cuda')
    pp.generate(kind, 1, d)
    host = torch.empty(d.numel(), dtype=torch.uint8, pin_memory=True); host.copy_(d)
    offs = np.arange(arrays + 1, dtype=np.uint64) * words
    rows = np.empty((arrays, k), np.uint64)
    for var in (None, "5,16,3", "5,16,6", "5,16,1"):
        if var: os.environ["POSPOP_SEG_VARIANT"] = var
        else: os.environ.pop("POSPOP_SEG_VARIANT", None)
        pp.pospopcnt_segmented(host.numpy(), offs, k, out=rows)
        t0 = time.perf_counter()
        for _ in range(3): pp.pospopcnt_segmented(host.numpy(), offs, k, out=rows)
        dt = (time.perf_counter() - t0) / 3
        do = torch.from_numpy(offs.view(np.int64)).cuda(); dr = torch.empty((arrays, k), dtype=torch.int64, device='cuda')
        torch.cuda.synchronize(); t1 = time.perf_counter()
        for _ in range(3): pp.segmented_async(d, do, dr, k)
        torch.cuda.synchronize(); da = (time.perf_counter() - t1) / 3
        print(k, var, "sync host %.1f ms" % (dt * 1e3), "async dev %.3f ms" % (da * 1e3), flush=True)
