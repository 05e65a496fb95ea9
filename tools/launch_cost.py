#!/usr/bin/env python
"""Host cost of one pospopcnt_async call through the C ABI (measurement tool):
CPU microseconds per call without synchronising, and per launch including the
device work, for a tiny, a 4 MiB and a 64 MiB input; plus the ctypes floor.

    python tools/launch_cost.py
"""
import time, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, ctypes as C
import paper_1911_02696_b200 as pp
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
lib = pp._load()
lib.pospopcnt_async.argtypes = [C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_void_p]
for nbytes in (4096, 4 << 20, 64 << 20):
    d = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    args = (16, d.data_ptr(), nbytes // 2, out.data_ptr(), 0, 65535, 0, 0, C.c_void_p(s.cuda_stream))
    for _ in range(100): lib.pospopcnt_async(*args)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n): lib.pospopcnt_async(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{nbytes}: host {1e6*(t1-t0)/n:.2f} us/call, total {1e6*(t2-t0)/n:.2f} us/launch")
    # python overhead floor: empty ctypes call
lib.pospop_kernel_launches.restype = C.c_uint64
t0 = time.perf_counter()
for _ in range(20000): lib.pospop_kernel_launches()
print(f"ctypes floor {1e6*(time.perf_counter()-t0)/20000:.2f} us")
