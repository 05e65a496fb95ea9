import sys, os, torch
sys.path.insert(0, '/root/repo')
import paper_1911_02696_b200 as pp
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
total = 1 << 30  # bytes of u32
d = torch.empty(total, dtype=torch.uint8, device='cuda')
pp.generate(pp.GEN_U32, 1, d, stream=s)
for arrays in (262144, 65536, 16384, 4096, 1024):
    words = (total // 4) // arrays
    offs = torch.arange(0, arrays + 1, dtype=torch.int64, device='cuda') * words
    o = torch.empty((arrays, 32), dtype=torch.int64, device='cuda')
    for _ in range(3): pp.segmented_async(d, offs, o, 32, stream=s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); pp.segmented_async(d, offs, o, 32, stream=s); b.record(s); b.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    print(arrays, words, round(total / (ts[len(ts)//2] * 1e-3) / 1e9, 1), "GB/s")
