import sys, time, ctypes as C
sys.path.insert(0, '/root/repo')
import torch, paper_1911_02696_b200 as pp
torch.cuda.set_device(0)
n = 1 << 32
d = torch.empty(n, dtype=torch.int16, device='cuda')
pp.generate(pp.GEN_FLAGMIX, 1, d)
lib = pp._load(); summ = pp._Summary()
def t(label):
    for _ in range(3): lib.pospop_flagstats(d.data_ptr(), n, C.byref(summ), None, None)
    ts = []
    for _ in range(7):
        a = time.perf_counter(); lib.pospop_flagstats(d.data_ptr(), n, C.byref(summ), None, None); ts.append(time.perf_counter() - a)
    ts.sort(); print(label, round(2 * n / ts[3] / 1e9, 1), "GB/s", flush=True)
t("mix (QC-fail 2^-16)")
d.bitwise_and_(0x0DFF); torch.cuda.synchronize()
t("mix without QC-fail")
pp.generate(pp.GEN_FLAGS, 1, d); torch.cuda.synchronize()
t("uniform")
d.bitwise_and_(0x0DFF); torch.cuda.synchronize()
t("uniform without QC-fail")
