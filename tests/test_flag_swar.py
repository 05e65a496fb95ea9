"""The SWAR FLAG transform used by the fused FLAG-statistics kernel
(flag_transform2 in paper_1911_02696_b200/csrc/pospop_stream.cuh), emulated
op for op in numpy and checked against the oracle's restatement of the
reference's flag_transform (proj/core/src/flagstats.cpp:94-125) on ALL
4096 x 4096 pairs of valid FLAG words packed in one 32-bit register.
Only the positions bucket_from_counts reads (flagstats.cpp:39-63) matter."""
import numpy as np

NEEDED = 0x1FCE  # positions 1,2,3,6,7,8,9,10,11,12


def umulhi(x, m):
    return ((x.astype(np.uint64) * np.uint64(m)) >> np.uint64(32)).astype(np.uint32)


def swar_transform(w):
    """Mirror of flag_transform2: returns (all, fail) planes."""
    L1 = np.uint32(0x00010001)
    g0 = w & ~umulhi(w, 1 << 24) & ~umulhi(w, 1 << 21)  # w & ~(w >> 8) & ~(w >> 11)
    g = g0 & L1
    gu = g0 & ~umulhi(w, 1 << 30) & L1                 # & ~(w >> 2)
    t = (g * np.uint32(0x00C0) + gu * np.uint32(0x100A)).astype(np.uint32)
    mf = ((umulhi(w, 1 << 23) & L1) * np.uint32(0xFFFF)).astype(np.uint32)  # (w >> 9) lane mask
    all_ = ((w & (t | np.uint32(0x07040704))) | (t & ~(w * np.uint32(1 << 9)) & np.uint32(0x10001000))
            | (w & ~(w * np.uint32(1 << 3)) & np.uint32(0x08000800)))
    return all_, all_ & mf


def test_swar_flag_transform_exhaustive(orc):
    refp = np.zeros(4096, np.uint32)
    reff = np.zeros(4096, np.uint32)
    for v in range(4096):
        refp[v], reff[v] = orc.flag_transform(v)
    lo = np.repeat(np.arange(4096, dtype=np.uint32), 4096)
    hi = np.tile(np.arange(4096, dtype=np.uint32), 4096)
    all_, fail = swar_transform(lo | (hi << np.uint32(16)))
    for shift, src in ((0, lo), (16, hi)):
        a = (all_ >> np.uint32(shift)) & np.uint32(NEEDED)
        f = (fail >> np.uint32(shift)) & np.uint32(NEEDED)
        assert (a == ((refp[src] | reff[src]) & NEEDED)).all()
        assert (f == (reff[src] & NEEDED)).all()
        # pass = all - fail position-wise, as the host derives it
        assert ((a & ~f) == (refp[src] & NEEDED)).all()
