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


def prmt(a, b, sel, sign_ok=True):
    """PTX prmt.b32 default mode: byte n of the result = byte (sel >> 4n) & 7 of
    {b, a}; selector msb set -> that byte's sign bit replicated."""
    src = (b.astype(np.uint64) << np.uint64(32)) | a.astype(np.uint64)
    out = np.zeros_like(a, dtype=np.uint32)
    for n in range(4):
        nib = (sel >> (4 * n)) & 0xF
        byte = ((src >> np.uint64(8 * (nib & 7))) & np.uint64(0xFF)).astype(np.uint32)
        if nib & 8:
            byte = np.where(byte & 0x80, np.uint32(0xFF), np.uint32(0)).astype(np.uint32)
        out |= byte << np.uint32(8 * n)
    return out


def flag_leaf(r0, r1):
    """Mirror of flag_leaf (byte-frame FLAG kernel, MODE 2): (al, fl, ahf, hb)."""
    u = np.uint32
    B1 = u(0x01010101)
    lb = prmt(r0, r1, 0x6420)
    hb = prmt(r0, r1, 0x7531)
    g = lb & ~hb & ~umulhi(hb, 1 << 29) & B1
    gu = g & ~umulhi(lb, 1 << 30)
    t = (g * u(0xC0) + gu * u(0x0B)).astype(u)
    al = lb & (t | u(0x04040404))
    mf = prmt((hb * u(1 << 6)).astype(u), np.zeros_like(hb), 0xBA98)
    fl = al & mf
    ah = hb & ~((hb * u(1 << 3)).astype(u) & u(0x08080808))
    ahf = ah | ((ah * u(1 << 4)).astype(u) & mf)
    return al, fl, ahf, hb


def byte_frame_positions(al, fl, ahf, slot):
    """Per-word transform positions (flagstats.cpp:39-49) rebuilt from the
    three byte planes the way the kernel's epilogue folds them."""
    u = np.uint32
    sh = u(8 * slot)
    a, f, h = (al >> sh) & u(0xFF), (fl >> sh) & u(0xFF), (ahf >> sh) & u(0xFF)

    def plane(x, hx):
        out = np.zeros_like(x)
        for p in (1, 2, 3, 6, 7):
            out |= ((x >> u(p)) & u(1)) << u(p)
        for j in range(4):
            out |= ((hx >> u(j)) & u(1)) << u(8 + j)
        out |= (((x & ~(x >> u(3))) & u(1))) << u(12)  # pair_map = GU & !(GU & mate_unmapped)
        return out
    return plane(a, h), plane(f, h >> u(4))


def test_byte_frame_flag_leaf_exhaustive(orc):
    refp = np.zeros(4096, np.uint32)
    reff = np.zeros(4096, np.uint32)
    for v in range(4096):
        refp[v], reff[v] = orc.flag_transform(v)
    rng = np.random.default_rng(7)
    n = 4096 * 32
    for slot in range(4):
        words = rng.integers(0, 4096, size=(n, 4), dtype=np.uint32)
        words[:, slot] = np.tile(np.arange(4096, dtype=np.uint32), 32)
        r0 = words[:, 0] | (words[:, 1] << np.uint32(16))
        r1 = words[:, 2] | (words[:, 3] << np.uint32(16))
        al, fl, ahf, hb = flag_leaf(r0, r1)
        assert not (hb & np.uint32(0xF0F0F0F0)).any()
        for s in range(4):
            a, f = byte_frame_positions(al, fl, ahf, s)
            src = words[:, s]
            assert (a == ((refp[src] | reff[src]) & NEEDED)).all(), (slot, s)
            assert (f == (reff[src] & NEEDED)).all(), (slot, s)


def test_byte_frame_reserved_bits_reach_bad():
    rng = np.random.default_rng(9)
    words = rng.integers(0, 4096, size=(4096, 4), dtype=np.uint32)
    slot = np.arange(4096) % 4
    words[np.arange(4096), slot] |= np.uint32(0x1000) << (np.arange(4096) % 4).astype(np.uint32)
    r0 = words[:, 0] | (words[:, 1] << np.uint32(16))
    r1 = words[:, 2] | (words[:, 3] << np.uint32(16))
    *_, hb = flag_leaf(r0, r1)
    assert ((hb & np.uint32(0xF0F0F0F0)) != 0).all()
