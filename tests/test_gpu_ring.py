"""The per-warp bulk-copy ring kernel (SCHED 6: each warp stages its next
warp tiles in its own shared-memory slots with cp.async.bulk + mbarrier and
reads them with swizzled LDS.128) -- bit-exact against the oracle on the
same cases as the LDG kernel: every k, unaligned starts and ragged ends
inside 0xFF guard bytes (the edge tiles take the masked LDG path), forced
flushes, full size, and the FLAG mode including the first-invalid-word
report (found by reloading the tile in canonical order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

RING_STREAM = [("7,32,0,256,6", "8,1"), ("7,32,0,256,6", "4,3"), ("6,32,0,256,6", "16,1"), ("6,32,0,256,6", "12,2")]
RING_STREAM64 = [("6,32,0,256,6", "8,1")]
RING_FLAG = [("5,32,0,512,6,2", "16,1"), ("5,32,0,512,6,2", "12,2"), ("5,32,0,512,6,2", "8,3"),
             ("4,32,0,512,6,2", "16,2"), ("4,32,0,512,6,2", "16,3")]


def guarded(a, offset, guard=64):
    raw = a.view(np.uint8)
    buf = torch.full((guard + offset + raw.size + guard,), 0xFF, dtype=torch.uint8, device="cuda")
    buf[guard + offset:guard + offset + raw.size] = torch.from_numpy(raw.copy()).cuda()
    return buf, buf[guard + offset:guard + offset + raw.size]


@pytest.fixture(scope="module")
def dev(pp):
    assert torch.cuda.is_available() and pp.device_available()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_ring_stream_lengths_offsets(pp, tuning, dev, orc, k, monkeypatch):
    wb = k // 8
    raw = orc.generate(6, 17 + k, (5 << 20) // 8).view(np.uint8)
    lengths = [0, 1, 7, 31, 33, 1000, 4097, 65537, 300_001, raw.size // wb - 8]
    for var, ring in (RING_STREAM64 if k == 64 else RING_STREAM):
        monkeypatch.setenv("POSPOP_STREAM_VARIANT", var)
        monkeypatch.setenv("POSPOP_RING", ring)
        for offset in sorted({0, wb, 3 * wb, 8, 16 - wb}):
            for n in lengths:
                sub = raw[:n * wb]
                _, view = guarded(sub, offset)
                assert pp.pospopcnt_k(view, k) == orc.pospopcnt(sub, k, threads=4), (var, ring, k, offset, n)


def test_ring_forced_flush_and_full_size(pp, tuning, dev, orc, monkeypatch):
    monkeypatch.setenv("POSPOP_STREAM_VARIANT", "7,32,0,256,6")
    monkeypatch.setenv("POSPOP_RING", "8,1")
    raw = orc.generate(6, 5, 1 << 18).view(np.uint8)
    d = torch.from_numpy(raw.copy()).cuda()
    want = orc.naive(raw, 16)
    for thr in (1, 3, 65535):
        assert pp.pospopcnt_k(d, 16, flush_threshold_blocks=thr) == want
    n = 1 << 31  # 4 GiB of u16
    big = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG4, 3, big)
    got = pp.pospopcnt(big)
    monkeypatch.setenv("POSPOP_STREAM_VARIANT", "7,32,0,256,2")  # the LDG kernel on the same bytes
    assert pp.pospopcnt(big) == got
    assert got == orc.pospopcnt(big.cpu().numpy().view(np.uint16), 16, threads=16)


@pytest.mark.parametrize("var,ring", RING_FLAG)
@pytest.mark.parametrize("flush", [None, "1"])
def test_ring_flagstats(pp, tuning, dev, orc, golden, var, ring, flush, monkeypatch):
    monkeypatch.setenv("POSPOP_FLAG_VARIANT", var)
    monkeypatch.setenv("POSPOP_RING", ring)
    if flush:
        monkeypatch.setenv("POSPOP_FLUSH_THRESHOLD", flush)
    streams = orc.acceptance_flag_streams()
    for i in range(0, 100, 7):
        assert pp.flagstats(torch.from_numpy(streams[i].view(np.int16).copy()).cuda()).as_list() == \
            golden["flagstats_acceptance"][i]
    w = orc.generate(7, 5, (1 << 22) + 3)
    w[123457] |= 0x1000
    w[2_000_001] |= 0x8000
    for offset in (0, 2, 6):
        _, view = guarded(w, offset)
        with pytest.raises(pp.InvalidFlagWordError) as e:
            pp.flagstats(view)
        assert e.value.offset == 123457
    w[123457] &= 0x0FFF
    w[2_000_001] &= 0x0FFF
    rc, want, _ = orc.flagstats(w)
    _, view = guarded(w, 2)
    assert pp.flagstats(view).as_list() == list(want)
    for kind in (7, 8):  # 64 MiB: uniform FLAG words and the paired-end-like mix (QC-fail fix-up path)
        w = orc.generate(kind, 11, 1 << 25)
        rc, want, _ = orc.flagstats(w)
        assert pp.flagstats(torch.from_numpy(w.view(np.int16)).cuda()).as_list() == list(want), kind
