"""The latency-path kernels: the single-CTA small-input
kernel and the one-cluster medium kernel (distributed-shared-memory reduce),
bit-exact against the oracle for every k at every length up to the switch
sizes, at unaligned starts inside 0xFF guard bytes, for overwrite and
accumulate, and equal to the multi-CTA stream kernel on the same bytes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(pp):
    assert torch.cuda.is_available() and pp.device_available()
    torch.cuda.set_device(0)


def guarded(raw, offset, guard=64):
    buf = torch.full((guard + offset + raw.size + guard,), 0xFF, dtype=torch.uint8, device="cuda")
    buf[guard + offset:guard + offset + raw.size] = torch.from_numpy(raw.copy()).cuda()
    return buf[guard + offset:guard + offset + raw.size]


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_small_path_lengths_offsets(pp, tuning, dev, orc, k, monkeypatch):
    wb = k // 8
    raw = orc.generate(6, 40 + k, (40 << 10) // 8).view(np.uint8)
    lengths = sorted({0, 1, 2, 3, 31, 32, 33, 255, 256, 1000, 1023, 1024, 4095, 4096, 4097,
                      (16 << 10) // wb + 1, (32 << 10) // wb - 1, (32 << 10) // wb})
    for offset in sorted({0, wb, 3 * wb, 8, 16 - wb}):
        for n in lengths:
            sub = raw[:n * wb]
            view = guarded(sub, offset)
            want = orc.naive(sub, k) if n < 4096 else orc.pospopcnt(sub, k, threads=2)
            got = pp.pospopcnt_k(view, k)
            assert got == want, (k, offset, n)
            monkeypatch.setenv("POSPOP_SMALL_BYTES", "0")  # the multi-CTA stream kernel
            assert pp.pospopcnt_k(view, k) == want, (k, offset, n)
            monkeypatch.delenv("POSPOP_SMALL_BYTES")


@pytest.mark.parametrize("k", [16, 64])
def test_small_kernel_multi_tile_and_accumulate(pp, tuning, dev, orc, k, monkeypatch):
    """Raising the switch size makes the one CTA loop over many tiles."""
    monkeypatch.setenv("POSPOP_SMALL_BYTES", str(4 << 20))
    raw = orc.generate(6, 7, (3 << 20) // 8 + 5).view(np.uint8)[: (3 << 20) + 24]
    want = orc.pospopcnt(raw, k, threads=4)
    d = torch.from_numpy(raw.copy()).cuda()
    assert pp.pospopcnt_k(d, k) == want
    out = torch.zeros(k, dtype=torch.int64, device="cuda")
    for _ in range(3):
        pp.count_async(d, out, k, accumulate=True)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().astype(np.uint64) == 3 * np.asarray(want, np.uint64)).all()


def test_small_path_launches_one_kernel(pp, dev, orc):
    words = orc.generate(1, 3, 1024)
    d = torch.from_numpy(words.view(np.int16).copy()).cuda()
    n0 = pp.kernel_launches()
    assert pp.pospopcnt(d) == orc.pospopcnt(words, 16)
    assert pp.kernel_launches() - n0 == 1


@pytest.mark.parametrize("k", [8, 16, 32, 64])
@pytest.mark.parametrize("csize", ["16", "8"])
def test_cluster_kernel_lengths_offsets_accumulate(pp, tuning, dev, orc, k, csize, monkeypatch):
    monkeypatch.setenv("POSPOP_SMALL_BYTES", "0")
    monkeypatch.setenv("POSPOP_CLUSTER_BYTES", str(64 << 20))
    monkeypatch.setenv("POSPOP_CLUSTER", csize)
    wb = k // 8
    raw = orc.generate(6, 90 + k, (5 << 20) // 8).view(np.uint8)
    for offset in sorted({0, wb, 3 * wb, 8, 16 - wb}):
        for n in (0, 1, 33, 4097, 65537, 300_001, (1 << 20) // wb + 3, raw.size // wb - 8):
            sub = raw[:n * wb]
            view = guarded(sub, offset)
            assert pp.pospopcnt_k(view, k) == orc.pospopcnt(sub, k, threads=4), (k, csize, offset, n)
    d = torch.from_numpy(raw.copy()).cuda()
    out = torch.zeros(k, dtype=torch.int64, device="cuda")
    for _ in range(3):
        pp.count_async(d, out, k, accumulate=True)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().astype(np.uint64) == 3 * np.asarray(orc.pospopcnt(raw, k, threads=4), np.uint64)).all()
