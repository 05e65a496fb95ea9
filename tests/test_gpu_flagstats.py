"""FLAG statistics on the GPU: the fused one-pass kernel
behind pospop_flagstats() against the reference's golden summaries and the oracle.
Bit-exact.  Restates the reference's criterion 5 (acceptance.cpp:271-291) and
the reserved-bit error (flagstats.cpp:34-36)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(pp):
    assert torch.cuda.is_available() and pp.device_available()
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(a.view(np.uint8).copy()).cuda()


def test_single_values_exhaustive(pp, dev, golden):
    words = np.arange(4096, dtype=np.uint16)
    d = to_dev(words)
    for v in range(4096):
        got = pp.flagstats((d.data_ptr() + 2 * v, 1)).as_list()
        assert got == golden["flagstats_single"][v], v


def test_all_values_in_one_stream_and_offsets(pp, dev, orc):
    words = np.tile(np.arange(4096, dtype=np.uint16), 37)
    rc, want, _ = orc.flagstats(words)
    assert rc == 0
    for off in range(0, 34, 2):  # unaligned starts: masked head vectors
        buf = torch.full((words.nbytes + 128,), 0xFF, dtype=torch.uint8, device="cuda")  # invalid guards
        buf[64 + off:64 + off + words.nbytes] = torch.from_numpy(words.view(np.uint8).copy()).cuda()
        got = pp.flagstats((buf.data_ptr() + 64 + off, words.size)).as_list()
        assert got == list(want), off


def test_acceptance_streams(pp, dev, orc, golden):
    streams = orc.acceptance_flag_streams()
    for i in range(100):
        assert pp.flagstats(to_dev(streams[i])).as_list() == golden["flagstats_acceptance"][i], i
    for i in range(0, 100, 10):  # host-memory path
        assert pp.flagstats(streams[i]).as_list() == golden["flagstats_acceptance"][i], i


def test_invalid_word_first_offset(pp, dev, orc):
    w = orc.generate(7, 5, 1 << 20)
    w[700001] |= 0x4000
    w[123457] |= 0x1000
    w[999999] |= 0x8000
    for data in (to_dev(w), w):
        with pytest.raises(pp.InvalidFlagWordError) as e:
            pp.flagstats(data)
        assert e.value.offset == 123457 and e.value.word == int(w[123457])


def test_invalid_word_in_a_later_host_chunk(pp, dev, orc):
    n = (70 << 20) // 2 + 5  # two 64 MiB staging chunks
    w = orc.generate(7, 6, n, threads=8)
    w[n - 3] |= 0x2000
    with pytest.raises(pp.InvalidFlagWordError) as e:
        pp.flagstats(w)
    assert e.value.offset == n - 3
    w[n - 3] &= 0x0FFF
    rc, want, _ = orc.flagstats(w)
    assert pp.flagstats(w).as_list() == list(want)


def test_empty_and_full_size(pp, dev, orc):
    assert pp.flagstats(np.zeros(0, np.uint16)).total() == 0
    n = 1 << 28
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_FLAGS, 9, d)
    got = pp.flagstats(d)
    host = d.cpu().numpy().view(np.uint16)
    rc, want, _ = orc.flagstats(host)
    assert rc == 0 and got.as_list() == list(want)
    assert got.total() == n


FLAG_VARIANTS = ["5,32,0,512,2,2", "4,32,0,512,2,2", "4,32,2,256,2,2", "4,16,0,512,2,2", "6,32,0,256,2,2",
                 "5,32,0,256,2,2", "4,32,0,512,4,2", "3,32,0,512,4,2", "4,32,0,256,4,2", "5,32,0,512,5,2",
                 "5,16,0,512,5,2", "6,32,0,256,5,2", "6,32,0,512,2"]


@pytest.mark.parametrize("variant", FLAG_VARIANTS)
@pytest.mark.parametrize("flush", [None, "1", "3"])
def test_flag_kernel_variants(pp, tuning, dev, orc, golden, variant, flush, monkeypatch):
    """Every FLAG kernel instantiation (byte-frame MODE 2 and the 16-bit-lane
    MODE 1), with forced lane flushes, on the golden acceptance streams, all
    4096 values at unaligned starts, and the first-invalid-word report."""
    monkeypatch.setenv("POSPOP_FLAG_VARIANT", variant)
    if flush:
        monkeypatch.setenv("POSPOP_FLUSH_THRESHOLD", flush)
    streams = orc.acceptance_flag_streams()
    for i in range(0, 100, 9):
        assert pp.flagstats(to_dev(streams[i])).as_list() == golden["flagstats_acceptance"][i], i
    words = np.tile(np.arange(4096, dtype=np.uint16), 301)
    rc, want, _ = orc.flagstats(words)
    for off in (0, 2, 6, 30):
        buf = torch.full((words.nbytes + 128,), 0xFF, dtype=torch.uint8, device="cuda")
        buf[64 + off:64 + off + words.nbytes] = torch.from_numpy(words.view(np.uint8).copy()).cuda()
        assert pp.flagstats((buf.data_ptr() + 64 + off, words.size)).as_list() == list(want), off
    w = orc.generate(7, 11, (1 << 21) + 7)
    w[1_500_001] |= 0x8000
    w[77_777] |= 0x1000
    with pytest.raises(pp.InvalidFlagWordError) as e:
        pp.flagstats(to_dev(w))
    assert e.value.offset == 77_777


def test_flag_byte_frame_full_size_flushes(pp, tuning, dev, orc, monkeypatch):
    """8 GiB-class input at the default variant: every thread crosses the
    255-block byte-lane flush several times."""
    n = 1 << 31
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_FLAGS, 21, d)
    got = pp.flagstats(d).as_list()
    monkeypatch.setenv("POSPOP_FLAG_VARIANT", "6,32,0,512,2")  # the 16-bit-lane kernel on the same words
    assert pp.flagstats(d).as_list() == got
    host = d.cpu().numpy().view(np.uint16)
    del d
    rc, want, _ = orc.flagstats(host[: 1 << 26])
    monkeypatch.delenv("POSPOP_FLAG_VARIANT")
    assert pp.flagstats(host[: 1 << 26]).as_list() == list(want)


@pytest.mark.parametrize("variant", ["", "5,16,0,512,2,2", "6,32,0,256,2,2"])
def test_qcfail_fast_path_and_fixup(pp, tuning, dev, orc, variant, monkeypatch):
    """The byte-frame kernel predicts fail-free tiles and counts only AL/AH
    there; a tile that turns out to hold a QC-fail read is reloaded and its
    fail planes added.  Paired-end-like mix (kind 8: QC-fail 2^-16, so most
    tiles take the fast path and some the fix-up), plus hand-placed QC-fail
    words at tile starts, ends and in isolated tiles, and a fail-free stream."""
    if variant:
        monkeypatch.setenv("POSPOP_FLAG_VARIANT", variant)
    n = (1 << 24) + 77
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_FLAGMIX, 5, d)
    host = d.cpu().numpy().view(np.uint16).copy()
    assert 0 < int(((host & 0x200) != 0).sum()) < n // 1000  # rare but present
    for w in (host, host & np.uint16(0x0DFF)):                # with and without any QC-fail read
        rc, want, _ = orc.flagstats(w)
        assert rc == 0
        assert pp.flagstats(torch.from_numpy(w.view(np.int16).copy()).cuda()).as_list() == list(want)
    w = host & np.uint16(0x0DFF)
    for pos in (0, 1, 4095, 4096, 65535, 1 << 20, (1 << 20) + 1, n - 1):
        w[pos] |= 0x200
    rc, want, _ = orc.flagstats(w)
    for off in (0, 2, 6):  # unaligned starts shift tile boundaries
        buf = torch.zeros(n + 64, dtype=torch.int16, device="cuda")
        buf[off // 2: off // 2 + n] = torch.from_numpy(w.view(np.int16).copy()).cuda()
        assert pp.flagstats(buf[off // 2: off // 2 + n]).as_list() == list(want), off


def test_flagmix_generator_matches_oracle(pp, dev, orc):
    n = (1 << 20) + 3
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_FLAGMIX, 11, d, base=12345)
    assert (d.cpu().numpy().view(np.uint16) == orc.generate(8, 11, n, base=12345)).all()


def test_small_host_inputs_read_in_place(pp, dev, orc):
    """Pinned FLAG words up to 2 MiB and pageable ones up to 1 MiB are read
    in place by the ring kernel (cp.async.bulk from mapped host memory):
    summaries and the first invalid word's offset as the reference."""
    w = orc.generate(7, 9, (1 << 20) - 3)  # just under 2 MiB
    t = torch.empty(w.nbytes + 64, dtype=torch.uint8, pin_memory=True)
    for off in (0, 2, 6, 34):
        pv = t.numpy()[off:off + w.nbytes].view(np.uint16)
        pv[:] = w
        rc, want, _ = orc.flagstats(w)
        assert pp.flagstats(pv).as_list() == list(want), off
        small = w[: (1 << 18) + 1]  # pageable, < 1 MiB
        rc, want_s, _ = orc.flagstats(small)
        assert pp.flagstats(small.copy()).as_list() == list(want_s), off
    pv = t.numpy()[2:2 + w.nbytes].view(np.uint16)
    pv[:] = w
    pv[777777] |= 0x4000
    pv[4099] |= 0x1000
    with pytest.raises(pp.InvalidFlagWordError) as e:
        pp.flagstats(pv)
    assert e.value.offset == 4099 and e.value.word == int(pv[4099])
