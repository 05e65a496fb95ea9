"""Parity of the sm_100a path against the oracle and the reference's golden
vectors.  Bit-exact (integer counts, zero tolerance).  Every call goes through
the C ABI (libpospopcnt_b200.so) via the package's ctypes mirror."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

COUNTRY = np.array([0x10, 0x10, 0x04, 0x10, 0x01, 0x04, 0x01, 0x01, 0x01, 0x20], np.uint16)


@pytest.fixture(scope="module")
def dev(pp):
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a GPU")
    torch.cuda.set_device(0)
    assert pp.device_available()
    return torch.device("cuda:0")


def to_dev(a: np.ndarray):
    return torch.from_numpy(a.view(np.uint8).copy()).cuda()


def guarded(a: np.ndarray, offset: int, guard: int = 64, fill: int = 0xFF):
    """Device copy of `a` placed `offset` bytes past a 256 B-aligned base, with
    0xFF guard bytes on both sides (an over-read would count them)."""
    raw = a.view(np.uint8)
    buf = torch.full((guard + offset + raw.size + guard,), fill, dtype=torch.uint8, device="cuda")
    buf[guard + offset:guard + offset + raw.size] = torch.from_numpy(raw.copy()).cuda()
    return buf, buf[guard + offset:guard + offset + raw.size]


def expect(got, want):
    assert [int(x) for x in got] == [int(x) for x in want]


# -- reference KATs through the reference entry point --------------------------------

def test_country_empty_allones(pp, dev):
    for data in (COUNTRY, to_dev(COUNTRY)):
        c = pp.pospopcnt(data)
        assert c[0] == 4 and c[2] == 2 and c[4] == 3 and c[5] == 1 and c.total() == 10
    assert pp.pospopcnt(np.zeros(0, np.uint16)) == pp.PositionalCounts()
    assert pp.pospopcnt(torch.zeros(0, dtype=torch.int16, device="cuda")) == pp.PositionalCounts()
    assert pp.pospopcnt(to_dev(np.array([0xFFFF], np.uint16))) == [1] * 16
    c = pp.pospopcnt(to_dev(np.full(100, 1, np.uint16)))
    assert c[0] == 100 and c.total() == 100


def test_exhaustive_single_word_domain_stream(pp, dev):
    words = np.arange(65536, dtype=np.uint16)
    d = to_dev(words)
    want = ((words[:, None].astype(np.uint32) >> np.arange(16)) & 1)
    for v in range(0, 65536, 1):
        got = pp.pospopcnt_k((d.data_ptr() + 2 * v, 1), 16)
        assert (got.counts == want[v]).all(), v


def test_exhaustive_single_word_domain_segmented(pp, dev):
    words = np.arange(65536, dtype=np.uint16)
    offs = torch.arange(65537, dtype=torch.int64, device="cuda")
    out = torch.zeros((65536, 16), dtype=torch.int64, device="cuda")
    pp.pospopcnt_segmented(to_dev(words), offs, 16, out=out)
    want = ((words[:, None].astype(np.int64) >> np.arange(16)) & 1)
    assert (out.cpu().numpy() == want).all()


@pytest.mark.parametrize("key", ["acceptance_random", "dispatcher_random", "csa_tails", "auto_boundary"])
def test_reference_random_streams(pp, dev, orc, golden, key):
    for seed, n, *want in golden[key]:
        w = orc.mt_generate_stream(seed, n)
        expect(pp.pospopcnt(to_dev(w)), want)
    for seed, n, *want in golden[key][:20]:  # host-memory path
        expect(pp.pospopcnt(orc.mt_generate_stream(seed, n)), want)


def test_concat_fork_join_order(pp, dev, orc, golden):
    for seed, n, cut, *want in golden["concat_cuts"]:
        d = to_dev(orc.mt_generate_stream(seed, n))
        a = pp.pospopcnt_k((d.data_ptr(), cut), 16)
        b = pp.pospopcnt_k((d.data_ptr() + 2 * cut, n - cut), 16)
        expect(pp.merge_counts(a, b), want)
    seed, n, *want = golden["fork_join"]
    d = to_dev(orc.mt_generate_stream(seed, n))
    parts = [pp.pospopcnt_k((d.data_ptr() + 2 * (i * n // 4), (i + 1) * n // 4 - i * n // 4), 16) for i in range(4)]
    total = parts[0]
    for p in parts[1:]:
        total = pp.merge_counts(total, p)
    expect(total, want)
    w = orc.mt_generate_stream(17, 1234)
    assert pp.pospopcnt(to_dev(w)) == pp.pospopcnt(to_dev(np.random.default_rng(4).permutation(w)))


def test_cfg1_uint32_counters(pp, dev, orc, golden):
    c = golden["cfg1"]
    w = orc.mt_generate_stream(c["seed"], c["len"])
    counters = np.zeros(16, np.uint32)
    pp.pospopcnt_u16_c32(to_dev(w), counters)
    expect(counters, c["counts"])
    pp.pospopcnt_u16_c32(w, counters)  # Fig. 6 accumulates
    expect(counters, [2 * x for x in c["counts"]])


def test_config_errors_like_reference(pp, dev):  # test_core.cpp:184-201
    w = to_dev(np.zeros(8, np.uint16))
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt(w, pp.PospopcntConfig(kernel=pp.KernelKind.Csa16, register_width_bits=128))
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt(w, pp.PospopcntConfig(flush_threshold_blocks=0))
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt(w, pp.PospopcntConfig(kernel=pp.KernelKind.Forest, register_width_bits=256))
    for kind in pp.KernelKind:  # every kind yields identical counts
        for width in [0] + pp.supported_csa_widths():
            if kind == pp.KernelKind.Forest and width > 64:
                continue
            if kind == pp.KernelKind.ByteBlend and width == 512:
                continue
            assert pp.pospopcnt(w, pp.PospopcntConfig(kernel=kind, register_width_bits=width)).total() == 0


# -- forced flushes, lane saturation --------------------------------------------------------

def test_forced_flush_thresholds(pp, dev, orc, golden):
    for key in ("acceptance_flush3", "csa_flush3"):
        for seed, n, *want in golden[key]:
            d = to_dev(orc.mt_generate_stream(seed, n))
            for thr in (1, 2, 3):
                expect(pp.pospopcnt(d, pp.PospopcntConfig(kernel=pp.KernelKind.Csa16,
                                                          flush_threshold_blocks=thr)), want)
                out = torch.zeros(16, dtype=torch.int64, device="cuda")
                for grid, block in ((1, 32), (1, 64), (3, 96), (0, 0)):
                    pp.count_async(d, out, 16, flush_threshold_blocks=thr, grid=grid, block=block)
                    torch.cuda.synchronize()
                    expect(out.cpu().numpy(), want)
    seed, n, *want = golden["csa_flush1"]
    expect(pp.pospopcnt(to_dev(orc.mt_generate_stream(seed, n)), pp.PospopcntConfig(flush_threshold_blocks=1)),
           want)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_forced_flush_all_k_small_grid(pp, dev, orc, k):
    raw = orc.generate(6, 7, 1 << 17).view(np.uint8)
    d = to_dev(raw)
    want = orc.naive(raw, k)
    out = torch.zeros(k, dtype=torch.int64, device="cuda")
    for thr in (1, 3, 7, 65535):
        for grid, block in ((1, 32), (2, 128), (5, 256)):
            pp.count_async(d, out, k, flush_threshold_blocks=thr, grid=grid, block=block)
            torch.cuda.synchronize()
            expect(out.cpu().numpy(), want)


def test_lane_saturation_single_warp(pp, dev):
    """test_csa.cpp:294-305 on the GPU: one CTA of 32 threads over all-ones
    input, > 65535 tree blocks per thread, so every 16-bit lane reaches 65535
    before the flush; one more block plus a tail proves no lane wrapped."""
    per_block_bytes = 32 * 512  # 32 threads x 128 registers x 4 B (depth 7; depth <= 7 sees more blocks)
    nbytes = per_block_bytes * 65537 + 6
    d = torch.full((nbytes,), 0xFF, dtype=torch.uint8, device="cuda")
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    pp.count_async(d, out, 16, grid=1, block=32)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == nbytes // 2).all()
    out8 = torch.zeros(8, dtype=torch.int64, device="cuda")
    pp.count_async(d, out8, 8, grid=1, block=32)
    torch.cuda.synchronize()
    assert (out8.cpu().numpy() == nbytes).all()


# -- ragged lengths x unaligned starts, all k -------------------------------------------------

@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_lengths_and_offsets(pp, dev, orc, k):
    wb = k // 8
    rng = np.random.default_rng(k)
    raw = orc.generate(6, 11, 1 << 13).view(np.uint8)  # 64 KiB of random bytes
    lengths = list(range(0, 70)) + [255, 256, 257, 1023, 1024, 1025, 4095, 4096, 4097] + \
        [int(x) for x in rng.integers(0, raw.size // wb - 8, size=30)]
    for offset in range(0, 16, wb):
        for n in lengths:
            sub = raw[:n * wb]
            buf, view = guarded(sub, offset)
            got = pp.pospopcnt_k(view, k)
            assert got == orc.naive(sub, k), (k, offset, n)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_medium_random_vs_oracle(pp, dev, orc, k):
    raw = orc.generate(6, 5, (3 << 20) + 5).view(np.uint8)
    for n_bytes in (1 << 20, (1 << 21) + 24, raw.size - 8):
        n = n_bytes // (k // 8)
        sub = raw[:n * k // 8]
        want = orc.pospopcnt(sub, k, threads=4)
        for offset in sorted({0, k // 8, 3 * (k // 8), 8, 16 - k // 8}):
            _, view = guarded(sub, offset)  # 0xFF guards: a missed head/tail mask counts them
            assert pp.pospopcnt_k(view, k) == want, (k, n, offset)
            _, view = guarded(sub[k // 8:], offset)  # ragged end too
            assert pp.pospopcnt_k(view, k) == orc.pospopcnt(sub[k // 8:], k, threads=4), (k, n, offset)


# -- host-memory (staged) path -----------------------------------------------------------------

def test_host_pageable_and_pinned_multi_chunk(pp, dev, orc):
    n = (150 << 20) // 2 + 7  # > two 64 MiB staging chunks, ragged
    w = orc.generate(4, 3, n, threads=8)
    want = orc.pospopcnt(w, 16, threads=8)
    assert pp.pospopcnt(w) == want
    pinned = torch.empty(n, dtype=torch.int16).pin_memory()
    pinned.numpy().view(np.uint16)[:] = w
    assert pp.pospopcnt(pinned) == want
    b = orc.generate(3, 9, (70 << 20) + 3, threads=8)
    assert pp.pospopcnt_k(b[3:], 8) == orc.pospopcnt(b[3:], 8, threads=8)


def test_threads_are_independent(pp, dev, orc):
    data = [orc.generate(6, s, 1 << 18) for s in range(6)]
    want = [orc.naive(d, 64) for d in data]
    errors = []

    def worker(i):
        try:
            d = to_dev(data[i])
            for _ in range(5):
                if pp.pospopcnt_k(d, 64) != want[i]:
                    errors.append(i)
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors


def test_async_accumulate(pp, dev, orc):
    w = orc.generate(1, 2, 1 << 20)
    d = to_dev(w)
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pp.count_async(d, out, 16, stream=s)
        pp.count_async(d, out, 16, accumulate=True, stream=s)
    s.synchronize()
    assert (out.cpu().numpy() == 2 * orc.naive(w).astype(np.int64)).all()


# -- segmented ---------------------------------------------------------------------------------

@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_segmented_ragged(pp, dev, orc, k):
    rng = np.random.default_rng(100 + k)
    n_words = 200_000
    data = orc.generate(6, 13, n_words * k // 64 + 1).view(DT[k])[:n_words]
    cuts = np.sort(rng.integers(0, n_words, size=3000))
    offs = np.concatenate([[0], cuts, [n_words], [n_words]]).astype(np.uint64)  # includes empty arrays
    got = pp.pospopcnt_segmented(to_dev(data), torch.from_numpy(offs.view(np.int64)).cuda(), k)
    want = orc.segmented(data, offs, k, threads=8)
    assert (got == want).all()
    # host inputs too
    assert (pp.pospopcnt_segmented(data, offs, k) == want).all()


DT = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_segmented_host_pipeline(pp, dev, orc, k):
    """Host data above 8 MiB takes the chunked path (H2D / launch / row D2H
    overlapped through the bounded staging ring, units cut at array
    boundaries): pinned and pageable data, rows in pageable / pinned host
    memory and on the device, host and device offsets, offsets[0] > 0 at an
    odd word, empty arrays, a 100 MiB array counted in pieces by the stream
    kernel, a 33 MiB one, and arrays straddling every unit edge."""
    wb = k // 8
    rng = np.random.default_rng(7 + k)
    n_words = (170 << 20) // wb + 5
    data = orc.generate(6, 21 + k, n_words * wb // 8 + 1, threads=8).view(DT[k])[:n_words]
    big_lo = n_words // 5
    big = (100 << 20) // wb + 1  # longer than a staging unit: four pieces through the stream kernel
    cuts = np.concatenate([rng.integers(3, big_lo, size=5000),
                           [big_lo, big_lo + big, big_lo + big, big_lo + big + (33 << 20) // wb],  # + empty, 33 MiB
                           rng.integers(big_lo + big + (33 << 20) // wb, n_words - 1, size=3000)])
    offs = np.concatenate([[3], np.sort(cuts), [n_words - 1]]).astype(np.uint64)
    want = orc.segmented(data, offs, k, threads=8)
    pinned = torch.empty(data.nbytes, dtype=torch.uint8).pin_memory()
    pinned.numpy()[:] = data.view(np.uint8)
    pinned_data = pinned.numpy().view(DT[k])
    n = offs.size - 1
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    for src in (data, pinned_data):
        assert (pp.pospopcnt_segmented(src, offs, k) == want).all()  # pageable rows
        rows = torch.zeros((n, k), dtype=torch.int64).pin_memory()
        pp.pospopcnt_segmented(src, d_offs, k, out=rows.numpy().view(np.uint64))  # pinned rows, device offsets
        assert (rows.numpy().view(np.uint64) == want).all()
        d_rows = torch.zeros((n, k), dtype=torch.int64, device="cuda")
        pp.pospopcnt_segmented(src, offs, k, out=d_rows)  # device rows
        assert (d_rows.cpu().numpy().view(np.uint64) == want).all()


# -- generators: device bytes == oracle bytes ------------------------------------------------

def test_device_generators_match_oracle(pp, dev, orc, golden_generators):
    esize = {1: 2, 2: 2, 3: 1, 4: 2, 5: 4, 6: 8, 7: 2, 8: 2}
    for key, v in golden_generators.items():
        kind, seed, base = (int(x) for x in key.split(":"))
        buf = torch.zeros((1 << 16) * esize[kind] + 8, dtype=torch.uint8, device="cuda")
        pp.generate(kind, seed, buf, base=base, n=1 << 16)
        torch.cuda.synchronize()
        host = buf[:(1 << 16) * esize[kind]].cpu().numpy()
        assert pp.digest(buf[:(1 << 16) * esize[kind]]) == v["digest"], key
        assert orc.digest(host) == v["digest"], key


# -- full-size BASELINE.json configs ------------------------------------------------------------

def test_cfg2_one_hot_zipf_full(pp, dev, orc):
    n = 1 << 28
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG2, 1, d)
    c = pp.pospopcnt(d)
    assert c.total() == n  # one-hot: exactly one bit per word
    assert c[0] > c[1] > c[2] > c[15]
    host = d.cpu().numpy().view(np.uint16)
    assert c == orc.pospopcnt(host, 16, threads=16)


def test_cfg3_bytes_offset3_full(pp, dev, orc):
    buf = torch.full(((1 << 30) + 64,), 0xFF, dtype=torch.uint8, device="cuda")
    n = (1 << 30) - 7
    pp.generate(pp.GEN_CFG3, 1, buf[3:3 + n])
    got = pp.pospopcnt_k(buf[3:3 + n], 8)
    host = buf.cpu().numpy()
    assert host[0] == 0xFF and host[3 + n] == 0xFF  # guards intact
    assert got == orc.pospopcnt(host[3:3 + n], 8, threads=16)


def test_cfg4_bernoulli_full_and_sharded(pp, dev, orc):
    n = 1 << 32
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, d)
    whole = pp.pospopcnt(d)
    for g in (2, 4, 8):  # shard boundaries as the G-GPU layout, all on device 0
        shards = [d[i * n // g:(i + 1) * n // g] for i in range(g)]
        assert pp.pospopcnt_sharded(shards, [0] * g) == whole
    # shard-local generation (index_base) gives the same bytes as the whole stream
    part = torch.empty(n // 8, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG4, 1, part, base=3 * (n // 8))
    assert torch.equal(part, d[3 * (n // 8):4 * (n // 8)])
    host = d.cpu().numpy().view(np.uint16)
    del d
    assert whole == orc.pospopcnt(host, 16, threads=16)
    assert abs(whole.total() / (16 * n) - 6554 / 65536) < 1e-4


@pytest.mark.parametrize("k,kind", [(32, 5), (64, 6)])
def test_cfg5_segmented_full(pp, dev, orc, k, kind):
    arrays, words = 65536, 4096
    d = torch.empty(arrays * words * k // 8, dtype=torch.uint8, device="cuda")
    pp.generate(kind, 1, d)
    offs = torch.arange(0, arrays + 1, dtype=torch.int64, device="cuda") * words
    out = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
    pp.segmented_async(d, offs, out, k)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint64)
    host = d.cpu().numpy().view(DT[k])
    want = orc.segmented(host, offs.cpu().numpy().view(np.uint64), k, threads=16)
    assert (got == want).all()
    assert (got.sum(1) == np.bitwise_count(host.reshape(arrays, words)).sum(1)).all()


# -- the reference's own harness driving the GPU path (C++ drop-in) ----------------------------

def test_reference_verify_kernels_with_gpu_runner():
    """oracle/_ref/verify_gpu: pospop::verify_kernels (proj/core/src/verify.cpp:33-75) with
    pospop_gpu::GpuRunner, the C++ drop-in against the reference's own types and errors."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "verify_gpu")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/verify_gpu not built (needs /root/reference at build time)")
    r = subprocess.run([exe, "3000"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 8 and "FAIL" not in r.stdout


_GROUPED = ["6,16,5,8", "6,16,5,4", "5,16,5,8", "6,32,5,8", "5,32,5,8", "5,16,5,4", "6,16,5,16", "5,32,5,4",
            "5,16,6", "5,32,6", "4,16,6", "4,32,6", "4,16,7", "4,32,7",  # + bit-plane epilogue (sched 6/7)
            "5,16,8", "5,16,9", "5,16,10,3", "5,16,10,2", "4,16,10,4"]  # sched 8/9/10
_TILE = ["7,32,11,1", "7,16,11,1", "6,32,11,1", "6,32,11,2", "6,16,11,2", "5,32,11,2", "7,32,12,1", "6,32,12,1",
         "6,32,12,2", "7,32,13,1", "6,32,13,2", "7,32,14,1", "6,32,14,1", "6,32,14,2", "5,16,16,2", "7,32,16,1", "5,32,16,2",
         "6,32,16,1"]
SEG_VARIANTS = {
    8: ["5,16,0", "5,16,1", "4,16,2", "5,16,2", "4,32,2", "5,32,2", "5,16,3", "5,32,3"] + _GROUPED + _TILE,
    16: ["5,16,0", "5,16,1", "4,16,2", "5,16,2", "4,32,2", "5,32,2", "5,16,3", "5,32,3"] + _GROUPED + _TILE,
    32: ["5,16,0", "5,16,1", "4,16,2", "5,16,2", "4,32,2", "5,32,2", "5,16,3", "5,32,3"] + _GROUPED + _TILE,
    64: ["5,16,0", "5,16,1", "4,16,2", "3,32,2", "4,32,2", "4,16,3", "3,32,3", "3,16,3",
         "4,16,5,8", "4,32,5,8", "4,16,5,4", "4,16,6", "4,32,6", "3,32,6", "3,16,7", "4,16,8", "3,16,10,4", "4,16,10,2",
         "6,32,11,1", "5,32,11,1", "5,32,11,2", "5,16,11,2", "6,32,12,1", "5,32,12,2", "6,32,13,1", "6,32,14,1", "5,16,16,2", "6,32,16,1"],
}


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_segmented_every_variant(pp, tuning, dev, orc, k, monkeypatch):
    """All segmented schedules (strided, dynamic, software-pipelined) on a ragged
    batch with empty arrays, tiny arrays and misaligned starts."""
    rng = np.random.default_rng(500 + k)
    n_words = 300_000
    data = orc.generate(6, 31, n_words * k // 64 + 1).view(DT[k])[:n_words]
    cuts = np.sort(np.concatenate([rng.integers(0, n_words, size=2000), np.arange(1000, 1100)]))
    offs = np.concatenate([[0, 0], cuts, [n_words, n_words]]).astype(np.uint64)
    want = orc.segmented(data, offs, k, threads=8)
    d = to_dev(data)
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    for var in SEG_VARIANTS[k]:
        monkeypatch.setenv("POSPOP_SEG_VARIANT", var)
        for per_sm in ("", "1"):
            if per_sm:
                monkeypatch.setenv("POSPOP_SEG_BLOCKS_PER_SM", per_sm)
            else:
                monkeypatch.delenv("POSPOP_SEG_BLOCKS_PER_SM", raising=False)
            out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
            pp.segmented_async(d, o, out, k)
            torch.cuda.synchronize()
            assert (out.cpu().numpy().view(np.uint64) == want).all(), (var, per_sm)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_segmented_grouped_big_arrays_and_flushes(pp, tuning, dev, orc, k, monkeypatch):
    """Grouped kernel (G lanes per array): batches holding an array above the
    big-array bound are counted one array at a time by the whole warp; forced
    flushes reduce inside each lane group; a few long arrays among many
    short ones; misaligned starts."""
    rng = np.random.default_rng(900 + k)
    n_words = 2_000_000
    data = orc.generate(6, 77, n_words * k // 64 + 1).view(DT[k])[:n_words]
    lens = rng.integers(0, 3000, size=600)
    lens[[5, 77, 300]] = [400_000, 250_001, 123_457]
    cuts = np.minimum(np.cumsum(lens), n_words)
    offs = np.concatenate([[0], cuts, [n_words]]).astype(np.uint64)
    want = orc.segmented(data, offs, k, threads=8)
    d = to_dev(data)
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    for var, big_kib, flush in [(v, b, f) for v in (("4,16,5,8", "4,16,6") if k == 64 else ("6,16,5,8", "5,16,6"))
                                for b, f in (("256", 65535), ("1", 65535), ("256", 1), ("1", 3))]:
        monkeypatch.setenv("POSPOP_SEG_VARIANT", var)
        monkeypatch.setenv("POSPOP_SEG_BIG_KIB", big_kib)
        out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
        pp.segmented_async(d, o, out, k, flush_threshold_blocks=flush)
        torch.cuda.synchronize()
        assert (out.cpu().numpy().view(np.uint64) == want).all(), (var, big_kib, flush)


def test_graph_replay_counts_current_contents(pp, dev, orc):
    """CUDA-graph replay (latency path): bit-exact, and it recounts the buffer's
    current contents at every replay."""
    for k, n_bytes in ((16, 8192), (8, 12345), (64, 1 << 20), (32, 5 << 20)):  # small, cluster, stream kernels
        a = orc.generate(6, 40 + k, (n_bytes + 7) // 8).view(np.uint8)[:n_bytes]
        b = orc.generate(6, 80 + k, (n_bytes + 7) // 8).view(np.uint8)[:n_bytes]
        buf = to_dev(a)
        out = torch.zeros(k, dtype=torch.int64, device="cuda")
        g = pp.CountGraph(buf, out, k)
        for _ in range(3):
            g.replay()
            torch.cuda.synchronize()
            assert (out.cpu().numpy().astype(np.uint64) == orc.naive(a, k)).all()
        buf.copy_(torch.from_numpy(b.copy()).cuda())
        g.replay()
        torch.cuda.synchronize()
        assert (out.cpu().numpy().astype(np.uint64) == orc.naive(b, k)).all()
        g.close()


def test_chained_async_launches_read_the_previous_output(pp, dev, orc):
    """A count whose input is the output of the previous launch on the same
    stream (our kernels let dependents start early) must see the finished
    output: the launcher drops programmatic dependent launch for it."""
    s = torch.cuda.current_stream()
    words = orc.generate(4, 11, 1 << 24)
    d = torch.from_numpy(words.view(np.int16).copy()).cuda()
    want = np.asarray(orc.pospopcnt(words, 16), np.uint64)
    for trial in range(20):
        out = torch.zeros(16, dtype=torch.int64, device="cuda")
        out2 = torch.zeros(64, dtype=torch.int64, device="cuda")
        pp.count_async(d, out, 16, stream=s)        # 16 counts ...
        pp.count_async(out, out2, 64, stream=s)     # ... counted as 16 u64 words
        torch.cuda.synchronize()
        assert (out.cpu().numpy().astype(np.uint64) == want).all()
        assert (out2.cpu().numpy().astype(np.uint64) == np.asarray(orc.pospopcnt(want, 64), np.uint64)).all(), trial
        seg = torch.empty((2, 16), dtype=torch.int64, device="cuda")
        offs = torch.tensor([0, 1 << 23, 1 << 24], dtype=torch.int64, device="cuda")
        pp.segmented_async(d, offs, seg, 16, stream=s)
        pp.count_async(seg, out2, 64, stream=s)     # rows of the segmented launch as input
        torch.cuda.synchronize()
        rows = seg.cpu().numpy().astype(np.uint64)
        assert (rows.sum(axis=0) == want).all()
        assert (out2.cpu().numpy().astype(np.uint64) == np.asarray(orc.pospopcnt(rows.ravel(), 64), np.uint64)).all()


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_segmented_few_huge_arrays(pp, dev, orc, k, monkeypatch):
    """Few arrays, some far larger than a warp's share (the adaptive kernel's
    range mode: even byte ranges per warp, arrays spanning ranges summed
    through workspace slots): one array over everything, a few hundred-MiB
    arrays with empty and tiny ones between them, offsets[0] > 0 at an odd
    word, repeated launches (the slots are left zero)."""
    wb = k // 8
    n_words = (300 << 20) // wb + 3
    data = orc.generate(6, 90 + k, n_words * wb // 8 + 1, threads=8).view(DT[k])[:n_words]
    d = to_dev(data)
    cases = [np.array([0, n_words], np.uint64),
             np.array([5, 5, 6, 6 + (100 << 20) // wb, 6 + (100 << 20) // wb, 7 + (100 << 20) // wb,
                       n_words - 9, n_words - 1, n_words - 1], np.uint64),
             np.array([1, 2, 3, 4], np.uint64),  # tiny arrays only
             np.array([17, 17], np.uint64)]       # one empty array
    for offs in cases:
        want = orc.segmented(data, offs, k, threads=8)
        o = torch.from_numpy(offs.view(np.int64)).cuda()
        for _ in range(3):
            out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
            pp.segmented_async(d, o, out, k)
            torch.cuda.synchronize()
            assert (out.cpu().numpy().view(np.uint64) == want).all(), offs[:4]
        assert (pp.pospopcnt_segmented(d, offs, k) == want).all()  # synchronous entry, host offsets


@pytest.mark.parametrize("k", [8, 32, 64])
@pytest.mark.parametrize("mode", ["lane", "grouped", "tile"])
def test_segmented_giant_queue(pp, tuning, dev, orc, k, mode, monkeypatch):
    """Giant arrays among many short ones: the lane / grouped / tile schedules
    publish arrays above the giant bound to the queue and every warp counts
    their chunks at its exit.  A 16 KiB bound makes hundreds of giants (more
    than the 512 queue entries: the overflow is counted by the publisher), with
    empty arrays, odd starts and a few huge arrays; repeated launches (the
    queue is reset by the last CTA)."""
    monkeypatch.setenv("POSPOP_SEG_VARIANT", "4,16,8" if k == 64 else "5,16,8")
    lane, group, tile = {"lane": (4096, 4096, 4096), "grouped": (0, 4096, 4096), "tile": (0, 0, 0)}[mode]
    monkeypatch.setenv("POSPOP_SEG_LANE_MEAN_BYTES", str(lane))
    monkeypatch.setenv("POSPOP_SEG_GROUP_MEAN_BYTES", str(group))
    monkeypatch.setenv("POSPOP_SEG_TILE_MEAN_BYTES", str(tile))
    monkeypatch.setenv("POSPOP_SEG_RANGE", "0")
    monkeypatch.setenv("POSPOP_SEG_GIANT_KIB", "16")
    wb = k // 8
    rng = np.random.default_rng(700 + k)
    lens = rng.integers(0, 24 if mode != "tile" else 600, size=40000)
    lens[rng.random(lens.size) < 0.1] = 0
    big = rng.choice(lens.size, size=800, replace=False)
    lens[big] = rng.integers((16 << 10) // wb + 1, (64 << 10) // wb, size=big.size)  # > 16 KiB
    lens[[17, 20000, 39999]] = [(40 << 20) // wb + 3, (5 << 20) // wb, (9 << 20) // wb + 1]
    offs = np.concatenate([[3], 3 + np.cumsum(lens)]).astype(np.uint64)
    n_words = int(offs[-1]) + 8
    data = orc.generate(6, 71, n_words * wb // 8 + 1, threads=8).view(DT[k])[:n_words]
    want = orc.segmented(data, offs, k, threads=8)
    d = to_dev(data)
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    for _ in range(3):
        out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
        pp.segmented_async(d, o, out, k)
        torch.cuda.synchronize()
        assert (out.cpu().numpy().view(np.uint64) == want).all(), mode


@pytest.mark.parametrize("var", ["", "7,32,13,1", "7,32,14,1", "6,32,14,2"])
def test_chained_segmented_launches(pp, tuning, dev, orc, var, monkeypatch):
    """Segmented kernels that read (and count) before waiting for the previous
    launch on the stream: a segmented input produced by the previous launch
    (RAW: programmatic dependent launch dropped), rows overwritten by the next
    launch (WAW) and rows written over the previous launch's input (WAR) --
    rows reach global memory only after the previous launch completed."""
    if var:
        monkeypatch.setenv("POSPOP_SEG_VARIANT", var)
    s = torch.cuda.current_stream()
    k, arrays, words = 32, 8192, 4096
    a = orc.generate(5, 61, arrays * words)  # u32 words
    b = orc.generate(5, 62, arrays * words)
    da, db = (torch.from_numpy(x.view(np.int64).copy()).cuda() for x in (a, b))
    offs = torch.arange(arrays + 1, dtype=torch.int64, device="cuda") * words
    want_b = orc.segmented(b, offs.cpu().numpy().view(np.uint64), k, threads=8)
    rows = torch.empty((arrays, k), dtype=torch.int64, device="cuda")
    small_offs = torch.tensor([0, 3, 16], dtype=torch.int64, device="cuda")
    cnt = torch.zeros(16, dtype=torch.int64, device="cuda")
    # RAW on the offsets: a count's output (non-decreasing by construction:
    # word i of a 16-word block sets bits i..15, so counts[p] = (p + 1) * blocks)
    # is the next segmented launch's offsets array
    blk = np.array([sum(1 << p for p in range(16) if p >= i) for i in range(16)], np.uint16)
    blocks = 1 << 16
    d_blk = torch.from_numpy(np.tile(blk, blocks).view(np.int16)).cuda()
    seg_words = torch.from_numpy(a[:blocks * 16].view(np.int64).copy()).cuda()
    off_dev = torch.zeros(16, dtype=torch.int64, device="cuda")
    want_offs = np.arange(1, 17, dtype=np.uint64) * blocks
    want_rows = orc.segmented(a[:blocks * 16].view(np.uint32), want_offs, 32, threads=8)
    for trial in range(5):
        off_dev.zero_()
        pp.count_async(d_blk, off_dev, 16, stream=s)
        rows_o = torch.empty((15, 32), dtype=torch.int64, device="cuda")
        pp.segmented_async(seg_words, off_dev, rows_o, 32, stream=s)
        torch.cuda.synchronize()
        assert (off_dev.cpu().numpy().view(np.uint64) == want_offs).all()
        assert (rows_o.cpu().numpy().view(np.uint64) == want_rows).all(), trial
    for trial in range(10):
        # WAW: the second launch's rows win
        pp.segmented_async(da, offs, rows, k, stream=s)
        pp.segmented_async(db, offs, rows, k, stream=s)
        # RAW: the previous launch's rows as the next segmented input (k = 64 words)
        rows2 = torch.empty((2, 64), dtype=torch.int64, device="cuda")
        pp.segmented_async(rows, small_offs, rows2, 64, stream=s)
        torch.cuda.synchronize()
        got = rows.cpu().numpy().view(np.uint64)
        assert (got == want_b).all(), trial
        w64 = got.ravel()[:16]
        want2 = orc.segmented(w64, np.array([0, 3, 16], np.uint64), 64)
        assert (rows2.cpu().numpy().view(np.uint64) == want2).all(), trial
        # WAR: a count reading `victim`, then rows written over it
        victim = torch.from_numpy(a.view(np.int64).copy()).cuda()
        pp.count_async(victim, cnt, 16, stream=s)
        pp.segmented_async(db, offs, victim[:arrays * k].view(arrays, k), k, stream=s)
        torch.cuda.synchronize()
        assert (cnt.cpu().numpy().view(np.uint64) == np.asarray(orc.pospopcnt(a.view(np.uint16), 16, threads=8),
                                                                np.uint64)).all(), trial
        assert (victim[:arrays * k].view(arrays, k).cpu().numpy().view(np.uint64) == want_b).all()


def test_k_widths_against_reference_fixtures(pp, dev, orc, golden):
    """The GPU on the k = 8/32/64 fixtures counted by the reference library's
    16-bit API (golden k_widths), at the fixture's byte offset inside 0xFF guards."""
    for seed, k, off, n, *counts in golden["k_widths"]:
        wb = k // 8
        stream = orc.mt_generate_stream(seed, (off + n * wb) // 2 + 2).view(np.uint8)
        buf = torch.full((stream.size + 128,), 0xFF, dtype=torch.uint8, device="cuda")
        buf[64:64 + stream.size] = torch.from_numpy(stream.copy()).cuda()
        view = buf[64 + off: 64 + off + n * wb]
        assert [int(x) for x in pp.pospopcnt_k(view, k).counts] == counts, (seed, k, off, n)


def test_sharded_repeated_calls_and_empty_shards(pp, dev, orc):
    """pospopcnt_sharded reuses per-device shard slots across calls: repeated
    calls, a varying shard count, empty shards, every k."""
    for k in (8, 16, 32, 64):
        raw = orc.generate(6, 60 + k, (3 << 20) // 8).view(np.uint8)
        d = torch.from_numpy(raw.copy()).cuda()
        want = orc.pospopcnt(raw, k, threads=4)
        wb = k // 8
        n = raw.size // wb
        for parts in (1, 3, 5, 2, 5):
            cuts = [n * i // parts for i in range(parts + 1)]
            shards = [d[cuts[i] * wb: cuts[i + 1] * wb] for i in range(parts)]
            shards.insert(1, d[:0])  # an empty shard
            assert pp.pospopcnt_sharded(shards, [0] * len(shards), k) == want, (k, parts)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
@pytest.mark.parametrize("mode", ["lane", "grouped", "tile", "range"])
def test_segmented_adaptive_modes(pp, tuning, dev, orc, k, mode, monkeypatch):
    """The adaptive kernel (sched 8) in each of its modes -- forced through the
    mean-length thresholds -- on tiny, ragged, empty and large arrays; in lane
    mode a batch with an array above the lane cap takes the full-warp path."""
    monkeypatch.setenv("POSPOP_SEG_VARIANT", "4,16,8" if k == 64 else "5,16,8")
    lane, group, tile, rounds = {"lane": (1 << 20, 1 << 20, 1 << 20, 0), "grouped": (0, 1 << 20, 1 << 20, 0),
                                 "tile": (0, 0, 0, 0), "range": (0, 0, 0, 255)}[mode]
    monkeypatch.setenv("POSPOP_SEG_LANE_MEAN_BYTES", str(lane))
    monkeypatch.setenv("POSPOP_SEG_GROUP_MEAN_BYTES", str(group))
    monkeypatch.setenv("POSPOP_SEG_TILE_MEAN_BYTES", str(tile))
    monkeypatch.setenv("POSPOP_SEG_RANGE", str(rounds))
    rng = np.random.default_rng(40 + k)
    n_words = 1_500_000
    data = orc.generate(6, 51, n_words * k // 64 + 1).view(DT[k])[:n_words]
    lens = rng.integers(0, 64, size=6000)
    lens[rng.random(lens.size) < 0.2] = 0
    lens[[10, 2000, 5999]] = [40_000, 100_001, 7]  # large arrays among tiny ones
    offs = np.minimum(np.concatenate([[0], np.cumsum(lens)]), n_words).astype(np.uint64)
    want = orc.segmented(data, offs, k, threads=8)
    d = to_dev(data)
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    for _ in range(2):  # claim counter and ticket are reset for the next launch
        out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
        pp.segmented_async(d, o, out, k)
        torch.cuda.synchronize()
        assert (out.cpu().numpy().view(np.uint64) == want).all(), mode


@pytest.mark.parametrize("k", [8, 16, 32, 64])
@pytest.mark.parametrize("mode", ["default", "lane"])
def test_segmented_rows_at_8_byte_aligned_output(pp, dev, orc, k, mode, monkeypatch, request):
    """Row stores at an output that is only 8-byte aligned: the default path
    (few arrays: the range kernel) and the adaptive kernel's lane mode (staged
    rows copied out with 8-byte stores)."""
    if mode == "lane":  # forced through the tuning build's knobs
        request.getfixturevalue("tuning")
        monkeypatch.setenv("POSPOP_SEG_VARIANT", "4,16,8" if k == 64 else "5,16,8")
        monkeypatch.setenv("POSPOP_SEG_RANGE", "0")
    rng = np.random.default_rng(70 + k)
    lens = rng.integers(0, 40, size=3001)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    total = int(offs[-1])
    data = orc.generate(6, 71, total * k // 64 + 1).view(DT[k])[:total]
    want = orc.segmented(data, offs, k, threads=4)
    d = to_dev(data)
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    n = offs.size - 1
    buf = torch.full((n * k + 2,), -1, dtype=torch.int64, device="cuda")
    out = buf[1:1 + n * k]  # 8-byte aligned, not 16
    pp.segmented_async(d, o, out, k)
    torch.cuda.synchronize()
    assert (out.view(n, k).cpu().numpy().view(np.uint64) == want).all()
    assert int(buf[0]) == -1 and int(buf[-1]) == -1


def test_typed_entry_points(pp, dev, orc):
    """The typed C entry points of SURVEY.md 8b (pospopcnt_u{8,16,32,64}_segmented,
    pospopcnt_u16_sharded, pospopcnt_u16_async) equal the generic ones."""
    import ctypes as C
    lib = pp._load()
    u64p = C.POINTER(C.c_uint64)
    raw = orc.generate(6, 33, 1 << 16).view(np.uint8)
    for k in (8, 16, 32, 64):
        wb = k // 8
        n_words = raw.size // wb
        offs = np.array([0, 1, 1, 777, n_words // 2, n_words], np.uint64)
        rows = np.zeros((offs.size - 1, k), np.uint64)
        fn = getattr(lib, f"pospopcnt_u{k}_segmented")
        fn.argtypes = [C.c_void_p, u64p, C.c_size_t, u64p]
        assert fn(raw.ctypes.data, offs.ctypes.data_as(u64p), offs.size - 1, rows.ctypes.data_as(u64p)) == 0
        assert (rows == orc.segmented(raw.view(DT[k]), offs, k)).all(), k
    d = to_dev(raw)
    lib.pospopcnt_u16_sharded.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_int), C.c_int,
                                          u64p]
    half = raw.size // 4  # words per shard (two shards)
    ptrs = (C.c_void_p * 2)(d.data_ptr(), d.data_ptr() + 2 * half)
    lens = (C.c_size_t * 2)(half, raw.size // 2 - half)
    devs = (C.c_int * 2)(0, 0)
    out = np.zeros(16, np.uint64)
    assert lib.pospopcnt_u16_sharded(ptrs, lens, devs, 2, out.ctypes.data_as(u64p)) == 0
    want = orc.naive(raw, 16)
    assert [int(x) for x in out] == [int(x) for x in want]
    lib.pospopcnt_u16_async.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    d_out = torch.full((16,), -1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    assert lib.pospopcnt_u16_async(d.data_ptr(), raw.size // 2, d_out.data_ptr(), C.c_void_p(s.cuda_stream)) == 0
    torch.cuda.synchronize()
    assert [int(x) for x in d_out.cpu().numpy()] == [int(x) for x in want]


@pytest.mark.parametrize("k", [16, 32, 64])
@pytest.mark.parametrize("mode", ["range_kernel", "adaptive_range"])
def test_segmented_range_mode_misaligned_data(pp, dev, orc, k, mode, monkeypatch, request):
    """Range mode with data that is word-aligned but not 16-byte aligned
    (+wb, +2wb, +3wb bytes) and offsets[0] = 0, so the first referenced byte
    sits in the first 16-byte block: every range must be counted and no
    workspace slot may be left dirty.  Misaligned and aligned calls alternate
    on one stream (a dirty slot would corrupt the next call's rows); the host
    path (pageable data staged at the caller's 32-byte phase) is checked too."""
    if mode == "adaptive_range":  # the tuning build (the release library routes this case to the range kernel)
        request.getfixturevalue("tuning")
        monkeypatch.setenv("POSPOP_SEG_VARIANT", "4,16,8" if k == 64 else "5,16,8")
        monkeypatch.setenv("POSPOP_SEG_RANGE", "63")
    wb = k // 8
    n_words = (3 << 20) // wb
    raw = orc.generate(6, 300 + k, n_words * wb // 8 + 8, threads=8).view(np.uint8)
    rng = np.random.default_rng(k)
    # few arrays (<= SM count: the host routes to the range kernel), some spanning many ranges
    cuts = np.sort(rng.choice(np.arange(1, n_words - 1), size=40, replace=False))
    offs = np.concatenate([[0, 0, 5], cuts, [n_words - 1, n_words]]).astype(np.uint64)
    if mode == "adaptive_range":  # more arrays than SMs: the adaptive kernel, range mode forced
        offs = np.unique(np.concatenate([offs, rng.integers(0, n_words, size=400).astype(np.uint64)]))
        offs = np.concatenate([[0], offs]).astype(np.uint64)
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    buf = torch.from_numpy(raw.copy()).cuda()  # 256-byte aligned base
    s = torch.cuda.Stream()
    for rep in range(2):
        for shift in (wb, 2 * wb, 3 * wb, 0):
            words = raw[shift:shift + n_words * wb].view(DT[k])
            want = orc.segmented(words, offs, k, threads=8)
            d = buf[shift:shift + n_words * wb]
            out = torch.full((offs.size - 1, k), -1, dtype=torch.int64, device="cuda")
            pp.segmented_async(d, o, out, k, stream=s)
            s.synchronize()
            assert (out.cpu().numpy().view(np.uint64) == want).all(), (k, shift, rep)
            if rep == 0:  # synchronous entry point: device data, host offsets; then pageable host data
                assert (pp.pospopcnt_segmented(d, offs, k) == want).all(), (k, shift)
                assert (pp.pospopcnt_segmented(words, offs, k) == want).all(), (k, shift, "host")


def test_counts_beyond_2_pow_32_words(pp, dev, orc):
    """size_t lengths past 2^32 words (16 GiB of u16, 2^31 + u64 words): the
    reference's uint32_t-length Fig. 6 API could not express these
    (PAPER.md:316); the stream kernel, the sharded path and the segmented
    range kernel (one array spanning every range) all agree with the oracle."""
    n = (1 << 33) + 3
    d = torch.empty(n, dtype=torch.int16, device="cuda")
    pp.generate(pp.GEN_CFG4, 5, d)
    host = d.cpu().numpy().view(np.uint16)
    want16 = orc.pospopcnt(host, 16, threads=16)
    assert pp.pospopcnt(d) == want16
    assert pp.pospopcnt_sharded([d[: n // 3], d[n // 3:]], [0, 0]) == want16
    want64 = orc.pospopcnt(host.view(np.uint8)[: (n * 2) // 8 * 8], 64, threads=16)
    assert pp.pospopcnt_k((d.data_ptr(), (n * 2) // 8), 64) == want64
    offs = torch.tensor([0, 1, n - 1, n], dtype=torch.int64, device="cuda")  # one array over 2^33 words
    rows = pp.pospopcnt_segmented(d, offs, 16)
    want_rows = orc.segmented(host, np.array([0, 1, n - 1, n], np.uint64), 16, threads=16)
    assert (np.asarray(rows, np.uint64) == want_rows).all()
