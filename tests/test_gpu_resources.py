"""Multi-link host ingestion (pospopcnt_sharded with host shards,
pospopcnt_split) and the resource lifecycle (per-device context pool,
per-stream workspaces, pospop_release_resources).  The reference's
scale-out contract is fork-join + merge over host memory
(proj/tests/test_core.cpp:155-175); all of its per-call state lives on the
stack (proj/core/src/detail/csa_engine.hpp:107-110), which the pool
bounds per device here.  Counts are bit-exact against the oracle."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(pp):
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a GPU")
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


def pinned_copy(a: np.ndarray) -> tuple[torch.Tensor, np.ndarray]:
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    v = t.numpy()
    v[:] = a.view(np.uint8)
    return t, v.view(a.dtype)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_split_host_memory_over_devices(pp, dev, orc, k):
    """One host buffer split over devices [0, 0] (two host links' worth of
    staging on one GPU), pageable and pinned; lengths not a multiple of the
    split and an odd byte start for k = 8."""
    rng = np.random.default_rng(k)
    raw = rng.integers(0, 256, size=(96 << 20) + 77, dtype=np.uint8)
    off = 3 if k == 8 else 0
    nbytes = (raw.size - off) // (k // 8) * (k // 8)
    view = raw[off:off + nbytes]
    want = orc.pospopcnt(view, k, threads=16)
    words = view.view({8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[k]) if off == 0 else view
    assert pp.pospopcnt_split(words, [0, 0], k) == want
    assert pp.pospopcnt_split(words, [0, 0, 0], k) == want
    keep, pv = pinned_copy(raw)
    pview = pv[off:off + nbytes]
    assert pp.pospopcnt_split(pview, [0, 0], k) == want
    assert pp.pospopcnt_split(pview, [0], k) == want


def test_sharded_mixes_host_and_device_shards(pp, dev, orc):
    n = (40 << 20) + 5
    host = orc.generate(4, 9, n)  # cfg4 Bernoulli(0.1) words
    want = orc.pospopcnt(host, 16, threads=16)
    d = torch.from_numpy(host.view(np.int16)).cuda()
    cut = [0, n // 5, n // 2, (3 * n) // 4, n]
    keep, pinned = pinned_copy(host)
    shards = [d[cut[0]:cut[1]], host[cut[1]:cut[2]], pinned[cut[2]:cut[3]], d[cut[3]:cut[4]]]
    assert pp.pospopcnt_sharded(shards, [0, 0, 0, 0]) == want
    # empty host shards and a single-word shard
    shards = [host[:0], host[:1], host[1:], d[:0]]
    assert pp.pospopcnt_sharded(shards, [0, 0, 0, 0]) == want


def test_sharded_rejects_a_missing_device(pp, dev):
    with pytest.raises(pp.InvalidArgument, match="no device"):
        pp.pospopcnt_sharded([np.ones(16, np.uint16)], [torch.cuda.device_count()])
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_split(np.ones(16, np.uint16), [], 16)


def _free_bytes():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info(0)[0]


def test_many_threads_and_streams_return_memory_after_release(pp, dev, orc):
    """64 threads and 64 streams: contexts stay bounded per device (at most 8),
    and device memory returns to its baseline after pospop_release_resources."""
    rng = np.random.default_rng(5)
    host_small = rng.integers(0, 1 << 16, size=1 << 18, dtype=np.uint16)        # bounce path
    host_big = rng.integers(0, 1 << 16, size=(3 << 20) + 11, dtype=np.uint16)   # staging ring
    d_words = torch.from_numpy(rng.integers(0, 1 << 16, size=1 << 22, dtype=np.uint16).view(np.int16)).cuda()
    offs = np.arange(0, 4097 * 64, 4096, dtype=np.uint64)
    seg_words = torch.from_numpy(rng.integers(0, 1 << 32, size=4096 * 64, dtype=np.uint32).view(np.int32)).cuda()
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    want_small = orc.pospopcnt(host_small, 16)
    want_big = orc.pospopcnt(host_big, 16, threads=8)
    want_dev = orc.pospopcnt(d_words.cpu().numpy().view(np.uint16), 16, threads=8)
    want_seg = orc.segmented(seg_words.cpu().numpy().view(np.uint32), offs, 32)
    outs = [torch.zeros(16, dtype=torch.int64, device="cuda") for _ in range(64)]
    seg_outs = [torch.zeros(64 * 32, dtype=torch.int64, device="cuda") for _ in range(64)]
    streams = [torch.cuda.Stream() for _ in range(64)]

    def one_round():
        errors = []

        def work(i):
            try:
                torch.cuda.set_device(0)
                assert pp.pospopcnt_k(host_small, 16) == want_small
                assert pp.pospopcnt_k(d_words, 16) == want_dev
                if i % 8 == 0:
                    assert pp.pospopcnt_k(host_big, 16) == want_big
                rows = pp.pospopcnt_segmented(seg_words, d_offs, 32)
                assert (np.asarray(rows, np.uint64) == want_seg).all()
            except Exception as e:  # noqa: BLE001
                errors.append(repr(e))

        threads = [threading.Thread(target=work, args=(i,)) for i in range(64)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors[:3]
        for i, s in enumerate(streams):  # async entry points: one workspace per stream
            pp.count_async(d_words, outs[i], 16, stream=s)
            pp.segmented_async(seg_words, d_offs, seg_outs[i], 32, stream=s)
        torch.cuda.synchronize()
        for i in range(64):
            assert outs[i].cpu().numpy().view(np.uint64).tolist() == [int(x) for x in want_dev]
            assert (seg_outs[i].cpu().numpy().view(np.uint64).reshape(64, 32) == want_seg).all()

    one_round()  # loads every kernel module the round uses
    pp.release_resources()
    base = _free_bytes()
    st = pp.resource_stats(0)
    assert st == {"contexts": 0, "idle_contexts": 0, "stream_workspaces": 0}, st
    one_round()
    st = pp.resource_stats(0)
    assert 1 <= st["contexts"] <= 8 and st["idle_contexts"] == st["contexts"], st
    assert st["stream_workspaces"] >= 32, st  # torch hands out a pool of 32 streams
    held = base - _free_bytes()
    pp.release_resources()
    after = _free_bytes()
    assert pp.resource_stats(0) == {"contexts": 0, "idle_contexts": 0, "stream_workspaces": 0}
    assert abs(base - after) <= (4 << 20), (base, after, held)
    # the library stays usable after a release
    assert pp.pospopcnt_k(host_small, 16) == want_small


def test_release_stream(pp, dev):
    s = torch.cuda.Stream()
    d = torch.ones(1 << 20, dtype=torch.int16, device="cuda")
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    before = pp.resource_stats(0)["stream_workspaces"]
    pp.count_async(d, out, 16, stream=s)
    assert pp.resource_stats(0)["stream_workspaces"] == before + 1
    pp.release_stream(s)
    assert pp.resource_stats(0)["stream_workspaces"] == before
    assert out.cpu()[0].item() == 1 << 20


def test_small_host_calls_read_in_place(pp, dev, orc):
    """Pinned host inputs up to 2 MiB and pageable ones up to 1 MiB are read
    in place by the kernel (zero-copy): bit-exact, and no device staging ring
    (3 x 64 MiB) is allocated for them; a larger input still uses it."""
    rng = np.random.default_rng(11)
    pageable = rng.integers(0, 1 << 16, size=(1 << 19) - 3, dtype=np.uint16)  # < 1 MiB
    keep, pinned = pinned_copy(rng.integers(0, 1 << 16, size=(1 << 20) - 5, dtype=np.uint16))  # < 2 MiB
    pp.release_resources()
    base = _free_bytes()
    for k in (8, 16, 32, 64):
        for words in (pageable, pinned):
            raw = words.view(np.uint8)
            n = raw.size // (k // 8) * (k // 8)
            assert pp.pospopcnt_k(raw[:n], k) == orc.pospopcnt(raw[:n], k, threads=4), k
    held = base - _free_bytes()
    assert held < (64 << 20), held  # contexts and workspaces only, no staging ring
    big = rng.integers(0, 1 << 16, size=(8 << 20) // 2, dtype=np.uint16)  # 8 MiB pageable: staged
    assert pp.pospopcnt_k(big, 16) == orc.pospopcnt(big, 16, threads=4)
    assert base - _free_bytes() >= (3 * 64 << 20), base - _free_bytes()
    pp.release_resources()


def test_more_host_shards_than_the_context_bound(pp, dev, orc):
    """12 host shards and a device shard on one device: the host-shard workers
    may exceed the per-device bound of 8 contexts for the call (waiting there
    could deadlock against other callers), and the surplus is freed when the
    call returns."""
    rng = np.random.default_rng(12)
    words = rng.integers(0, 1 << 16, size=(12 << 20) + 7, dtype=np.uint16)
    want = orc.pospopcnt(words, 16, threads=8)
    cuts = np.linspace(0, words.size, 14).astype(np.int64)
    shards = [words[cuts[i]:cuts[i + 1]] for i in range(12)]
    shards.append(torch.from_numpy(words[cuts[12]:].view(np.int16).copy()).cuda())
    assert pp.pospopcnt_sharded(shards, [0] * 13) == want
    st = pp.resource_stats(0)
    assert st["contexts"] <= 8 and st["idle_contexts"] == st["contexts"], st


def test_split_device_resident_data(pp, dev, orc):
    """pospopcnt_split on device memory: every range is a device shard on the
    device holding it, counted in place."""
    rng = np.random.default_rng(13)
    host = rng.integers(0, 1 << 16, size=(5 << 20) + 3, dtype=np.uint16)
    d = torch.from_numpy(host.view(np.int16)).cuda()
    want = orc.pospopcnt(host, 16, threads=8)
    for n in (1, 2, 3, 7):
        assert pp.pospopcnt_split(d, [0] * n, 16) == want, n
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_split(d, [torch.cuda.device_count()], 16)


@pytest.mark.parametrize("k", [8, 32, 64])
def test_segmented_split_over_devices(pp, dev, orc, k):
    """Segmented fork-join over devices [0, 0, 0] from host memory (the
    batched variant shards by arrays, no exchange): ragged arrays, empty
    ones, one long array, pageable and pinned data; rows equal the oracle."""
    rng = np.random.default_rng(20 + k)
    wb = k // 8
    lens = rng.integers(0, 5000, size=3000)
    lens[[7, 1500]] = [0, 3_000_000 // wb]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    raw = rng.integers(0, 256, size=int(offs[-1]) * wb + 16, dtype=np.uint8)
    words = raw[: int(offs[-1]) * wb]
    want = orc.segmented(words, offs, k, threads=8)
    for devs in ([0], [0, 0], [0, 0, 0], [0] * 5):
        got = pp.pospopcnt_segmented_split(words, offs, k, devs)
        assert (np.asarray(got, np.uint64) == want).all(), devs
    keep, pinned = pinned_copy(words)
    assert (np.asarray(pp.pospopcnt_segmented_split(pinned, offs, k, [0, 0]), np.uint64) == want).all()
    d = torch.from_numpy(words.copy()).cuda()  # device-resident: one device counts it all
    assert (np.asarray(pp.pospopcnt_segmented_split(d, offs, k, [0, 0]), np.uint64) == want).all()


def test_concurrent_splits_and_releases(pp, dev, orc):
    """Four threads running host-memory splits over [0, 0] while a fifth keeps
    calling pospop_release_resources (safe against synchronous calls): every
    result exact, nothing leaked afterwards."""
    rng = np.random.default_rng(14)
    inputs = [rng.integers(0, 1 << 16, size=(3 << 20) + i, dtype=np.uint16) for i in range(4)]
    wants = [orc.pospopcnt(x, 16, threads=4) for x in inputs]
    errors, stop = [], threading.Event()

    def worker(i):
        try:
            torch.cuda.set_device(0)
            for _ in range(6):
                assert pp.pospopcnt_split(inputs[i], [0, 0], 16) == wants[i]
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    def releaser():
        torch.cuda.set_device(0)
        while not stop.is_set():
            pp.release_resources()

    r = threading.Thread(target=releaser)
    r.start()
    threads = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    stop.set()
    r.join()
    assert not errors, errors[:3]
    pp.release_resources()
    assert pp.resource_stats(0)["contexts"] == 0
