"""Property-based fuzzing of the product paths against the oracle (hypothesis):
random k, lengths, byte offsets inside 0xFF guards, flush thresholds, value
distributions (generator kinds), accumulate, segmented offsets with empty,
tiny and giant arrays in every adaptive-kernel mode (lane / grouped / tile /
range, giant queue on and off), and every host/device placement.  Bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=60, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])


@pytest.fixture(scope="module")
def dev(pp):
    assert torch.cuda.is_available() and pp.device_available()
    torch.cuda.set_device(0)


def guarded(raw, offset, guard=64):
    buf = torch.full((guard + offset + raw.size + guard,), 0xFF, dtype=torch.uint8, device="cuda")
    buf[guard + offset:guard + offset + raw.size] = torch.from_numpy(raw.copy()).cuda()
    return buf[guard + offset:guard + offset + raw.size]


@SETTINGS
@given(k=st.sampled_from([8, 16, 32, 64]), n=st.integers(0, 600_000), off_words=st.integers(0, 7),
       kind=st.sampled_from([1, 2, 4, 6]), seed=st.integers(0, 2**32 - 1),
       flush=st.sampled_from([1, 2, 3, 255, 65535]), where=st.sampled_from(["device", "pinned", "pageable"]))
def test_fuzz_counts(pp, dev, orc, k, n, off_words, kind, seed, flush, where):
    wb = k // 8
    esize = np.dtype(orc.GEN_DTYPE[kind]).itemsize
    raw = orc.generate(kind, seed, (n * wb + esize - 1) // esize + 1).view(np.uint8)[: n * wb]
    want = orc.pospopcnt(raw, k, threads=4)
    if where == "device":
        data = guarded(raw, off_words * wb)
    elif where == "pinned":
        t = torch.empty(raw.size + 64, dtype=torch.uint8, pin_memory=True)
        t.numpy()[off_words * wb: off_words * wb + raw.size] = raw
        data = t[off_words * wb: off_words * wb + raw.size].numpy()
    else:
        host = np.empty(raw.size + 64, np.uint8)
        host[off_words * wb: off_words * wb + raw.size] = raw
        data = host[off_words * wb: off_words * wb + raw.size]
    assert pp.pospopcnt_k(data, k, flush_threshold_blocks=flush) == want


# Adaptive-kernel mode forced through its bounds (lane, grouped, tile, range mean bytes / rounds).
MODES = {"auto": {}, "lane": {"LANE_MEAN_BYTES": 4000, "GROUP_MEAN_BYTES": 4000, "RANGE": 0},
         "grouped": {"LANE_MEAN_BYTES": 0, "GROUP_MEAN_BYTES": 4000, "RANGE": 0},
         "tile": {"LANE_MEAN_BYTES": 0, "GROUP_MEAN_BYTES": 0, "TILE_MEAN_BYTES": 0, "RANGE": 0},
         "range": {"RANGE": 63}}


@settings(SETTINGS, max_examples=300)
@given(k=st.sampled_from([8, 16, 32, 64]), n_arrays=st.integers(1, 12000),
       max_len=st.sampled_from([1, 17, 300, 5000, 40000]),
       seed=st.integers(0, 2**32 - 1), empty_frac=st.floats(0, 0.5), flush=st.sampled_from([1, 3, 65535]),
       mode=st.sampled_from(sorted(MODES)), giant_kib=st.sampled_from([1024, 16]), start=st.integers(0, 9),
       huge=st.booleans())
def test_fuzz_segmented(pp, tuning, dev, orc, k, n_arrays, max_len, seed, empty_frac, flush, mode, giant_kib, start, huge):
    import os
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, size=n_arrays)
    lens[rng.random(n_arrays) < empty_frac] = 0
    if huge:  # a few arrays far above the giant bound
        lens[rng.integers(0, n_arrays, size=3)] = rng.integers(1 << 16, 1 << 19, size=3) * 8 // k
    offs = np.concatenate([[start], start + np.cumsum(lens)]).astype(np.uint64)
    env = {f"POSPOP_SEG_{key}": str(v) for key, v in MODES[mode].items()}
    env["POSPOP_SEG_GIANT_KIB"] = str(giant_kib)
    saved = {key: os.environ.get(key) for key in env}
    os.environ.update(env)
    try:
        _check_segmented(pp, orc, k, offs, n_arrays, seed, flush)
    finally:
        for key, v in saved.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


def _check_segmented(pp, orc, k, offs, n_arrays, seed, flush):
    total = int(offs[-1])
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[k]
    data = orc.generate(6, seed, total * k // 64 + 1).view(dt)[:total]
    want = orc.segmented(data, offs, k, threads=4)
    d = torch.from_numpy(data.view(np.uint8).copy()).cuda() if total else torch.zeros(8, dtype=torch.uint8,
                                                                                        device="cuda")
    o = torch.from_numpy(offs.view(np.int64)).cuda()
    out = torch.full((n_arrays, k), -1, dtype=torch.int64, device="cuda")
    pp.segmented_async(d, o, out, k, flush_threshold_blocks=flush)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint64) == want).all()
    assert (np.asarray(pp.pospopcnt_segmented(data, offs, k), np.uint64) == want).all()  # host path
