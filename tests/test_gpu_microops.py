"""The DEVICE primitives of the counting kernels, pinned
against the reference's micro-op KATs (proj/tests/test_csa.cpp:32-216) restated
on 32-bit registers (two 16-bit lanes) and against the oracle's Backend64
restatement on random inputs.  Runs through pospop_microop in the C ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M32 = 0xFFFFFFFF
LOW_IMM, HIGH_IMM = 0b10010110, 0b11101000  # test_csa.cpp:29-30


@pytest.fixture(scope="module")
def dev(pp):
    assert pp.device_available()


def test_csa_truth_table_and_examples(pp, dev):
    triples = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    out = pp.microop(0, 1, [x for t in triples for x in t], 2 * len(triples))
    for i, (a, b, c) in enumerate(triples):
        h, l = int(out[2 * i]), int(out[2 * i + 1])
        m = a + 2 * b + 4 * c
        assert 2 * h + l == a + b + c and l == (LOW_IMM >> m) & 1 and h == (HIGH_IMM >> m) & 1
    out = pp.microop(0, 1, [0b1010, 0b0110, 0b1100], 2)  # test_csa.cpp:45-50
    assert list(out) == [0b1110, 0]


def test_csa_wide_identity_vs_oracle(pp, dev, orc):
    rng = np.random.default_rng(12345)
    t = rng.integers(0, 2**32, size=(2000, 3), dtype=np.uint64)
    out = pp.microop(0, 1, t.ravel(), 4000)
    for i, (a, b, c) in enumerate(t):
        h, l = orc.csa(int(a), int(b), int(c))
        assert int(out[2 * i]) == h & M32 and int(out[2 * i + 1]) == l & M32


def test_tree_kats(pp, dev):
    # four all-ones inputs, zero carries -> top all ones, carries zero (test_csa.cpp:71-78)
    out = pp.microop(1, 2, [0, 0] + [M32] * 4, 1 + 2)
    assert list(out) == [M32, 0, 0]
    # a carried bit completes a four (test_csa.cpp:80-88)
    out = pp.microop(1, 2, [1, 0, 1, 1, 1, 0], 3)
    assert list(out) == [1, 0, 0]
    # zeros in, zeros out (depth 3)
    assert not pp.microop(1, 3, [0] * (3 + 8), 1 + 3).any()


@pytest.mark.parametrize("depth", [2, 3, 4, 5, 6, 7])
def test_tree_matches_oracle_and_conserves(pp, dev, orc, depth):  # test_csa.cpp:115-139
    rng = np.random.default_rng(777 + depth)
    blocks = 25
    inputs = rng.integers(0, 2**32, size=blocks << depth, dtype=np.uint64)
    carries0 = rng.integers(0, 2**32, size=depth, dtype=np.uint64)
    out = pp.microop(1, depth, np.concatenate([carries0, inputs]), blocks + depth)
    tops, carries = out[:blocks].astype(np.uint64), out[blocks:].astype(np.uint64)
    mine = np.zeros(8, np.uint64)
    mine[:depth] = carries0
    want_tops = [orc.csa_tree(depth, mine, np.ascontiguousarray(inputs[b << depth:(b + 1) << depth]))[0] & M32
                 for b in range(blocks)]
    assert [int(x) for x in tops] == want_tops and (carries == mine[:depth]).all()
    ch = np.arange(32, dtype=np.uint64)
    bits = lambda v: ((np.asarray(v, np.uint64)[..., None] >> ch) & np.uint64(1)).astype(np.int64)
    fed = bits(inputs).sum(0) + sum(bits(carries0[j]) << j for j in range(depth))
    left = sum(bits(carries[j]) << j for j in range(depth))
    assert (left + (bits(tops).sum(0) << depth) == fed).all()


def test_extract_kats(pp, dev, orc):
    out = pp.microop(2, 1, [0x0003_0001], 16)  # lanes [1, 3]
    assert out[0] == 0x0001_0001 and out[1] == 0x0001_0000 and not out[2:].any()
    assert not pp.microop(2, 1, [0], 16).any()
    assert (pp.microop(2, 1, [M32, M32], 16) == 0x0002_0002).all()
    tops = np.random.default_rng(3).integers(0, 2**32, size=300, dtype=np.uint64)
    out = pp.microop(2, 1, tops, 16)
    for p in range(16):
        lo = int(((tops >> np.uint64(p)) & np.uint64(1)).sum())
        hi = int(((tops >> np.uint64(p + 16)) & np.uint64(1)).sum())
        assert int(out[p]) == (hi << 16) | lo


def test_drain_kats(pp, dev):  # finalize_carries KATs, test_csa.cpp:180-216
    out = pp.microop(3, 2, [0x0010, 0x0001], 16)  # channel 4 weight 1, channel 0 weight 2
    assert out[4] == 1 and out[0] == 2 and int(out.sum()) == 3
    assert not pp.microop(3, 4, [0, 0, 0, 0], 16).any()
    out = pp.microop(3, 3, [0, 0, M32], 16)  # all-ones B2: 4 per lane
    assert (out == 0x0004_0004).all()
    rng = np.random.default_rng(9)
    for depth in range(1, 8):
        car = rng.integers(0, 2**32, size=depth, dtype=np.uint64)
        out = pp.microop(3, depth, car, 16)
        for p in range(16):
            lo = sum(((int(car[j]) >> p) & 1) << j for j in range(depth))
            hi = sum(((int(car[j]) >> (p + 16)) & 1) << j for j in range(depth))
            assert int(out[p]) == (hi << 16) | lo


def test_warp_channel_totals(pp, dev):
    rng = np.random.default_rng(10)
    lanes = rng.integers(0, 65536, size=(32, 16, 2), dtype=np.uint64)  # 16-bit lane counters per lane
    shift = 7
    inp = np.zeros((32, 17), np.uint64)
    inp[:, :16] = lanes[:, :, 0] | (lanes[:, :, 1] << np.uint64(16))
    inp[:, 16] = shift
    out = pp.microop(4, 1, inp.ravel(), 32)
    for c in range(32):
        want = int((lanes[:, c % 16, c // 16] << np.uint64(shift)).sum()) & M32
        assert int(out[c]) == want
