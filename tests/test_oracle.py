"""Pins the CPU oracle (oracle/pospop_oracle.c) before anything trusts it.

* against the reference's own known-answer tests, restated from
  proj/tests/test_core.cpp, test_csa.cpp and acceptance.cpp;
* against golden vectors produced by the reference library itself
  (tests/golden/reference_counts.json, tests/golden/make_golden.py);
* against the reference library live, when oracle/_ref was built here.
"""
import numpy as np
import pytest

COUNTRY = np.array([0x10, 0x10, 0x04, 0x10, 0x01, 0x04, 0x01, 0x01, 0x01, 0x20], np.uint16)
LOW_IMM, HIGH_IMM = 0b10010110, 0b11101000  # test_csa.cpp:29-30


def expect(counts, row):
    assert [int(x) for x in counts] == list(row)


# -- ground truth KATs (test_core.cpp:46-82) ------------------------------------

def test_empty_stream(orc):
    assert not orc.naive(np.zeros(0, np.uint16)).any()
    assert not orc.run_csa64(np.zeros(0, np.uint16)).any()


def test_country_histogram(orc):  # common.hpp:24-31, test_core.cpp:51-60
    for c in (orc.naive(COUNTRY), orc.run_csa64(COUNTRY), orc.pospopcnt(COUNTRY, 16)):
        assert c[0] == 4 and c[2] == 2 and c[4] == 3 and c[5] == 1 and c.sum() == 10


def test_all_ones_and_repeated(orc):  # test_core.cpp:62-73
    assert (orc.naive(np.array([0xFFFF], np.uint16)) == 1).all()
    c = orc.run_csa64(np.full(100, 1, np.uint16))
    assert c[0] == 100 and c[1:].sum() == 0


def test_invariants(orc):  # test_core.cpp:75-82
    s = orc.mt_generate_stream(7, 333)
    c = orc.naive(s)
    assert c.sum() == sum(bin(int(w)).count("1") for w in s)
    assert (c <= s.size).all()


def test_exhaustive_single_word_domain(orc):  # test_kernels.cpp:120-136, verify.cpp:40-55
    words = np.arange(65536, dtype=np.uint16)
    # one call per word would be 65536 FFI calls; the segmented oracle does it in one
    got = orc.segmented(words, np.arange(65537, dtype=np.uint64), 16)
    want = ((words[:, None].astype(np.uint32) >> np.arange(16)) & 1).astype(np.uint64)
    assert (got == want).all()


# -- mt19937_64 / generate_stream pinned against the reference's output ------------

def test_generate_stream_vectors(orc, golden):
    for case in golden["generate_stream"]:
        w = orc.mt_generate_stream(case["seed"], 4096)
        assert [int(x) for x in w[:32]] == case["first32"]
        expect(orc.naive(w), case["counts4096"])


def test_cfg1_counts(orc, golden):
    c = golden["cfg1"]
    w = orc.mt_generate_stream(c["seed"], c["len"])
    expect(orc.run_csa64(w), c["counts"])
    expect(orc.naive(w), c["counts"])


# -- the reference tests' random streams (golden counts from the reference) ----------

@pytest.mark.parametrize("key", ["acceptance_random", "dispatcher_random", "csa_tails", "auto_boundary"])
def test_reference_random_streams(orc, golden, key):
    for row in golden[key]:
        seed, n, want = row[0], row[1], row[2:]
        w = orc.mt_generate_stream(seed, n)
        expect(orc.run_csa64(w, 4), want)
        expect(orc.pospopcnt(w, 16), want)
    # naive on a subset (it is the slow path)
    for row in golden[key][:50]:
        expect(orc.naive(orc.mt_generate_stream(row[0], row[1])), row[2:])


def test_forced_flush(orc, golden):  # test_csa.cpp:252-278, acceptance.cpp:119-146
    for key in ("acceptance_flush3", "csa_flush3"):
        for seed, n, *want in golden[key]:
            w = orc.mt_generate_stream(seed, n)
            for depth in (2, 3, 4):
                expect(orc.run_csa64(w, depth, 3), want)
    seed, n, *want = golden["csa_flush1"]
    expect(orc.run_csa64(orc.mt_generate_stream(seed, n), 2, 1), want)


def test_lane_saturation(orc):  # test_csa.cpp:294-305
    n = 16 * 4 * 65536 + 3
    c = orc.run_csa64(np.full(n, 0xFFFF, np.uint16), 2, 65535)
    assert (c == n).all()


def test_concatenation_and_fork_join(orc, golden):  # test_core.cpp:143-175
    for seed, n, cut, *want in golden["concat_cuts"]:
        w = orc.mt_generate_stream(seed, n)
        expect(orc.run_csa64(w[:cut]) + orc.run_csa64(w[cut:]), want)
    seed, n, *want = golden["fork_join"]
    w = orc.mt_generate_stream(seed, n)
    expect(orc.pospopcnt(w, 16, threads=4), want)


def test_order_independence(orc):  # test_core.cpp:177-182
    w = orc.mt_generate_stream(17, 1234)
    assert (orc.run_csa64(w) == orc.run_csa64(np.random.default_rng(4).permutation(w))).all()


def test_config_range_rejected(orc):
    with pytest.raises(ValueError):
        orc.run_csa64(np.zeros(8, np.uint16), 4, 0)
    with pytest.raises(ValueError):
        orc.run_csa64(np.zeros(8, np.uint16), 4, 65536)


# -- CSA micro-op KATs (test_csa.cpp:32-216) ---------------------------------------

def test_csa_truth_table(orc):
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                h, l = orc.csa(a, b, c)
                m = a + 2 * b + 4 * c
                assert 2 * h + l == a + b + c
                assert l == (LOW_IMM >> m) & 1 and h == (HIGH_IMM >> m) & 1


def test_csa_examples_and_wide_identity(orc):
    assert orc.csa(0b1010, 0b0110, 0b1100) == (0b1110, 0)
    rng = np.random.default_rng(12345)
    for a, b, c in rng.integers(0, 2**63, size=(500, 3), dtype=np.uint64):
        a, b, c = int(a) * 2 + 1, int(b), int(c)
        a &= (1 << 64) - 1
        h, l = orc.csa(a, b, c)
        for ch in range(0, 64, 7):
            bit = lambda v: (v >> ch) & 1
            assert 2 * bit(h) + bit(l) == bit(a) + bit(b) + bit(c)


def test_csa_block_kats(orc):
    carries = np.zeros(8, np.uint64)
    top, calls = orc.csa_tree(2, carries, np.full(4, 2**64 - 1, np.uint64))
    assert top == 2**64 - 1 and not carries.any() and calls == 3
    carries = np.zeros(8, np.uint64)
    carries[0] = 1
    top, _ = orc.csa_tree(2, carries, np.array([1, 1, 1, 0], np.uint64))
    assert top == 1 and not carries.any()
    for depth in (2, 3, 4):
        carries = np.zeros(8, np.uint64)
        _, calls = orc.csa_tree(depth, carries, np.full(1 << depth, 0xDEADBEEF, np.uint64))
        assert calls == (1 << depth) - 1


def test_csa_conservation(orc):  # test_csa.cpp:115-139
    rng = np.random.default_rng(777)
    for depth in (2, 3, 4, 5, 6):
        carries = np.zeros(8, np.uint64)
        fed = np.zeros(64, np.int64)
        emitted = np.zeros(64, np.int64)
        for _ in range(25):
            inputs = rng.integers(0, 2**64 - 1, size=1 << depth, dtype=np.uint64)
            fed += ((inputs[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).sum(0).astype(np.int64)
            top, _ = orc.csa_tree(depth, carries, inputs)
            emitted += ((np.uint64(top) >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(np.int64)
        residual = sum(((carries[j] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(np.int64) << j
                       for j in range(depth))
        assert (residual + (emitted << depth) == fed).all()


def test_extract_flush_finalize_kats(orc):
    bank = np.zeros(16, np.uint64)
    blocks = orc.extract_top(0x0002_0000_0003_0001, bank, 0)
    assert blocks == 1 and bank[0] == 0x0000_0000_0001_0001 and bank[1] == 0x0001_0000_0001_0000
    assert not bank[2:].any()
    bank = np.zeros(16, np.uint64)
    orc.extract_top(2**64 - 1, bank, 0)
    orc.extract_top(2**64 - 1, bank, 1)
    assert (bank == 0x0002_0002_0002_0002).all()
    bank = np.zeros(16, np.uint64)
    bank[0] = 0x0001_0000_0002_0003
    counts = np.zeros(16, np.uint64)
    assert orc.flush_bank(bank, 3, counts, 16) == 0
    assert counts[0] == 96 and not counts[1:].any() and not bank.any()
    carries = np.zeros(8, np.uint64)
    carries[0], carries[1] = 0x0010, 0x0001
    counts = np.zeros(16, np.uint64)
    orc.finalize_carries(carries, 2, counts)
    assert counts[4] == 1 and counts[0] == 2 and counts.sum() == 3
    carries = np.zeros(8, np.uint64)
    carries[2] = 2**64 - 1
    counts = np.zeros(16, np.uint64)
    orc.finalize_carries(carries, 3, counts)
    assert (counts == 16).all()


# -- k != 16 restatements ---------------------------------------------------------------

@pytest.mark.parametrize("k", [8, 16, 32, 64])
@pytest.mark.parametrize("offset", [0, 1, 3, 8])
def test_k_restatement_vs_naive(orc, k, offset):
    raw = orc.generate(6, 99, 3000).view(np.uint8)
    if offset % (k // 8):
        pytest.skip("word-misaligned start")
    for n in (0, 1, 7, 4096 * 8 // k, (raw.size - offset) * 8 // k):
        buf = raw[offset:offset + n * k // 8]
        assert (orc.pospopcnt(buf, k) == orc.naive(buf, k)).all(), (k, offset, n)
        assert (orc.pospopcnt(buf, k, threads=3) == orc.naive(buf, k)).all()


def test_k32_needs_deinterleave(orc):  # 0x00010000 -> position 16, not 0
    c = orc.pospopcnt(np.array([0x00010000], np.uint32), 32)
    assert c[16] == 1 and c.sum() == 1


def test_segmented_oracle(orc):
    data = orc.generate(5, 3, 10000)
    offs = np.array([0, 0, 1, 17, 4113, 9999, 10000], np.uint64)
    got = orc.segmented(data, offs, 32, threads=2)
    for a in range(len(offs) - 1):
        assert (got[a] == orc.naive(data[int(offs[a]):int(offs[a + 1])], 32)).all()


# -- the synthetic-input generators ---------------------------------------------------------

def test_generator_fixtures(orc, golden_generators):
    for key, v in golden_generators.items():
        kind, seed, base = (int(x) for x in key.split(":"))
        a = orc.generate(kind, seed, 1 << 16, base=base, threads=3)
        assert [int(x) for x in a[:16]] == v["first16"], key
        assert orc.digest(a) == v["digest"], key


def test_generator_properties(orc):
    z = orc.generate(2, 1, 1 << 18)
    assert (np.bitwise_count(z) == 1).all()  # one-hot
    c = orc.naive(z)
    assert c.sum() == z.size and c[0] > c[1] > c[15]  # Zipf ranks
    b = orc.naive(orc.generate(4, 1, 1 << 18))
    assert abs(b.sum() / (16 * (1 << 18)) - 6554 / 65536) < 2e-3  # Bernoulli(0.1)
    by = orc.generate(3, 1, 1 << 14)
    assert (np.bitwise_count(by[:4096]) == 1).all()  # even run: one-hot


# -- live cross-check against the reference library, when built here ------------------------

def test_oracle_matches_reference_live(orc, ref):
    rng = np.random.default_rng(5)
    for n in list(range(0, 70)) + [4095, 4096, 10007, 1 << 16]:
        w = rng.integers(0, 65536, size=n, dtype=np.uint16)
        rc, c = ref.pospopcnt(w)
        assert rc == 0 and (c == orc.run_csa64(w)).all() and (c == orc.naive(w)).all()
    for seed in (0, 1, 2**64 - 1):
        assert (ref.generate_stream(seed, 1000) == orc.mt_generate_stream(seed, 1000)).all()


def test_micro_ops_match_reference_live(orc, ref):
    rng = np.random.default_rng(6)
    for _ in range(200):
        a, b, c = (int(x) for x in rng.integers(0, 2**63, size=3))
        assert orc.csa(a, b, c) == ref.csa(a, b, c)
    for depth in (2, 3, 4):
        regs = rng.integers(0, 2**63, size=4, dtype=np.uint64)
        regs[depth:] = 0
        inputs = rng.integers(0, 2**63, size=1 << depth, dtype=np.uint64)
        mine = np.zeros(8, np.uint64)
        mine[:4] = regs
        top, calls = orc.csa_tree(depth, mine, inputs)
        rc, rtop, rcalls = ref.csa_block(depth, regs, inputs)
        assert rc == 0 and top == rtop and calls == rcalls and (mine[:4] == regs).all()


def test_reference_validation_semantics(ref):  # test_core.cpp:184-201
    assert ref.validate(flush=0) == 1 and ref.validate(flush=65536) == 1 and ref.validate(flush=1) == 0
    assert ref.validate(width=100) == 1
    rc, _ = ref.pospopcnt(np.zeros(8, np.uint16), kernel="csa16", width=128)
    assert rc == 2


# -- FLAG statistics (acceptance.cpp:271-291) ----------------------------

def test_flagstats_oracle_vs_golden(orc, golden):
    for v in range(4096):  # exhaustive single flag values
        w = np.array([v], np.uint16)
        rc, got, _ = orc.flagstats(w)
        rc2, got2, _ = orc.flagstats(w, "pospop")
        assert rc == rc2 == 0 and list(got) == golden["flagstats_single"][v] == list(got2), v
    streams = orc.acceptance_flag_streams()
    for i in range(0, 100, 9):
        rc, got, _ = orc.flagstats(streams[i])
        rc2, got2, _ = orc.flagstats(streams[i], "pospop")
        assert rc == rc2 == 0 and list(got) == golden["flagstats_acceptance"][i] == list(got2), i


def test_flagstats_invalid_word_first_offset(orc):
    w = orc.generate(7, 3, 5000)
    assert w.max() < 0x1000
    w[4000] |= 0x2000
    w[1234] |= 0x8000
    for route in ("reference", "pospop"):
        rc, _, bad = orc.flagstats(w, route)
        assert rc == 1 and bad == 1234


def test_flagstats_oracle_matches_reference_live(orc, ref):
    w = orc.generate(7, 11, 200000)
    rc, a, _ = orc.flagstats(w)
    rr, b, _ = ref.flagstats(w)
    assert rc == rr == 0 and (a == b).all()
    w[77] |= 0x1000
    assert orc.flagstats(w)[0::2] == ref.flagstats(w)[0::2] == (1, 77)


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_reference_segmented_restatement_matches_oracle(orc, ref, k):
    """The reference-based cfg5 baseline (ref_segmented: the reference's 16-bit
    pospopcnt per array after the SURVEY 8c deinterleave / fold) equals the
    oracle's segmented count, including odd byte starts for k = 8."""
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[k]
    data = orc.generate(6, 8 + k, 5000).view(dt)
    n = data.size
    rng = np.random.default_rng(k)
    offs = np.concatenate([[0, 0, 1], np.sort(rng.integers(1, n, 40)), [n]]).astype(np.uint64)
    assert (ref.segmented(data, offs, k, threads=3) == orc.segmented(data, offs, k, threads=2)).all()


def test_k_widths_against_reference_fixtures(orc, golden):
    """k = 8/32/64 counts from the reference library's own 16-bit API (golden
    k_widths, make_golden.py) reproduced by the oracle."""
    ref_words = {}
    for seed, k, off, n, *counts in golden["k_widths"]:
        wb = k // 8
        raw = orc.mt_generate_stream(seed, (off + n * wb) // 2 + 2).view(np.uint8)[off:off + n * wb]
        assert [int(x) for x in orc.pospopcnt(raw, k)] == counts, (seed, k, off, n)
