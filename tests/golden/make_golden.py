"""Regenerates tests/golden/*.json from the REFERENCE library itself.

Run in the dev container (needs oracle/_ref/libpospop_ref.so, which
oracle/Makefile compiles from /root/reference):

    python tests/golden/make_golden.py

The rng replays below follow the reference's own test sources so the
fixtures are exactly the cases those tests check:

* acceptance.cpp:103-146   -- 1000 random streams (seed 0xACCE97), then the
                              forced-flush lengths 7003 / 9216 from the same rng
* test_core.cpp:109-125    -- 40 random streams (seed 2024), len 10007 seed 5
* test_core.cpp:136-141    -- Auto boundary 4095 / 4096 (seed 11)
* test_core.cpp:143-153    -- concatenation cuts (seed 31337)
* test_csa.cpp:252-292     -- forced flush (seed 555), threshold 1, tail lengths (seed 2)
* bench.cpp:115-120        -- generate_stream words for several seeds; cfg1 (seed 1, 2^20)
* acceptance.cpp:271-291   -- 100 FLAG streams of 10^5 words (seed 0xF1A6) and the 4096
                              single-value summaries, from flagstats_reference
* k = 8/32/64              -- generate_stream bytes as k-bit words, counted by the
                              reference's 16-bit API after the SURVEY 8c restatement

Counts come from pospop::pospopcnt (Auto and every CSA width) and
pospop::oracle_pospopcnt; the script asserts they agree before writing.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle  # noqa: E402


class MT64:
    """std::mt19937_64 draws through the C restatement (pinned below)."""

    def __init__(self, oracle: pyoracle.Oracle, seed: int):
        import ctypes
        self._lib = oracle.lib
        self._state = ctypes.create_string_buffer(312 * 8 + 8)
        self._lib.orc_mt64_seed.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        self._lib.orc_mt64_next.argtypes = [ctypes.c_void_p]
        self._lib.orc_mt64_next.restype = ctypes.c_uint64
        self._lib.orc_mt64_seed(self._state, seed)

    def __call__(self) -> int:
        return int(self._lib.orc_mt64_next(self._state))


def counts_of(ref: pyoracle.Reference, words: np.ndarray, **kw) -> list[int]:
    rc, c = ref.pospopcnt(words, **kw)
    assert rc == 0, rc
    o = ref.oracle(words)
    assert (c == o).all()
    return [int(x) for x in c]


def main() -> None:
    pyoracle.build()
    ref = pyoracle.Reference()
    orc = pyoracle.Oracle()
    out: dict = {"source": "reference library proj/core compiled by oracle/Makefile",
                 "widths_on_generating_host": ref.supported_widths()}

    # generate_stream vectors (bench.cpp:115-120)
    gs = []
    for seed in [0, 1, 7, 40, 0xBE9C, 2**63 + 5]:
        w = ref.generate_stream(seed, 4096)
        gs.append({"seed": seed, "first32": [int(x) for x in w[:32]],
                   "counts4096": counts_of(ref, w)})
    out["generate_stream"] = gs

    # cfg1: 2^20 uniform words, seed 1, uint32 counters
    w = ref.generate_stream(1, 1 << 20)
    out["cfg1"] = {"seed": 1, "len": 1 << 20, "counts": counts_of(ref, w)}

    # acceptance.cpp:103-146
    rng = MT64(orc, 0xACCE97)
    acc = []
    for _ in range(1000):
        n = rng() % 10001
        seed = rng()
        acc.append([seed, n] + counts_of(ref, ref.generate_stream(seed, n)))
    out["acceptance_random"] = acc
    flush3 = []
    for n in (7003, 9216):
        seed = rng()
        w = ref.generate_stream(seed, n)
        expected = counts_of(ref, w)
        for kern in ("csa4", "csa8", "csa16"):
            for width in ref.supported_widths():
                assert counts_of(ref, w, kernel=kern, width=width, flush=3) == expected
        flush3.append([seed, n] + expected)
    out["acceptance_flush3"] = flush3

    # test_core.cpp:109-125
    rng = MT64(orc, 2024)
    disp = []
    for _ in range(40):
        n = rng() % 3000
        seed = rng()
        disp.append([seed, n] + counts_of(ref, ref.generate_stream(seed, n)))
    out["dispatcher_random"] = disp
    out["scalar_vs_csa16"] = [5, 10007] + counts_of(ref, ref.generate_stream(5, 10007), kernel="csa16")
    out["auto_boundary"] = [[11, n] + counts_of(ref, ref.generate_stream(11, n)) for n in (4095, 4096)]

    # test_core.cpp:143-153 concatenation homomorphism
    rng = MT64(orc, 31337)
    cuts = []
    for _ in range(20):
        seed = rng()
        n = 1 + rng() % 2000
        cut = rng() % (n + 1)
        w = ref.generate_stream(seed, n)
        cuts.append([seed, n, cut] + counts_of(ref, w))
    out["concat_cuts"] = cuts

    # test_csa.cpp:252-292
    rng = MT64(orc, 555)
    f3 = []
    for n in (4000, 9000):
        seed = rng()
        w = ref.generate_stream(seed, n)
        f3.append([seed, n] + counts_of(ref, w, kernel="csa4", flush=3))
    out["csa_flush3"] = f3
    out["csa_flush1"] = [8, 1000] + counts_of(ref, ref.generate_stream(8, 1000), kernel="csa4", flush=1)
    rng = MT64(orc, 2)
    tails = []
    for n in (1, 3, 63, 64, 65, 511, 512, 513, 1023):
        seed = rng()
        tails.append([seed, n] + counts_of(ref, ref.generate_stream(seed, n), kernel="csa16"))
    out["csa_tails"] = tails
    # fork-join over 40000 words (test_core.cpp:155-175)
    w = ref.generate_stream(77, 40000)
    out["fork_join"] = [77, 40000] + [int(x) for x in ref.pospopcnt_mt(w, 4)]

    # acceptance.cpp:271-291 (criterion 5): 100 FLAG streams of 10^5 words,
    # mt19937_64(0xF1A6), word = rng() & 0x0FFF; summaries from the reference.
    rng = MT64(orc, 0xF1A6)
    flag_rows = []
    for _ in range(100):
        words = np.array([rng() & 0x0FFF for _ in range(100000)], np.uint16)
        rc, summ, _ = ref.flagstats(words, use_pospopcnt=False)
        rc2, summ2, _ = ref.flagstats(words, use_pospopcnt=True)
        assert rc == 0 and rc2 == 0 and (summ == summ2).all()
        flag_rows.append([int(x) for x in summ])
    out["flagstats_acceptance"] = flag_rows
    single = []
    for v in range(4096):
        rc, summ, _ = ref.flagstats(np.array([v], np.uint16), use_pospopcnt=False)
        single.append([int(x) for x in summ])
    out["flagstats_single"] = single

    # k = 8 / 32 / 64 (no reference function): streams of the
    # reference's generate_stream bytes read as k-bit words at several byte
    # offsets and lengths, counted by the reference's own 16-bit pospopcnt
    # after the 8c restatement (ref_segmented: k=8 fold with a direct odd
    # head/tail byte, k=32/64 deinterleave).  [seed, k, byte_offset, n_words, counts...]
    kw = []
    for seed, k, off, n in ((21, 8, 0, 100003), (22, 8, 1, 65537), (23, 8, 3, 7), (24, 32, 0, 50001),
                            (25, 32, 4, 4097), (26, 64, 0, 30011), (27, 64, 8, 513), (28, 64, 0, 1)):
        wb = k // 8
        raw = ref.generate_stream(seed, (off + n * wb) // 2 + 2).view(np.uint8)[off:off + n * wb]
        dt = {8: np.uint8, 32: np.uint32, 64: np.uint64}[k]
        words = np.frombuffer(raw.tobytes(), dt)
        rows = ref.segmented(words, np.array([0, n], np.uint64), k, threads=1)
        assert (rows[0] == orc.naive(raw, k)).all()
        kw.append([seed, k, off, n] + [int(x) for x in rows[0]])
    out["k_widths"] = kw

    with open(os.path.join(HERE, "reference_counts.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))

    # Generator fixtures (counter-based synthetic inputs).  These
    # pin the device generators; produced by the C restatement.
    gens = {}
    for kind in range(1, 9):
        for seed, base in ((1, 0), (1, 123456789), (42, 2**33 + 17)):
            a = orc.generate(kind, seed, 1 << 16, base=base)
            gens[f"{kind}:{seed}:{base}"] = {"first16": [int(x) for x in a[:16]],
                                             "digest": orc.digest(a)}
    with open(os.path.join(HERE, "generators.json"), "w") as f:
        json.dump(gens, f, indent=1)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
