"""Host ingestion from files and pipes and the CLI mirror,
on the GPU: bit-exact against the oracle; errors as the reference tool
(proj/tools/pospopcnt.cpp:43-75)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COUNTRY = np.array([0x10, 0x10, 0x04, 0x10, 0x01, 0x04, 0x01, 0x01, 0x01, 0x20], np.uint16)


def cli(*args, stdin=None):
    return subprocess.run([sys.executable, "-m", "paper_1911_02696_b200", *args], cwd=ROOT, input=stdin,
                          capture_output=True, timeout=300)


def test_country_histogram_through_the_cli(tmp_path):  # acceptance.cpp:231-267 (criterion 4)
    path = tmp_path / "country.bin"
    path.write_bytes(COUNTRY.astype("<u2").tobytes())
    r = cli("count", "--input", str(path), "--json")
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    assert out["counts"] == [4, 0, 2, 0, 3, 1] + [0] * 10 and out["total_words"] == 10
    r = cli("count", "--input", "-", stdin=COUNTRY.tobytes())
    assert r.returncode == 0 and b"words: 10" in r.stdout and b"bit  0: 4" in r.stdout


def test_odd_byte_length_is_an_input_error(tmp_path):  # pospopcnt.cpp:53-55
    path = tmp_path / "odd.bin"
    path.write_bytes(b"\x01\x02\x03")
    r = cli("count", "--input", str(path))
    assert r.returncode == 2 and b"odd byte length" in r.stderr


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_file_ingestion_multi_chunk(pp, orc, tmp_path, k):
    n_bytes = (150 << 20) + 8 * 13  # > two 64 MiB chunks, ragged last chunk
    data = orc.generate(6, 21 + k, n_bytes // 8, threads=8).view(np.uint8)
    path = tmp_path / "words.bin"
    data.tofile(path)
    counts, n = pp.pospopcnt_file(str(path), k)
    assert n == n_bytes * 8 // k
    assert counts == orc.pospopcnt(data, k, threads=8)


def test_pipe_ingestion(pp, orc, tmp_path):
    data = orc.generate(4, 8, (3 << 20) + 5, threads=4)
    src = tmp_path / "src.bin"
    data.tofile(src)
    # a separate writer process streams the bytes through a pipe in odd-sized writes
    writer = subprocess.Popen([sys.executable, "-c",
                               "import sys\nraw = open(sys.argv[1], 'rb').read()\n"
                               "for i in range(0, len(raw), 99991):\n    sys.stdout.buffer.write(raw[i:i + 99991])\n"
                               "    sys.stdout.buffer.flush()\n", str(src)], stdout=subprocess.PIPE)
    try:
        counts, n = pp.pospopcnt_file(writer.stdout.fileno(), 16)
    finally:
        writer.stdout.close()
        writer.wait(timeout=60)
    assert n == data.size and counts == orc.pospopcnt(data, 16, threads=4)


def test_empty_and_ragged_files(pp, tmp_path):
    empty = tmp_path / "empty.bin"
    empty.write_bytes(b"")
    counts, n = pp.pospopcnt_file(str(empty), 16)
    assert n == 0 and counts.total() == 0
    ragged = tmp_path / "ragged.bin"
    ragged.write_bytes(b"\x00" * 4097)
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_file(str(ragged), 16)
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_file(str(tmp_path / "missing.bin"), 16)


def test_flagstats_cli(orc, tmp_path, golden):
    streams = orc.acceptance_flag_streams(count=1)
    path = tmp_path / "flags.bin"
    path.write_bytes(streams[0].astype("<u2").tobytes())
    r = cli("flagstats", "--input", str(path), "--json")
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    fields = ["total", "secondary", "supplementary", "n_pair_good", "n_read1", "n_read2", "n_sgltn", "pair_map",
              "mapped", "dup"]
    assert [out["pass"][f] for f in fields] + [out["fail"][f] for f in fields] == golden["flagstats_acceptance"][0]


def test_flagstats_cli_text_and_modes(pp, orc, tmp_path, golden):
    """Text output = the reference's format_flag_summary (flagstats.cpp:147-164);
    --mode reference|pospopcnt|differential as the reference tool; a reserved
    bit is a usage error (exit 2)."""
    streams = orc.acceptance_flag_streams(count=1)
    path = tmp_path / "flags.bin"
    path.write_bytes(streams[0].astype("<u2").tobytes())
    g = golden["flagstats_acceptance"][0]
    names = ["total", "secondary", "supplementary", "n_pair_good", "n_read1", "n_read2", "n_sgltn", "pair_map",
             "mapped", "dup"]
    want = "field           QC-pass\tQC-fail\n" + "".join(
        f"{n}{' ' * (16 - len(n))}{g[i]}\t{g[10 + i]}\n" for i, n in enumerate(names))
    for mode in ("reference", "pospopcnt"):
        r = cli("flagstats", "--input", str(path), "--mode", mode)
        assert r.returncode == 0 and r.stdout.decode() == want, (mode, r.stdout, r.stderr)
    r = cli("flagstats", "--input", str(path), "--mode", "differential")
    assert r.returncode == 0
    assert r.stdout.decode() == f"reference and pospopcnt summaries agree ({streams[0].size} words)\n" + want
    assert cli("flagstats", "--input", str(path), "--mode", "bogus").returncode == 2
    bad = streams[0].copy()
    bad[5] |= 0x2000
    path.write_bytes(bad.astype("<u2").tobytes())
    r = cli("flagstats", "--input", str(path))
    assert r.returncode == 2 and "offset 5" in r.stderr.decode()


def test_plain_c_caller_counts_on_gpu(pp, tmp_path):
    """A strict-C11 caller of include/pospopcnt_b200.h (tests/c/abi_c_smoke.c)."""
    from test_abi import build_c_smoke
    exe = build_c_smoke(pp, tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout)
