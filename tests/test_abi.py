"""CPU-side checks of the C ABI library: it loads, exports every symbol the
header declares, validates like the reference, and refuses to count without
a GPU (there is no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pospopcnt_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(pospop[a-z_0-9]*)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pospopcnt_u8", "pospopcnt_u16", "pospopcnt_u32", "pospopcnt_u64", "pospopcnt_u16_config",
                 "pospopcnt_u16_c32", "pospopcnt_segmented", "pospopcnt_sharded", "pospopcnt_async",
                 "pospop_last_error", "pospop_validate"):
        assert must in names


def test_library_exports_every_declared_symbol(pp):
    lib = ctypes.CDLL(pp.library_path())
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", pp.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\S+)", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a_only(pp):
    out = subprocess.run(["cuobjdump", "-lelf", pp.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")), out


def _kernel_sass(pp, pattern):
    """SASS of the kernels whose mangled names match `pattern` (cuobjdump -fun)."""
    names = subprocess.run(["cuobjdump", "-symbols", pp.library_path()], capture_output=True, text=True).stdout
    funs = sorted(set(re.findall(r"STO_ENTRY\s+(\S*" + pattern + r"\S*)", names)))
    assert funs, pattern
    return funs, subprocess.run(["cuobjdump", "-sass", "-fun", funs[0], pp.library_path()],
                                capture_output=True, text=True).stdout


def test_sass_uses_lop3_csa_and_256bit_loads(pp):
    """The default k <= 32 counting kernel, stream_kernel<1,7,32,0,256,2,0,1>
    (DESIGN.md 3.1): LOP3 CSAs with the reference's vpternlogd immediates and
    256-bit non-allocating vector loads."""
    funs, sass = _kernel_sass(pp, r"stream_kernelILi1ELi7ELi32ELi0ELi256ELi2ELi0ELi1E")
    assert "LOP3.LUT" in sass and "0xe8" in sass and "0x96" in sass
    assert "LDG.E.NA.ENL2.256.CONSTANT" in sass, funs


def test_sass_flag_ring_kernel_uses_bulk_copies_and_mbarriers(pp):
    """The default FLAG kernel, stream_ring_kernel<3,5,2,16,1>:
    per-warp cp.async.bulk (UBLKCP) into shared memory completing on mbarriers
    (SYNCS.*), swizzled LDS.128 reads, PRMT byte regrouping and LOP3 CSAs."""
    funs, sass = _kernel_sass(pp, r"stream_ring_kernelILi3ELi5ELi2ELi16ELi1E")
    for op in ("UBLKCP", "SYNCS.ARRIVE.TRANS64", "SYNCS.PHASECHK.TRANS64", "LDS.128", "PRMT", "LOP3.LUT"):
        assert op in sass, (op, funs)


def _entries(path):
    out = subprocess.run(["cuobjdump", "-symbols", path], capture_output=True, text=True).stdout
    return sorted(set(re.findall(r"STO_ENTRY\s+(\S+)", out)))


def test_release_library_holds_only_production_kernels(pp):
    """The release .so instantiates the production kernels only (<= 20
    entries) and reads no tuning knob; the tuning build carries the measured
    alternatives and the POSPOP_* knobs (tools/ sweeps, tuning tests)."""
    release = _entries(pp.library_path("release"))
    assert 0 < len(release) <= 20, release
    strings = subprocess.run(["strings", pp.library_path("release")], capture_output=True, text=True).stdout
    for knob in ("POSPOP_STREAM_VARIANT", "POSPOP_FLUSH_THRESHOLD", "POSPOP_SEG_VARIANT", "POSPOP_FLAG_VARIANT",
                 "POSPOP_SMALL_BYTES", "POSPOP_TMA", "POSPOP_PDL"):
        assert knob not in strings, knob
    tuning = _entries(pp.library_path("tuning"))
    assert set(release) < set(tuning) and len(tuning) > 100
    tstrings = subprocess.run(["strings", pp.library_path("tuning")], capture_output=True, text=True).stdout
    assert "POSPOP_STREAM_VARIANT" in tstrings and "POSPOP_FLUSH_THRESHOLD" in tstrings


def test_validate_like_reference(pp):  # test_core.cpp:184-201
    pp.validate(pp.PospopcntConfig(flush_threshold_blocks=1))
    with pytest.raises(pp.InvalidArgument):
        pp.validate(pp.PospopcntConfig(flush_threshold_blocks=0))
    with pytest.raises(pp.InvalidArgument):
        pp.validate(pp.PospopcntConfig(flush_threshold_blocks=65536))
    with pytest.raises(pp.InvalidArgument):
        pp.validate(pp.PospopcntConfig(register_width_bits=100))
    pp.validate(pp.PospopcntConfig(register_width_bits=128))  # shape-valid; availability is per kernel


def test_kernel_names_round_trip(pp):  # test_core.cpp:203-211
    for kind in pp.KernelKind:
        assert pp.KernelKind.from_string(str(kind)) == kind
    assert pp.KernelKind.from_string("warp") is None


def test_supported_widths(pp):  # test_core.cpp:213-219
    w = pp.supported_csa_widths()
    assert w == sorted(w) and w[0] == 64 and pp.native_csa_width() >= 64


def test_merge_counts_and_total(pp):  # test_core.cpp:84-107
    a = pp.PositionalCounts(range(16))
    b = pp.PositionalCounts([3] * 16)
    assert pp.merge_counts(a, b) == pp.merge_counts(b, a)
    assert pp.merge_counts(pp.PositionalCounts(), a) == a
    assert a.total() == sum(range(16))


def test_no_gpu_means_loud_failure(pp):
    """Without an sm_100 device the product path raises; it never counts on the CPU."""
    if pp.device_available():
        pytest.skip("a GPU is present")
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt(np.arange(100, dtype=np.uint16))
    with pytest.raises(pp.KernelUnavailableError):
        pp.pospopcnt_k(np.zeros(64, np.uint8), 8)


def test_argument_errors_before_device(pp):
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_k(np.zeros(4, np.uint8), 12)
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_k(np.zeros(8, np.uint8), 16, flush_threshold_blocks=0)
    lib = pp._load()
    u64 = (ctypes.c_uint64 * 16)()
    assert lib.pospopcnt_u16(None, 5, u64) == 1  # NULL with len > 0
    buf = np.zeros(9, np.uint8)
    assert lib.pospopcnt_u16(ctypes.c_void_p(buf.ctypes.data + 1), 4, u64) == 1  # misaligned u16*


def test_package_does_not_import_the_oracle():
    """The product package must never route through the checker."""
    pkg = os.path.join(ROOT, "paper_1911_02696_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                bad = re.search(r"import\s+pyoracle|from\s+pyoracle|#include[^\n]*pospop_oracle|liboracle\.so|"
                                r"libpospop_ref|oracle/_ref", text)
                assert not bad, (f, bad)


def test_cli_usage_errors_without_gpu(tmp_path):
    """Exit code 2 for usage/input errors (proj/tools/pospopcnt.cpp:43-45); no CPU fallback."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-m", "paper_1911_02696_b200", "count"], cwd=ROOT, capture_output=True)
    assert r.returncode == 2
    r = subprocess.run([sys.executable, "-m", "paper_1911_02696_b200", "count", "--input", str(tmp_path / "nope")],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 2 and "error" in r.stderr


def build_c_smoke(pp, tmp_path):
    exe = tmp_path / "abi_c_smoke"
    libdir = os.path.dirname(pp.library_path())
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-pedantic",
                           "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "abi_c_smoke.c"),
                           "-L", libdir, "-lpospopcnt_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    return exe


def test_header_is_plain_c_and_fails_loudly_without_gpu(pp, tmp_path):
    """include/pospopcnt_b200.h compiles as strict C11; without a GPU the library
    answers POSPOP_EUNAVAILABLE (exit 2) instead of counting on the CPU."""
    exe = build_c_smoke(pp, tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    if pp.device_available():
        assert r.returncode == 0, r.stdout
    else:
        assert r.returncode == 2, (r.returncode, r.stdout)


def test_segmented_wrappers_check_offsets_and_rows(pp):
    """Offsets must be 64-bit integers with >= 1 element; rows must hold
    exactly n_arrays * k 8-byte integers (checked before any device work)."""
    data = np.zeros(64, np.uint16)
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_segmented(data, np.zeros(0, np.uint64), 16)
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_segmented(data, np.array([0, 4], np.float64), 16)
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_segmented(data, np.array([0, 4, 8], np.uint64), 16, out=np.zeros((1, 16), np.uint64))
    with pytest.raises(pp.InvalidArgument):
        pp.pospopcnt_segmented(data, np.array([0, 4], np.uint64), 16, out=np.zeros(16, np.float64))
    torch = pytest.importorskip("torch")
    with pytest.raises(pp.InvalidArgument):
        pp.segmented_async(data, torch.tensor([0, 4], dtype=torch.int32), np.zeros(16, np.uint64), 16)
    with pytest.raises(pp.InvalidArgument):
        pp.segmented_async(data, torch.zeros(0, dtype=torch.int64), np.zeros(0, np.uint64), 16)
    with pytest.raises(pp.InvalidArgument):
        pp.segmented_async(data, torch.tensor([0, 4], dtype=torch.int64), torch.zeros(15, dtype=torch.int64), 16)
