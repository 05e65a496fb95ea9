"""Every kernel family against the bounds-checked build of the library
(libpospopcnt_b200_debug.so, -DPOSPOP_DEBUG_BOUNDS: each vector load traps
unless its index is inside the valid range of the stream or array) on
unaligned starts, ragged ends and ragged segment tables, results still
checked against the oracle.  compute-sanitizer is unavailable on the GPU
pool, so out-of-range loads are caught by the kernels' own asserts."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_out_of_range_vector_loads():
    lib = os.path.join(ROOT, "paper_1911_02696_b200", "libpospopcnt_b200_debug.so")
    if not os.path.exists(lib):
        pytest.skip("bounds-checked library not built (make -C paper_1911_02696_b200/csrc debug)")
    env = dict(os.environ, POSPOP_LIBRARY=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "bounds_worker.py")], capture_output=True,
                       text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0 and "bounds ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
