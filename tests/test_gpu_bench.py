"""bench.py on one leased GPU: the N = 1 line keeps the driver contract, and
`--gpus 2` without torchrun launches two ranks by itself, which find that
they share one GPU and refuse to print a headline (their aggregate would be
total bytes / max rank time, above any single GPU's ceiling)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _bench(args, env=None, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=dict(os.environ, **(env or {})), cwd=ROOT)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r, lines


def test_n1_line_contract():
    r, lines = _bench(["--workload", "cfg2", "--steps", "5", "--warmup", "3", "--no-cpu"])
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and "rejected" not in d
    assert d["roofline"]["kernel_ms_single_launch"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == (1 << 29)


def test_self_launch_refuses_shared_gpu():
    r, lines = _bench(["--gpus", "2", "--workload", "cfg2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"],
                      env={"POSPOP_BENCH_DIST_BACKEND": "gloo"})
    assert "launching 2 ranks" in r.stderr
    assert r.returncode != 0
    assert len(lines) == 1, r.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] is None and "share a GPU" in d["rejected"]


def test_shared_gpu_override_runs_the_n2_host_path():
    """Tests only: POSPOP_BENCH_ALLOW_SHARED_GPU=1 runs the two-rank path on
    one GPU (NCCL-fallback exchange over gloo; no kernel waits on another
    rank) and marks the line rejected."""
    r, lines = _bench(["--gpus", "2", "--workload", "cfg2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"],
                      env={"POSPOP_BENCH_DIST_BACKEND": "gloo", "POSPOP_BENCH_ALLOW_SHARED_GPU": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and "share a GPU" in d["rejected"]
    assert d["config"]["collective"] == "nccl"
