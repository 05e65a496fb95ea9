"""bench.py's reference arm on CPU (no GPU needed): one JSON line with the
driver contract's keys, for every workload (with --ref-words capping the
words per step so the CPU suite stays fast; the driver's run times the whole
workload), silent non-zero ranks under a two-rank launch (rank 0 alone
prints), and no self-launch for the reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


@pytest.mark.parametrize("workload", ["cfg4", "cfg3", "cfg5", "cfg5_u64", "flag"])
def test_reference_arm_line(workload):
    lines = _run(["--steps", "1", "--warmup", "1", "--workload", workload, "--ref-words", str(1 << 22)])
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["metric"].startswith("pospopcnt_u16 input GB/s" if workload != "flag" else "flagstats_pospopcnt")
    assert d["config"]["same_config_as_ours"] is False  # capped here; the full workload otherwise
    assert "correctness gate vs the oracle passed" in d["cpu_baseline"]["sample"]


def test_reference_arm_rank1_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    assert _run(["--steps", "1", "--warmup", "1", "--gpus", "2", "--ref-words", "65536"], env=env) == []


def test_reference_arm_does_not_self_launch():
    """--gpus 8 without torchrun: the reference arm runs once (rank 0's work) and prints one line."""
    lines = _run(["--steps", "1", "--warmup", "1", "--gpus", "8", "--ref-words", "65536"])
    assert len(lines) == 1 and lines[0]["n_gpus"] == 8
