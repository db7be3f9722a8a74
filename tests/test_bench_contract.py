"""bench.py's reference arm on CPU: the JSON line the driver reads (keys, units,
impl tag), and the N>1 convention that only rank 0 runs and prints."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from oracle.oracle import Ref  # noqa: E402


def run_bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=e, cwd=ROOT)


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = run_bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "TOPS" and line["value"] > 0
    assert line["warmup"] >= 3 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_reference_arm_other_ranks_are_silent():
    r = run_bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1", env={"RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""
