"""bench.py contract pieces that run without a GPU: the reference arm (the
fp64 oracle, timed on the host) prints one JSON line with the base
contract's keys, and the cpu_baseline sampler covers all six benchmarks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--bench", "vec"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is False
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("name", ["vec", "bs", "img", "ml", "hits", "dl"])
def test_cpu_baseline_all_benchmarks(name):
    sys.path.insert(0, ROOT)
    import bench
    v, sample, cores = bench.cpu_oracle_rate(name, budget_s=0.05)
    assert v is not None and v > 0 and cores == 1 and sample
