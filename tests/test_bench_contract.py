"""bench.py driver contract on CPU (-m "not gpu"): the reference arm (the
oracle, as it stands) prints one JSON line with the keys the driver reads,
for the diagonal and the DIC workloads; the GPU arm's helpers name the
workloads as BASELINE.json's configs."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


@pytest.mark.parametrize("extra", [[], ["--precond", "DIC"]])
def test_reference_arm_json_line(extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "2", "--warmup", "1", *extra], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("cube10^3")
    if extra:
        assert d["config"]["precond"] == "DIC" and d["config"]["renumber"] == 2


def test_workload_names():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.workload_name(2) == "cube100^3"
    assert bench.workload_name(5) == "cube200^3-permuted"
    assert bench.workload_name(2, corrected=1) == "skewed-cube100^3-corrected-1corr"
    assert bench.workload_name(3, precond="DIC") == "cube200^3-DIC"
