"""The bench.py contract on CPU: the reference arm (the oracle, BASELINE's metric and workload) prints ONE
JSON line with the keys the driver reads; the GPU arm's keys are checked in the GPU runs (profiles/)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(300)
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=280)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "DOF*it/s"
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2")


def test_committed_gpu_bench_lines_carry_the_contract_keys():
    """The committed round's GPU bench lines (profiles/bench_r02_C*.json) carry roofline, cpu_baseline, e2e,
    clocks and gpu_launches, with the roofline fraction consistent with achieved / peak."""
    for c in ("C1", "C2", "C3", "C4", "C5"):
        with open(os.path.join(ROOT, "profiles", f"bench_r02_{c}.json")) as f:
            d = json.loads(f.read().strip().splitlines()[-1])
        for k in ("roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches", "config"):
            assert k in d, (c, k)
        r = d["roofline"]
        assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 * max(1.0, r["frac"])
        assert d["gpu_launches"] > 0 and d["clocks"]["reasons"] == []
        assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
