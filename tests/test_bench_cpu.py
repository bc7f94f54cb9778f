"""bench.py's CPU-side contract (no GPU): the reference arm's JSON line and the CPU-baseline
extrapolation (fixed cost counted once, per-view slope from two view samples)."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT


def test_extrapolation_counts_the_fixed_cost_once():
    sys.path.insert(0, str(ROOT))
    import bench

    V = bench.CONFIGS[3][1]
    # t(v) = F + v s with F = 5, s = 0.1 for A^T; A has no fixed cost
    k = 32
    t1 = (k * 0.07, 5.0 + k * 0.1)
    t2 = (2 * k * 0.07, 5.0 + 2 * k * 0.1)
    ex = bench.cpu_extrapolate(3, k, t1, t2)
    assert ex["t_A"] == pytest.approx(V * 0.07)
    assert ex["t_AT"] == pytest.approx(5.0 + V * 0.1)
    assert ex["t_AT_fixed"] == pytest.approx(5.0)
    # noise that makes the 2k sample no slower falls back to proportional scaling of the 2k sample
    ex = bench.cpu_extrapolate(3, k, (1.0, 9.0), (0.9, 8.0))
    assert ex["t_AT"] == pytest.approx(8.0 / (2 * k) * V)


def test_reference_arm_line_config1():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "CGLS iterations/sec" and line["unit"] == "it/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("config1")
