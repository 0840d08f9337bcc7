"""bench.py contract pieces that run without a GPU: the reference arm (the
oracle on the host cores) prints one JSON line with the contract keys, on
the uniform cell and on the finite chain; the flops model matches SURVEY.md
§8(d)."""
import json
import math
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def run_ref(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_uniform_cell():
    d = run_ref("--config", "c1", "--steps", "2", "--warmup", "1")
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "steps/s" and d["value"] > 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["metric"] == bench.METRIC


def test_reference_arm_finite_chain():
    d = run_ref("--config", "c5small", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["scaling"] == "strong"


@pytest.mark.parametrize("cfg,expect_on,expect_off", [
    ("c1", 6.90e7, 5.65e7), ("c2", 2.36e10, 1.96e10), ("north", 1.50e12, 1.24e12)])
def test_flops_model_matches_survey(cfg, expect_on, expect_off):
    """flops per update, explicit error on / off."""
    c = bench.CONFIGS[cfg]
    _, d, chi, scheme, _, _ = c
    eta, kk = bench.widths(c)
    on = bench.flops_per_update(d, chi, eta, kk, True)
    off = bench.flops_per_update(d, chi, eta, kk, False)
    assert math.isclose(on, expect_on, rel_tol=0.01) and math.isclose(off, expect_off, rel_tol=0.01)


def test_cbe_flops_match_survey():
    c = bench.CONFIGS["c2cbe"]
    _, d, chi, _, _, _ = c
    eta, kk = bench.widths(c)
    assert eta == 356
    assert math.isclose(bench.flops_per_update(d, chi, eta, kk, True, cbe=True), 3.23e10, rel_tol=0.01)
