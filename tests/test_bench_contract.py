"""bench.py keeps the driver's JSON contract: one line with the metric, value, timing fields, the
roofline / cpu_baseline / e2e objects, gpu_launches and clocks (GPU arm), and the reference
arm's line.  Runs the small config 0 (n = 1,000) so the check takes seconds."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, cwd=REPO,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _check_base(d):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["metric"].startswith("GLS solves (SNPs/sec)") and d["unit"] == "SNPs/s"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["dtype"] == "f64" and "workload" in d["config"]
    assert d["warmup"] >= 3


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "0", "--steps", "1", "--warmup", "3"])
    _check_base(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["h2d_bytes_per_step"] == 0
    assert e2e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_contract(gpu):
    d = _run(["--config", "0", "--steps", "3", "--warmup", "3"])
    _check_base(d)
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3 and "traffic" in r
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["parity"]["within"] and d["parity"]["status_mismatches"] == 0
