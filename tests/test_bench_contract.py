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
    # the reference arm names OUR arm's workload (the static config object of both arms)
    import bench

    want = bench.workload_config(0, 10000, 1, 8192, "f64")
    assert d["config"] == want and d["sample"]["snps_per_step"] > 0


def test_reference_arm_config4_form_names_the_distributed_workload():
    """--config 4 --individuals N: the reference arm prints the config-4 workload object of our
    arm (block-cyclic prepare + sharded sweep; 125,000 markers per GPU unless --snps)."""
    import bench

    d = _run(["--impl", "reference", "--config", "4", "--individuals", "600", "--snps", "2048",
              "--steps", "1", "--warmup", "3"])
    _check_base(d)
    assert d["config"] == bench.workload_config(4, 2048, 1, 8192, "f64", n=600, nb=512)
    assert "2D block-cyclic" in d["config"]["parallelism"] and d["config"]["n"] == 600
    full = bench.workload_config(4, 125_000, 8, 8192, "i8")
    assert full["n"] == 150_000 and full["m_total"] == 1_000_000 and "full m" in full["workload"]


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [1, 2])
def test_gpu_arm_config4_form(gpu, ranks):
    """bench.py --config 4 runs the distributed engine's prepare (block-cyclic M and L, fused
    Cholesky + inverse, replicated int8 slices, no dense M or FP64 inverse) and the SNP-sharded
    sweep; here at a reduced n, on one rank and on two ranks sharing the GPU over gloo."""
    env = dict(os.environ)
    if ranks > 1:
        env["GG_BENCH_BACKEND"] = "gloo"
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(ranks),
                          "--config", "4", "--individuals", "1500", "--snps", "3000",
                          "--block-snps", "1024", "--steps", "2", "--warmup", "3"],
                         cwd=REPO, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    _check_base(d)
    assert d["n_gpus"] == ranks and d["config"]["n"] == 1500
    dp = d["prepare"]["distributed"]
    assert dp["grid"] == ("1x1" if ranks == 1 else "1x2")
    assert d["parity"]["within"] and d["parity"]["status_mismatches"] == 0
    assert d["e2e"]["bitwise_equal_to_device_resident_sweep"] is True
    assert (d["cpu_baseline"] is not None) == (ranks == 1)


@pytest.mark.gpu
def test_gpu_arm_contract(gpu):
    d = _run(["--config", "0", "--steps", "3", "--warmup", "3", "--no-secondary"])
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
    import bench

    assert d["config"] == bench.workload_config(0, 10000, 1, 8192, "f64")   # = the reference arm's
    assert d["prepare"]["t_prepare_s"] > 0 and d["all_snps_ok"] in (True, False)
    # north_star's other counters: the epilogue's HBM rate and the TRSM on the FP64 pipe itself
    assert r["epilogue_hbm"]["achieved_gbs"] > 0 and r["epilogue_hbm"]["bytes_per_launch"] > 0
    assert r["fp64_dmma_path"]["tflops"] > 0 and 0 < r["fp64_dmma_path"]["frac"] < 1.05


def test_gpus_flag_starts_n_ranks():
    """`python bench.py --gpus N` without torchrun re-executes itself under
    torch.distributed.run with N ranks (here: the gloo launch probe, no GPU needed)."""
    env = dict(os.environ, GG_BENCH_LAUNCH_PROBE="1")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2"],
                         cwd=REPO, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d == {"n_gpus": 2, "ranks_seen": 2}


def test_gpus_flag_mismatch_fails_loudly():
    env = dict(os.environ, GG_BENCH_LAUNCH_PROBE="1", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4"],
                         cwd=REPO, capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stderr + out.stdout)


def test_parity_sample_covers_first_interior_and_last_partial_blocks():
    sys.path.insert(0, REPO)
    import bench

    m, blk = 2_000_000, 8192
    cols, picks = bench.sample_columns(m, blk, 512)
    nb = -(-m // blk)
    assert picks[0] == 0 and picks[-1] == nb - 1 and len(picks) == 4
    assert len(cols) == 4 * 512                         # the last block has 1,152 >= 512
    assert cols.min() == 0 and cols.max() == m - 1
    for b in picks:               # both edges of every sampled block
        f = b * blk
        c = min(blk, m - f)
        assert f in cols and f + c - 1 in cols
    small, _ = bench.sample_columns(300, 128, 512)      # blocks shorter than the sample
    assert small.max() == 299 and len(set(small.tolist())) == len(small)


def test_kinship_host_lean_matches_reference_construction():
    sys.path.insert(0, REPO)
    import numpy as np

    import bench
    from paper_1304_2272_b200 import datagen

    spec = datagen.BaselineSpec(n=300, m=10, p=4, m_kin=200, a=0.5)
    assert np.array_equal(bench.kinship_host_lean(spec), datagen.kinship_covariance_host(spec))
