"""Shared fixtures.  Markers: ``gpu`` = needs a B200 (run with ``-m gpu``); everything else runs
on CPU.  Golden fixtures come from the reference implementation (tests/golden/make_golden.py)."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def make_spd(n, seed):
    """Well-conditioned SPD test matrix G G^T / (2n) + I with exact stored symmetry
    (the construction of the reference's tests/conftest.py:10-14)."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, 2 * n))
    M = G @ G.T / (2 * n) + np.eye(n)
    return np.tril(M) + np.tril(M, -1).T


def maxnorm(A):
    return float(np.max(np.abs(A)))


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: GPU tests must fail loudly (not skip) when the device path is broken."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test run without a CUDA device"
    from paper_1304_2272_b200 import _capi

    _capi.lib()
    return torch.device("cuda", 0)


def write_golden_dataset(tmp_path, g, int8=False, name="ds"):
    """Write a golden case as GWA* files; returns SolvePaths-like paths."""
    from paper_1304_2272_b200 import fileio
    from paper_1304_2272_b200.pipeline import SolvePaths

    d = tmp_path / name
    d.mkdir(exist_ok=True)
    fileio.write_matrix(str(d / "cov.gwam"), "GWAM", g["M"])
    fileio.write_matrix(str(d / "cov.gwac"), "GWAC", g["XL"])
    fileio.write_matrix(str(d / "phe.gway"), "GWAY", g["y"])
    if int8:
        geno = str(d / "geno.gwai")
        fileio.write_matrix(geno, "GWAI", g["G"].astype(np.int8))
    else:
        geno = str(d / "geno.gwax")
        fileio.write_matrix(geno, "GWAX", g["G"].astype(np.float64))
    return SolvePaths(cov=str(d / "cov.gwam"), covariates=str(d / "cov.gwac"),
                      pheno=str(d / "phe.gway"), geno=geno, out=str(d / "out.gwab"))
