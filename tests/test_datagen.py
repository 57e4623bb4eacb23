"""CPU: the BASELINE generator reproduces the reference's counter streams bit for bit and builds
well-posed datasets."""

import numpy as np

from conftest import golden
from paper_1304_2272_b200 import datagen, fileio


def test_streams_match_reference():
    g = golden("streams")
    for seed, stream in ((42, 1), (42, 2), (7, 3), (123456789, 5)):
        idx = np.arange(1000, 1064, dtype=np.uint64)
        assert np.array_equal(datagen.stream_u64(seed, stream, idx), g[f"u64_{seed}_{stream}"])
        assert np.array_equal(datagen.stream_uniform(seed, stream, 0, 64),
                              g[f"unif_{seed}_{stream}"])


def test_genotypes_match_reference_gen_dataset():
    # same construction as the reference's gen_dataset (datagen.py:139-146): bitwise equal
    g = golden("seed42")
    G = datagen.genotypes_host(42, 100, 500, 0, 500)
    assert np.array_equal(G, g["G"])
    part = datagen.genotypes_host(42, 100, 500, 123, 77)
    assert np.array_equal(part, g["G"][:, 123:200])


def test_baseline_generator_pinned():
    g = golden("baseline_p4")
    spec = datagen.BaselineSpec(n=300, m=2000, p=4, m_kin=500, a=0.6)
    assert np.array_equal(datagen.genotypes_host(spec.seed, spec.n, spec.m, 0, spec.m), g["G"])
    XL, y = datagen.covariates_host(spec)
    assert np.array_equal(XL, g["XL"]) and np.array_equal(y, g["y"])
    M = datagen.kinship_covariance_host(spec)
    assert np.array_equal(M, M.T)
    assert np.max(np.abs(M - g["M"])) <= 1e-14 * np.max(np.abs(g["M"]))
    ev = np.linalg.eigvalsh(M)
    assert ev.min() >= 0.4 - 1e-9     # M = 0.6 K + 0.4 I with K PSD


def test_genotype_distribution():
    G = datagen.genotypes_host(5, 2000, 50, 0, 50)
    assert set(np.unique(G)) <= {0, 1, 2}
    f = datagen.marker_freqs(5, datagen.STREAM_MAF, 0, 50)
    assert np.all((f >= 0.05) & (f < 0.5))
    assert np.max(np.abs(G.mean(axis=0) - 2 * f)) < 0.1


def test_write_dataset_int8(tmp_path):
    spec = datagen.BaselineSpec(n=40, m=100, p=3, m_kin=50)
    paths = datagen.write_dataset(spec, str(tmp_path), int8=True, chunk=32)
    assert fileio.genotype_kind(paths.geno) == "GWAI"
    G = fileio.read_matrix(paths.geno, "GWAI")
    assert np.array_equal(G, datagen.genotypes_host(spec.seed, 40, 100, 0, 100))
    assert fileio.read_dims(paths.covariates, "GWAC") == (40, 2)
