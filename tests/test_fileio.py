"""CPU: GWA* formats and the asynchronous block agents (reference tests/test_fileio.py behaviour)."""

import struct

import numpy as np
import pytest

from paper_1304_2272_b200 import fileio, kernel
from paper_1304_2272_b200.errors import (
    AsymmetricCovariance,
    BadMagic,
    OverlappingBuffer,
    TruncatedFile,
    UnsupportedVersion,
)


def test_header_bytes(tmp_path):
    p = str(tmp_path / "a.gwax")
    fileio.write_matrix(p, "GWAX", np.zeros((3, 2)))
    raw = open(p, "rb").read()
    assert raw[:4] == b"GWAX"
    assert struct.unpack("<I", raw[4:8])[0] == 1
    assert struct.unpack("<2Q", raw[8:24]) == (3, 2)
    assert len(raw) == 24 + 8 * 6


@pytest.mark.parametrize("kind,shape", [("GWAM", (5, 5)), ("GWAX", (7, 3)), ("GWAC", (7, 2)),
                                        ("GWAY", (7,)), ("GWAI", (9, 4))])
def test_round_trip_bitwise(tmp_path, kind, shape):
    rng = np.random.default_rng(1)
    if kind == "GWAI":
        a = rng.integers(0, 3, shape).astype(np.int8)
    elif kind == "GWAM":
        a = rng.standard_normal(shape)
        a = a + a.T
    else:
        a = rng.standard_normal(shape)
    p = str(tmp_path / ("f." + kind.lower()))
    fileio.write_matrix(p, kind, a)
    b = fileio.read_matrix(p, kind)
    assert b.dtype == a.dtype and np.array_equal(a, b)


def test_results_round_trip(tmp_path):
    betas = np.arange(12.0).reshape(4, 3)
    betas[2] = np.nan
    sinv = np.arange(24.0).reshape(4, 6)
    p = str(tmp_path / "r.gwab")
    fileio.write_matrix(p, "GWAB", fileio.ResultPayload(betas=betas, sinv=sinv))
    back = fileio.read_matrix(p, "GWAB")
    assert np.array_equal(back.betas, betas, equal_nan=True)
    assert np.array_equal(back.sinv, sinv)
    assert list(back.statuses) == ["ok", "ok", "degenerate", "ok"]


def test_errors(tmp_path):
    p = str(tmp_path / "x.gwax")
    fileio.write_matrix(p, "GWAX", np.ones((4, 4)))
    with pytest.raises(BadMagic):
        fileio.read_matrix(p, "GWAM")
    raw = bytearray(open(p, "rb").read())
    open(p, "wb").write(bytes(raw[:-8]))
    with pytest.raises(TruncatedFile):
        fileio.read_matrix(p, "GWAX")
    raw[4] = 2
    open(p, "wb").write(bytes(raw))
    with pytest.raises(UnsupportedVersion):
        fileio.read_matrix(p, "GWAX")
    q = str(tmp_path / "m.gwam")
    A = np.eye(3)
    A[0, 1] = 1e-300
    fileio.write_matrix(q, "GWAM", A)
    with pytest.raises(AsymmetricCovariance):
        fileio.read_matrix(q, "GWAM")


def test_block_reader_and_overlap(tmp_path):
    rng = np.random.default_rng(2)
    X = rng.integers(0, 3, (11, 30)).astype(np.int8)
    p = str(tmp_path / "g.gwai")
    fileio.write_matrix(p, "GWAI", X)
    r = fileio.BlockReader(p)
    assert (r.n, r.m, r.kind) == (11, 30, "GWAI")
    buf = np.zeros((11, 8), dtype=np.int8, order="F")
    t = r.start(5, 8, buf)
    with pytest.raises(OverlappingBuffer):
        r.start(0, 8, buf)
    blk = r.wait(t)
    assert blk.first_index == 5 and np.array_equal(blk.data, X[:, 5:13])
    t = r.start(24, 6, buf)
    assert np.array_equal(r.wait(t).data, X[:, 24:30])
    r.close()
    assert fileio.total_genotype_bytes(p) == (11 * 30, 11, 30)


def test_writer_out_of_order_and_array_encode(tmp_path):
    p = str(tmp_path / "o.gwab")
    m, pp = 10, 3
    w = fileio.BlockWriter(p, m, pp, 1)
    beta = np.arange(30.0).reshape(10, 3)
    status = np.full(10, -1, dtype=np.int32)
    status[4] = 1
    sinv = np.arange(60.0).reshape(10, 6)
    arrays = kernel.ResultArrays(first_index=5, beta=beta[5:], status=status[5:], sinv=sinv[5:])
    w.wait(w.start(kernel.ResultBlock.from_arrays(arrays)))
    arrays0 = kernel.ResultArrays(first_index=0, beta=beta[:5], status=status[:5], sinv=sinv[:5])
    rb = kernel.ResultBlock.from_arrays(arrays0)
    # the per-SNP path and the array path encode identically
    rb_list = kernel.ResultBlock(first_index=0, results=list(rb.results))
    assert np.array_equal(w.encode(rb), w.encode(rb_list), equal_nan=True)
    w.wait(w.start(rb))
    w.close()
    back = fileio.read_matrix(p, "GWAB")
    expect = beta.copy()
    expect[4] = np.nan
    assert np.array_equal(back.betas, expect, equal_nan=True)
    assert np.all(np.isnan(back.sinv[4])) and np.array_equal(back.sinv[5:], sinv[5:])
    assert w.bytes_written == m * fileio.record_size(pp, 1)


def test_lazy_results_view():
    arrays = kernel.ResultArrays(first_index=100, beta=np.ones((3, 2)),
                                 status=np.array([-1, 0, -1], dtype=np.int32), sinv=None)
    rb = kernel.ResultBlock.from_arrays(arrays)
    assert len(rb.results) == 3
    assert [r.snp_index for r in rb.results] == [100, 101, 102]
    assert rb.results[1].status == "degenerate" and np.all(np.isnan(rb.results[1].beta))
    assert rb.results[-1].status == "ok" and rb.results[-1].s_inv is None
