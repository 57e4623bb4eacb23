"""CPU: the plugin rebinds the reference namespace (no compute; the GPU path itself is covered by
the gpu tests).  Skipped where the reference package is not importable."""

import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture()
def gwasgls():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present on this machine")
    sys.path.insert(0, REF_SRC)
    try:
        import gwasgls
        yield gwasgls
    finally:
        sys.path.remove(REF_SRC)


def test_install_and_uninstall(gwasgls):
    from gwasgls import errors as rerr
    from gwasgls import kernel as rk
    from gwasgls import pipeline as rp

    from paper_1304_2272_b200 import kernel as ok
    from paper_1304_2272_b200 import pipeline as op
    from paper_1304_2272_b200 import plugin

    before = {n: getattr(rk, n) for n in plugin.KERNEL_FUNCS}
    run_ooc = rp.run_ooc
    h = plugin.install(gwasgls, engines=True)
    try:
        for n in plugin.KERNEL_FUNCS:
            assert getattr(rk, n) is getattr(ok, n)
        assert rk.gls_oracle is not ok.gls_oracle          # the checking route stays on the CPU
        assert rp.run_ooc is op.run_ooc
        assert ok.NotPositiveDefinite is rerr.NotPositiveDefinite
        assert ok.DimensionMismatch is rerr.DimensionMismatch
        # shape validation happens before any device work and raises the reference's class
        with pytest.raises(rerr.DimensionMismatch):
            rk.cholesky_spd(__import__("numpy").ones((2, 3)))
    finally:
        h.uninstall()
    for n in plugin.KERNEL_FUNCS:
        assert getattr(rk, n) is before[n]
    assert rp.run_ooc is run_ooc
    from paper_1304_2272_b200 import errors as oerr

    assert ok.NotPositiveDefinite is oerr.NotPositiveDefinite


def test_install_rebinds_the_distributed_entry_points(gwasgls):
    from gwasgls import distgrid as rd
    from gwasgls import transport as rt

    from paper_1304_2272_b200 import distgrid as od
    from paper_1304_2272_b200 import plugin

    before = {n: getattr(rd, n) for n in plugin.DIST_FUNCS}
    spmd = rt.run_spmd
    h = plugin.install(gwasgls)
    try:
        for n in plugin.DIST_FUNCS:
            assert getattr(rd, n) is getattr(od, n)
        assert rt.run_spmd is not spmd
        # the reference's own transports still run (here: a trivial SPMD body, no device work)
        assert rt.run_spmd(3, lambda t: t.rank * 10) == [0, 10, 20]
        with pytest.raises(ValueError):
            rt.run_spmd(2, lambda t: 0, transport="bogus")
    finally:
        h.uninstall()
    for n in plugin.DIST_FUNCS:
        assert getattr(rd, n) is before[n]
    assert rt.run_spmd is spmd
