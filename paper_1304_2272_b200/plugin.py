"""Route the reference package's hot path through the B200 library (the drop-in binding).

    import gwasgls
    from paper_1304_2272_b200 import plugin
    handle = plugin.install(gwasgls)      # gwasgls.kernel.* now run on the GPU
    ...
    handle.uninstall()

The reference resolves every numerical call through module attributes at call time
(pipeline.py:130,155,214; distgrid.py:21,261-435; kernel.py:245-256,325-328 — SURVEY.md §8b), so
rebinding those attributes re-targets every caller, including ``run_incore``/``run_ooc``/
``run_dist`` and the reference's own tests.  The exception classes are unified first: our modules
raise the reference's classes, so ``except gwasgls.errors.NotPositiveDefinite`` keeps working.
``gls_oracle`` (the reference's checking route) is deliberately left on the CPU.
"""

from __future__ import annotations

import importlib
import importlib.util
import sys

KERNEL_FUNCS = ("cholesky_spd", "trsolve_lower", "gram", "cholesky_solve_batch",
                "solve_small_spd", "gls_prepare", "solve_whitened_block", "gls_solve_block")
ENGINE_FUNCS = ("run_incore", "run_ooc")
DIST_FUNCS = ("run_dist", "dist_cholesky", "dist_trsolve")
OUR_MODULES = ("errors", "kernel", "fileio", "pipeline", "shard", "_capi", "_device", "distgrid",
               "comm", "transport")


class Handle:
    def __init__(self):
        self._saved = []

    def set(self, obj, name, value):
        self._saved.append((obj, name, getattr(obj, name, None)))
        setattr(obj, name, value)

    def uninstall(self):
        for obj, name, old in reversed(self._saved):
            setattr(obj, name, old)
        self._saved.clear()


def _spmd_with_nccl(orig, ours):
    """The reference's run_spmd (transport.py:267-327) plus transport="nccl": one process per
    GPU over torch.distributed (paper_1304_2272_b200.transport); other transports unchanged."""

    def run_spmd(size, fn, *args, transport="inproc"):
        if transport == "nccl":
            return ours.run_spmd(size, fn, *args, transport="nccl")
        return orig(size, fn, *args, transport=transport)

    run_spmd.__doc__ = orig.__doc__
    return run_spmd


def install(ref=None, engines=False, dist=True):
    """Install into the reference package ``ref`` (default: ``import gwasgls``).

    engines=True also replaces ``pipeline.run_incore``/``run_ooc`` with the GPU stream engines
    (pinned double buffers + copy stream); by default the reference's own drivers run and call the
    GPU kernels block by block.  dist=True (default) replaces ``distgrid.run_dist`` /
    ``dist_cholesky`` / ``dist_trsolve`` with the B200 distributed engine (same signatures: the
    reference's transports and element-cyclic DistMatrix2D in, results out) and adds
    transport="nccl" to ``transport.run_spmd``."""
    if ref is None:
        ref = importlib.import_module("gwasgls")
    rk = importlib.import_module(ref.__name__ + ".kernel")
    rerr = importlib.import_module(ref.__name__ + ".errors")
    h = Handle()
    ours = {m: importlib.import_module(f"{__package__}.{m}") for m in OUR_MODULES}
    # 1. one exception hierarchy: ours raise the reference's classes
    for name in dir(rerr):
        cls = getattr(rerr, name)
        if isinstance(cls, type) and issubclass(cls, Exception):
            for mod in ours.values():
                if hasattr(mod, name):
                    h.set(mod, name, cls)
    # 2. numerical core
    k = ours["kernel"]
    for name in KERNEL_FUNCS:
        h.set(rk, name, getattr(k, name))
    # 3. optionally the engines
    if engines:
        rp = importlib.import_module(ref.__name__ + ".pipeline")
        for name in ENGINE_FUNCS:
            h.set(rp, name, getattr(ours["pipeline"], name))
    # 4. the distributed entry points and the NCCL launcher
    if dist:
        rd = importlib.import_module(ref.__name__ + ".distgrid")
        for name in DIST_FUNCS:
            h.set(rd, name, getattr(ours["distgrid"], name))
        rt = importlib.import_module(ref.__name__ + ".transport")
        h.set(rt, "run_spmd", _spmd_with_nccl(rt.run_spmd, ours["transport"]))
    return h


def pytest_configure(config):   # pragma: no cover - used as `pytest -p paper_1304_2272_b200.plugin`
    """pytest plugin hook: install before the reference's tests are collected."""
    if "gwasgls" in sys.modules or importlib.util.find_spec("gwasgls") is not None:
        config._gwasgls_b200 = install()
