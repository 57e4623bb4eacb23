"""Ozaki GEMM (gg_gemm_ozaki_f64) on the prepare's shapes at n = 4e4, device-resident operands,
CUDA-event timing (slicing + GEMM launches per call).  Effective rate = 28 int8 MACs per useful
FP64 MAC (triangular shapes count only their nonzero products) x 2 ops.
    python tools/prof_ozaki.py [--only NAME] [--reps R] [--libs tools/alt/a.so ...]
(--libs: time the same shapes through other builds of the library, round-robin per shape)"""
import ctypes as C
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1304_2272_b200 import _capi  # noqa: E402
from paper_1304_2272_b200._capi import check, ptr, stream_handle  # noqa: E402

# name: (m, ncols, k, flags, same, useful MACs)
SHAPES = {
    "syrk_first": (38912, 38912, 1024, 4, True, 38912 * 38913 / 2 * 1024),
    "syrk_mid": (19968, 19968, 1024, 4, True, 19968 * 19969 / 2 * 1024),
    "trtri_top_T": (20032, 20032, 20032, 2, False, 20032 ** 3 / 2),      # B lower
    "trtri_top_X": (20032, 20032, 20032, 1, False, 20032 ** 3 / 2),      # A lower
    "square_8k": (8192, 8192, 8192, 0, False, 8192 ** 3),
}
ap = argparse.ArgumentParser()
ap.add_argument("--only", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--libs", nargs="*", default=[])
args = ap.parse_args()
dev = _capi.device()
libs = [("in-tree", _capi.lib())]
for path in args.libs:
    cl = C.CDLL(path)
    for nm in ("gg_gemm_ozaki_workspace_bytes", "gg_gemm_ozaki_f64"):
        f = getattr(cl, nm)
        f.restype, f.argtypes = _capi.SIGNATURES[nm]
    libs.append((os.path.basename(path), cl))
g = torch.Generator(device=dev).manual_seed(1)
for name, (m, nc, k, flags, same, macs) in SHAPES.items():
    if args.only and name not in args.only.split(","):
        continue
    A = torch.randn(k, m, device=dev, dtype=torch.float64, generator=g)   # column-major m x k
    B = None if same else torch.randn(k, nc, device=dev, dtype=torch.float64, generator=g)
    C = torch.randn(nc, m, device=dev, dtype=torch.float64, generator=g)
    C0 = C.clone()
    ref = None
    for lname, lib in libs:
        wsb = int(lib.gg_gemm_ozaki_workspace_bytes(m, nc, k, int(same)))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        times = []
        for r in range(args.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = lib.gg_gemm_ozaki_f64(m, nc, k, ptr(A), 1, m, None if same else ptr(B), 1, nc,
                                       ptr(C), m, -1.0, 1.0, flags, ptr(ws), wsb, stream_handle())
            check(rc, "gg_gemm_ozaki_f64")
            e1.record()
            torch.cuda.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        t = min(times) / 1e3
        # correctness across builds: one more call from the same C0
        C.copy_(C0)
        lib.gg_gemm_ozaki_f64(m, nc, k, ptr(A), 1, m, None if same else ptr(B), 1, nc, ptr(C), m,
                              -1.0, 1.0, flags, ptr(ws), wsb, stream_handle())
        torch.cuda.synchronize()
        if ref is None:
            ref = C.clone()
        diff = float((C - ref).abs().max() / ref.abs().max())
        print(f"{lname:10s} diff={diff:.1e} {name:12s} m={m} n={nc} k={k} flags={flags}: {t * 1e3:8.2f} ms  "
              f"{28 * 2 * macs / t / 1e12:7.0f} int8 TOPS eff  ({2 * macs / t / 1e12:5.1f} FP64 TF/s)",
              flush=True)
        del ws
    del A, B, C, C0, ref
    torch.cuda.empty_cache()
