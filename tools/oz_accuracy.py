"""Ozaki GEMM accuracy against an 80-bit (long double) product, per library build, next to the
FP64 GEMM's own error: max |C - C_exact| / (|A(i,:)|max |B(j,:)|max sqrt(k)) and the RMS of the same
ratio.  python tools/oz_accuracy.py --libs tools/alt/oz7.so tools/alt/oz8.so"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1304_2272_b200 import _capi  # noqa: E402
from paper_1304_2272_b200._capi import ptr, stream_handle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--libs", nargs="+", required=True)
args = ap.parse_args()
dev = _capi.device()


def cases():
    rng = np.random.default_rng(11)
    m, nc, k = 512, 384, 1024
    A = rng.standard_normal((m, k))
    B = rng.standard_normal((nc, k))
    yield "normal", A, B
    yield "row-scaled 2^+-20", A * np.ldexp(1.0, rng.integers(-20, 20, (m, 1))), \
        B * np.ldexp(1.0, rng.integers(-20, 20, (nc, 1)))
    yield "uniform [0,1)", rng.random((m, k)), rng.random((nc, k))
    # a Cholesky panel of a kinship-like covariance (what the SYRK multiplies)
    Z = rng.integers(0, 3, (m + nc, 3000)).astype(np.float64)
    Z = (Z - Z.mean(axis=0)) / (Z.std(axis=0) + 1e-12)
    M = 0.6 * (Z @ Z.T) / 3000 + 0.4 * np.eye(m + nc)
    L = np.linalg.cholesky(M)
    P = np.ascontiguousarray(L[:, : min(k, m + nc)])
    yield "kinship panel", P[:m, :], P[m:m + nc, :]
    yield "heavy-tailed", rng.standard_cauchy((m, k)), rng.standard_cauchy((nc, k))


def run(lib, A, B):
    m, k = A.shape
    nc = B.shape[0]
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).to(dev)
    Cd = torch.zeros((nc, m), dtype=torch.float64, device=dev)
    wsb = int(lib.gg_gemm_ozaki_workspace_bytes(m, nc, k, 0))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    rc = lib.gg_gemm_ozaki_f64(m, nc, k, ptr(Ad), 1, m, ptr(Bd), 1, nc, ptr(Cd), m, 1.0, 0.0, 0,
                               ptr(ws), wsb, stream_handle())
    assert rc == 0, rc
    return Cd.cpu().numpy().T


libs = []
for path in args.libs:
    h = C.CDLL(os.path.abspath(path))
    for name, (res, argt) in _capi.SIGNATURES.items():
        if name.startswith("gg_gemm_ozaki"):
            f = getattr(h, name)
            f.restype, f.argtypes = res, argt
    libs.append((os.path.basename(path), h))

for name, A, B in cases():
    k = A.shape[1]
    exact = A.astype(np.longdouble) @ B.astype(np.longdouble).T
    scale = np.outer(np.abs(A).max(axis=1), np.abs(B).max(axis=1)) * np.sqrt(k)
    f64 = A @ B.T
    e64 = np.abs(f64 - exact).astype(np.float64) / scale
    line = f"{name:20s} FP64 GEMM max {e64.max():.2e} rms {np.sqrt((e64 ** 2).mean()):.2e}"
    for lname, h in libs:
        e = np.abs(run(h, A, B) - exact).astype(np.float64) / scale
        line += f" | {lname} max {e.max():.2e} rms {np.sqrt((e ** 2).mean()):.2e}"
    print(line, flush=True)
