"""A/B timing of the fused int8 TRSM across library builds on one box (config-1 block).  Each
library cuts its own slices from the packed FP64 inverse (so slice layouts may differ); the
libraries are timed round-robin to cancel clock / power drift.
    python tools/ab_i8.py tools/alt/lib_a.so [...]   (the in-tree library is always included)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1304_2272_b200 import _capi, datagen, kernel  # noqa: E402
from paper_1304_2272_b200._capi import ptr  # noqa: E402

n, cnt = int(os.environ.get("GG_AB_N", "10000")), 8192
spec = datagen.BaselineSpec(n=n, m=cnt, p=int(os.environ.get("GG_AB_P", "4")))
ctx = kernel.gls_prepare(datagen.kinship_covariance_device(spec), *datagen.covariates_host(spec))
d = ctx._dev
n16 = -(-n // 16) * 16
G16 = datagen.genotypes_device(spec, 0, cnt, ld=n16)
P = torch.empty(int(_capi.lib().gg_partials_bytes(n, cnt, d.q)) // 8, dtype=torch.float64,
                device="cuda")
s = _capi.stream_handle()
W = _capi.i8_work()
libs = []
for path in [_capi.LIB_PATH] + sys.argv[1:]:
    lib = C.CDLL(path)
    f = lib.gg_trsm_lower_i8_partials
    f.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_int,
                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                  C.c_void_p, C.c_void_p]
    lib.gg_inverse_slices_bytes.restype = C.c_size_t
    lib.gg_inverse_slices_bytes.argtypes = [C.c_int]
    lib.gg_slice_packed_inverse_i8.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_void_p]
    sl = torch.empty(int(lib.gg_inverse_slices_bytes(n)), dtype=torch.int8, device="cuda")
    meta = torch.zeros(2 * _capi.pad(n), dtype=torch.int32, device="cuda")
    assert lib.gg_slice_packed_inverse_i8(n, ptr(d.LinvP), ptr(sl), ptr(meta), s) == 0
    libs.append((os.path.basename(path), f, sl, meta, []))
# in-tree library under environment variants: GG_AB_ENVS="GG_I8_CLUSTER=4;GG_I8_MAX_PAIRS=66"
envs = {}
for spec_ in filter(None, os.environ.get("GG_AB_ENVS", "").split(";")):
    k_, v_ = spec_.split("=", 1)
    name, f, sl, meta, _ = libs[0]
    libs.append((f"in-tree {spec_}", f, sl, meta, []))
    envs[f"in-tree {spec_}"] = (k_, v_)


class _Env:
    def __init__(self, name):
        self.kv = envs.get(name)

    def __enter__(self):
        if self.kv:
            os.environ[self.kv[0]] = self.kv[1]

    def __exit__(self, *exc):
        if self.kv:
            del os.environ[self.kv[0]]
torch.cuda.synchronize()
d.slices = None
Pref = None
for rep in range(8):
    for name, f, sl, meta, ts in libs:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with _Env(name):
            a.record()
            rc = f(n, cnt, ptr(sl), ptr(meta), ptr(G16), n16, d.q, ptr(d.XLy), ptr(d.ybar),
                   ptr(P), None, 0, None, 0, ptr(W), s)
            b.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        ts.append(a.elapsed_time(b))
        if rep == 0:
            if Pref is None:
                Pref = P.clone()
            else:   # partial dots of the candidates vs the in-tree library's
                rel = float(((P - Pref).abs().max() / Pref.abs().max()))
                print(f"{name}: max rel diff of partials vs in-tree {rel:.2e}")
for name, f, sl, meta, ts in libs:
    t = sorted(ts[1:])
    print(f"{name}: {t[0]:.3f} ms (median {t[len(t) // 2]:.3f})")
# sustained: GG_AB_SUSTAIN seconds of back-to-back launches per library (power-capped clocks),
# timing the second half
sustain = float(os.environ.get("GG_AB_SUSTAIN", "0"))
for rnd in range(2 if sustain > 0 else 0):
    for name, f, sl, meta, ts in libs:
        reps = max(int(sustain / 2.0e-3), 10)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with _Env(name):
            for r in range(reps):
                if r == reps // 2:
                    a.record()
                f(n, cnt, ptr(sl), ptr(meta), ptr(G16), n16, d.q, ptr(d.XLy), ptr(d.ybar),
                  ptr(P), None, 0, None, 0, ptr(W), s)
            b.record()
        torch.cuda.synchronize()
        print(f"sustained round {rnd} {name}: {a.elapsed_time(b) / (reps - reps // 2):.3f} ms")
