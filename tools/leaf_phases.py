"""Phase timeline of the factoring leaf (clock64 at every barrier) from a GG_LEAF_PROFILE build:
    GG_ALT_FLAGS=-DGG_LEAF_PROFILE bash tools/build_alt.sh leafprof
    python tools/leaf_phases.py tools/alt/leafprof.so"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import make_spd  # noqa: E402
from paper_1304_2272_b200 import _capi  # noqa: E402

lib = C.CDLL(sys.argv[1])
for nm in ("gg_potrf_workspace_bytes", "gg_potrf_f64"):
    f = getattr(lib, nm)
    f.restype, f.argtypes = _capi.SIGNATURES[nm]
W0 = ("[diag update +] factor32", "L_JJ stored", "inverse32", "T_J stored + barrier")
NAMES = (["start", "loaded"] + [f"J{j} {p}" for j in range(3) for p in W0 + ("panel",)]
         + [f"J3 {p}" for p in W0] + ["L written + inv (a)", "inv (b)", "inv (c)", "inv (d)",
                                      "Dinv written"])
n = 128
M = torch.from_numpy(np.ascontiguousarray(make_spd(n, 3).T)).cuda()
L = torch.zeros(n, n, dtype=torch.float64, device="cuda")
Li = torch.zeros_like(L)
ws = torch.empty(int(lib.gg_potrf_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
info = (C.c_int * 2)()
for rep in range(5):
    assert lib.gg_potrf_f64(n, _capi.ptr(M), n, 0, _capi.ptr(L), _capi.ptr(Li), n, _capi.ptr(ws), info,
                            _capi.stream_handle()) == 0
    torch.cuda.synchronize()
ts = (C.c_longlong * 64)()
assert lib.gg_leaf_profile_read(ts, 64) == 0
t = np.array(ts[:len(NAMES)], dtype=np.int64)
print(f"leaf total {t[-1] - t[0]} cycles")
for i in range(1, len(NAMES)):
    print(f"{NAMES[i]:20s} {t[i] - t[i - 1]:8d} cycles")
