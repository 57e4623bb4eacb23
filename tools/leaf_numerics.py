"""GLS accuracy on hard covariances vs extended precision (tests/test_gpu_numerics.py cases),
GPU (int8 path) and CPU oracle errors per case.  python tools/leaf_numerics.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import test_gpu_numerics as T  # noqa: E402
from oracle import gls_ref as O  # noqa: E402
from paper_1304_2272_b200 import kernel  # noqa: E402

for kind, param in (("cond", 1e6), ("cond", 1e8), ("ar1", 0.99), ("ar1", 0.999)):
    rng = np.random.default_rng(7)
    n = 400
    M = T._spd_with_cond(n, param, rng) if kind == "cond" else T._ar1(n, param)
    XL = np.column_stack([np.ones(n), rng.standard_normal((n, 2))])
    y = rng.standard_normal(n)
    G = rng.integers(0, 3, (n, 24)).astype(np.float64)
    truth = T._gls_ld(M, XL, y, G)
    ctx = kernel.gls_prepare(M, XL, y)
    rb8 = kernel.gls_solve_block(ctx, kernel.SnpBlock(0, np.asfortranarray(G.astype(np.int8))))
    got = np.array([r.beta for r in rb8.results])
    octx = O.gls_prepare(M, XL, y)
    ob, _ = O.gls_solve_block(octx, G)
    print(f"{kind}={param:g}: GPU {T._rel(got, truth):.2e} "
          f"oracle {T._rel(ob, truth):.2e}", flush=True)
