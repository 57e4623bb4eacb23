import numpy as np, time, sys
sys.path.insert(0, "/root/repo")
from paper_1304_2272_b200 import kernel as K
import scipy.linalg as sl
rng = np.random.default_rng(0)
for n in (5, 50, 130, 300, 1000):
    G = rng.standard_normal((n, 2*n)); M = G @ G.T/(2*n) + np.eye(n); M = np.tril(M)+np.tril(M,-1).T
    L = K.cholesky_spd(M)
    Lr = sl.cholesky(M, lower=True)
    print(n, "chol err", np.max(np.abs(L-Lr))/np.max(np.abs(Lr)), "upper0", np.all(np.triu(L,1)==0))
    B = rng.standard_normal((n, 37))
    X = K.trsolve_lower(L, B)
    Xr = sl.solve_triangular(Lr, B, lower=True)
    print(n, "trsm err", np.max(np.abs(X-Xr))/np.max(np.abs(Xr)))
    XL = np.hstack([np.ones((n,1)), rng.standard_normal((n,2))]); y = rng.standard_normal(n)
    ctx = K.gls_prepare(M, XL, y)
    Xs = rng.integers(0,3,(n,20)).astype(float) if n > 8 else rng.standard_normal((n,20))
    rb = K.gls_solve_block(ctx, K.SnpBlock(0, Xs))
    worst=0
    for i in range(20):
        e = np.linalg.solve(*(lambda Xi: (Xi.T@np.linalg.solve(M,Xi), Xi.T@np.linalg.solve(M,y)))(np.hstack([XL, Xs[:,i:i+1]])))
        worst=max(worst, np.max(np.abs(rb.results[i].beta-e))/np.max(np.abs(e)))
    print(n, "beta err", worst, rb.results[0].status)
