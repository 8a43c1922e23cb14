"""compute-sanitizer target: the TMA-staged stencil kernel on small Laplacians (boundary tiles
with clipped runs, flagged slices, all column counts), checked against scipy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S

ctx = Context(0)
for gen in (lambda: M.laplacian3d(24), lambda: M.laplacian2d(61)):
    n, rp, ci, va = gen()
    A = DeviceMatrix(ctx, n, rp, ci, va)
    As = M.csr_to_scipy(n, rp, ci, va)
    cf = S.indicator_coefficients(-0.3, 0.25, 6)
    for r in (1, 2, 3, 4):
        X = np.random.default_rng(r).standard_normal((n, r))
        Y = A.filter_apply(cf, 4.0, 4.5, X)
        Z = A.spmm(X)
        assert np.abs(Z - As @ X).max() < 1e-12
        assert np.isfinite(Y).all()
print("ok")
