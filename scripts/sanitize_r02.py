"""compute-sanitizer target for the kernels added in round 2: hybrid layout (dense tasks, slices,
overlapped gather + finish), tall-skinny update, cooperative block QR, speculative operator
application — small shapes, results checked against scipy / orthogonality."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S
from paper_2409_15053_b200.device import Basis

ctx = Context(0)
n, rp, ci, va = M.parsec_like(radius=12.0, n_atoms=12)
A = DeviceMatrix(ctx, n, rp, ci, va)
print(A.k1_info(3)["kernel"])
As = M.csr_to_scipy(n, rp, ci, va)
cf = S.indicator_coefficients(-0.3, 0.25, 6)
for r in (1, 2, 3, 4):
    X = np.random.default_rng(r).standard_normal((n, r))
    Y = A.filter_apply(cf, 4.0, 4.5, X)
    Z = A.spmm(X)
    assert np.abs(Z - As @ X).max() < 1e-11 * np.abs(Z).max()
    assert np.isfinite(Y).all()
for r in (1, 3, 6):
    X = np.linalg.qr(np.random.default_rng(r).standard_normal((n, r)))[0]
    B = Basis(ctx, A, X, 12 * r)
    for k in range(10):
        B.step(cf, 4.0, 4.5)
    err = B.ortho_error()
    assert err < 1e-12, err
    B.close()
print("ok")
