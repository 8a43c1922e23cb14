"""ncu target: a few fused Clenshaw steps on one bench matrix (c2 | c3 | c4), r columns."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
r = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = int(sys.argv[3]) if len(sys.argv) > 3 else 12
csr = {"c2": lambda: M.laplacian3d(100), "c3": lambda: M.parsec_like(ball_radius=3.384),
       "c4": lambda: M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2)}[name]()
n, rp, ci, va = csr
ctx = Context()
A = DeviceMatrix(ctx, n, rp, ci, va)
cf = S.indicator_coefficients(-0.3, -0.25, m)
X = np.random.default_rng(0).standard_normal((n, r))
ms, _ = A.filter_bench(cf, 1.0, 2.0, X, reps=2)
print(name, A.stats(), f"{ms / 2 / m * 1e3:.1f} us/step")
