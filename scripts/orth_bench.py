"""Orthogonalization cost of the block Lanczos step (K3/K4 + intra-block QR) on bench-like
shapes: python scripts/orth_bench.py [c1|c3|c2] — plain A q steps (cheap operator), basis grown
to the bench's final size; prints the device time of the orthogonalization part, the basis
bytes CGS2 streams (4 sweeps of the basis per block step) and the rate."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M
from paper_2409_15053_b200.device import Basis

shapes = {"c1": (lambda: M.laplacian2d(200), 1, 1740), "c3": (lambda: M.laplacian3d(48), 3, 630),
          "c2": (lambda: M.laplacian3d(100), 3, 210), "c4": (lambda: M.laplacian3d(64), 3, 540)}
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
gen, r, cols = shapes[name]
n, rp, ci, va = gen()
ctx = Context()
A = DeviceMatrix(ctx, n, rp, ci, va)
for rep in range(2):
    X = np.linalg.qr(np.random.default_rng(rep).standard_normal((n, r)))[0]
    B = Basis(ctx, A, X, cols)
    t0 = time.perf_counter()
    steps = cols // r - 1
    for k in range(steps):
        B.step()
    wall = time.perf_counter() - t0
    mv, orth = B.times()
    err = B.ortho_error()
    B.close()
nbytes = sum(4 * (k + 1) * r * n * 8 for k in range(steps))
print(f"{name}: n={n} r={r} cols={cols} steps={steps} orth {orth*1e3:.1f} ms ({orth/steps*1e6:.1f} us/step) "
      f"mv {mv*1e3:.1f} ms wall {wall*1e3:.1f} ms  basis stream {nbytes/1e9:.2f} GB -> {nbytes/orth/1e12:.2f} TB/s  "
      f"ortho_error {err:.2e} launches {ctx.launches}")
