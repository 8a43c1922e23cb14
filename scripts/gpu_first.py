"""First GPU contact: parity of the device layer against the oracle + a rough filter timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2409_15053_b200 import Context, DeviceMatrix, Basis, matrices as M

ref = oracle.best()
print("oracle:", ref.kind)
ctx = Context()
rng = np.random.default_rng(0)

def check_filter(name, csr, lo, hi, alpha, beta, r, degree=0, sigma=0):
    n, rp, ci, va = csr
    Ar = ref.matrix_from_csr(n, rp, ci, va)
    cf, _, _, _ = ref.build_filter(lo, hi, alpha, beta, degree)
    X = rng.standard_normal((n, r))
    c, e = 0.5 * (lo + hi), 0.5 * (hi - lo)
    A = DeviceMatrix(ctx, n, rp, ci, va, sigma=sigma)
    ref.set_backend("scalar")
    Ys = ref.filter_apply(Ar, cf, lo, hi, X)
    ctx.set_exact(True)
    Ye = A.filter_apply(cf, c, e, X)
    ctx.set_exact(False)
    Yf = A.filter_apply(cf, c, e, X)
    scale = np.abs(Ys).max()
    print(f"{name}: n={n} r={r} m={len(cf)-1} stats={A.stats()} exact-bit-equal={np.array_equal(Ye, Ys)} "
          f"max|exact-ref|={np.abs(Ye-Ys).max():.2e} fast rel={np.abs(Yf-Ys).max()/scale:.2e}")
    Z = A.spmm(X); Zr = np.stack([ref.csr_matvec(n, rp, ci, va, X[:, j]) for j in range(r)], 1)
    print("   spmm rel", np.abs(Z - Zr).max() / np.abs(Zr).max())
    return A

lap = M.laplacian2d(30)
for r in (1, 2, 3, 4, 5):
    check_filter("lap2d30", lap, -0.02, 8.02, 3.0, 3.8, r)
rs = M.random_sparse_sym(400, 0.04, 7)
check_filter("rand400", rs, -12.0, 12.0, -1.0, 1.0, 3, degree=64)
check_filter("rand400-sig", rs, -12.0, 12.0, -1.0, 1.0, 3, degree=64, sigma=64)
pk = M.parsec_like(radius=12.0, n_atoms=12)
check_filter("parsec-small", pk, -1.5, 34.0, -0.6, 0.0, 3, degree=50)

# ---- lanczos step vs reference expand
n, rp, ci, va = lap
Ar = ref.matrix_from_csr(n, rp, ci, va)
lo, hi = ref.estimate_bounds(Ar)
cf, _, _, _ = ref.build_filter(lo, hi, 3.0, 3.8)
c, e = 0.5 * (lo + hi), 0.5 * (hi - lo)
X0 = ref.init_block(n, 3)
ref.set_backend("avx2")
F = ref.factorization(Ar, X0, 300, cf, (lo, hi), (3.0, 3.8))
F.expand(10)
Qr, Dr, Sr, deadr = F.get()
A = DeviceMatrix(ctx, n, rp, ci, va)
B = Basis(ctx, A, X0, 300)
maxd = maxs = 0
for k in range(10):
    Dk, Sk, scale, dead = B.step(cf, c, e)
    Dsym = 0.5 * (Dk + Dk.T)
    maxd = max(maxd, np.abs(Dsym - Dr[k]).max()); maxs = max(maxs, np.abs(Sk - Sr[k]).max())
Q = B.get(0, 33)
print("lanczos 10 steps: max|D-Dref|", maxd, "max|S-Sref|", maxs, "max|Q-Qref|", np.abs(Q - Qr).max(),
      "ortho", B.ortho_error(), "ref ortho", F.ortho_error(), "times", B.times())

# bounds lanczos
q0 = rng.standard_normal(n); q0 /= np.linalg.norm(q0)
dd, ee, beta = A.bounds_lanczos(q0, 50)
import scipy.linalg as sl
th = sl.eigvalsh_tridiagonal(dd, ee)
print("bounds ritz extremes", th[0], th[-1], "beta", beta)

# ---- rough timing
def bench(name, csr, r, m, sigma=0):
    n, rp, ci, va = csr
    t = time.time(); A = DeviceMatrix(ctx, n, rp, ci, va, sigma=sigma); tu = time.time() - t
    cf = ref.indicator_coefficients(-0.3, -0.25, m)
    X = rng.standard_normal((n, r))
    A.filter_bench(cf, 1.0, 2.0, X, reps=1)
    ms, _ = A.filter_bench(cf, 1.0, 2.0, X, reps=3)
    nnz = len(va)
    bytes_step = 12 * nnz + 4 * (n + 1) + 32 * n * r
    gbs = 3 * m * bytes_step / (ms * 1e-3) / 1e9
    print(f"{name}: n={n} nnz={nnz} r={r} m={m} upload {tu:.2f}s stats={A.stats()} {ms/3/m*1e3:.1f} us/step  {gbs:.0f} GB/s algorithmic")

bench("lap3d-100 r=3", M.laplacian3d(100), 3, 50)
bench("lap3d-100 r=1", M.laplacian3d(100), 1, 50)
pk = M.parsec_like()
bench("parsec r=3 sigma=auto", pk, 3, 50)
bench("parsec r=3 sigma=1", pk, 3, 50, sigma=1)
bench("lap2d-200 r=1", M.laplacian2d(200), 1, 50)
print("launches", ctx.launches)
