"""K1 (fused Clenshaw-step SpMM) timing + fast-vs-exact agreement on the bench shapes."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S

ctx = Context()
rng = np.random.default_rng(0)
PEAK = 6533.2

def bench(name, csr, r, m=50, sigma=0, check=True):
    n, rp, ci, va = csr
    A = DeviceMatrix(ctx, n, rp, ci, va, sigma=sigma)
    cf = S.indicator_coefficients(-0.3, -0.25, m)
    X = rng.standard_normal((n, r))
    if check:
        ctx.set_exact(True); _, Ye = A.filter_bench(cf, 1.0, 2.0, X, reps=1, want_output=True)
        ctx.set_exact(False); _, Yf = A.filter_bench(cf, 1.0, 2.0, X, reps=1, want_output=True)
        err = np.abs(Yf - Ye).max() / np.abs(Ye).max()
    else:
        err = float('nan')
    A.filter_bench(cf, 1.0, 2.0, X, reps=1)
    ms, _ = A.filter_bench(cf, 1.0, 2.0, X, reps=4)
    nnz = len(va)
    bytes_step = 12 * nnz + 4 * (n + 1) + 32 * n * r
    gbs = 4 * m * bytes_step / (ms * 1e-3) / 1e9
    st = A.stats()
    stride = 4 if (r == 3 and nnz >= 16 * n) else r
    if os.environ.get("FLZ_K1_LAYOUT", "")[:1] == "p" or (not os.environ.get("FLZ_K1_LAYOUT") and r == 3 and nnz < 16 * n):
        stride = r
    if os.environ.get("FLZ_K1_LAYOUT", "")[:1] == "4" and r == 3:
        stride = 4
    moved = st["matrix_bytes"] + 8 * n * (3 * stride + r)
    print(f"{name:28s} n={n:8d} nnz/row={nnz/n:5.1f} r={r} fill={st['fill']:.3f} sigma={st['sigma']:6d} "
          f"uniform={st['uniform_entries']/nnz:5.1%} moved/formula={moved/bytes_step:.3f} "
          f"{ms/4/m*1e3:7.1f} us/step {gbs:7.0f} GB/s ({100*gbs/PEAK:5.1f}% of measured peak; moved bytes "
          f"{4*m*moved/(ms*1e-3)/1e9:6.0f} GB/s) fast-vs-exact {err:.1e}", flush=True)
    return ms / 4 / m * 1e3

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which == "stencil":
    st = M.stencil3d(48, potential=(-1.2, 0.3))
    for r in (3, 1):
        bench("stencil37-48^3 r=%d" % r, st, r)
    sys.exit(0)
if which == "parsec":   # long ragged rows only (C3 with the Ge99H100 nonzero count, C3 old, C4)
    bench("parsec-c3 8.44M r=3", M.parsec_like(ball_radius=3.384), 3, check=False)
    bench("parsec-c3 7.41M r=3", M.parsec_like(), 3, check=False)
    bench("parsec-c4 r=3", M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2), 3, m=20, check=False)
    sys.exit(0)
if which == "lap":
    bench("lap3d-100 r=3", M.laplacian3d(100), 3, check=False)
    bench("lap3d-100 r=1", M.laplacian3d(100), 1, check=False)
    sys.exit(0)
if which == "sweep":
    lap = M.laplacian3d(100)
    pk = M.parsec_like()
    for batch in (4, 8):
        for spc in (4, 16, 64):
            ctx.set_tuning(spc, 0, batch)
            print("batch", batch, "slices_per_cta", spc, end=": ")
            bench("lap3d-100 r=3", lap, 3, check=False)
    ctx.set_tuning(0, 0)
    for tpc in (1, 2, 4, 8):
        ctx.set_tuning(0, tpc)
        print("tasks_per_cta", tpc, end=": ")
        bench("parsec r=3", pk, 3, check=False)
    sys.exit(0)
lap = M.laplacian3d(100)
bench("lap3d-100 r=3", lap, 3)
bench("lap3d-100 r=1", lap, 1)
bench("lap3d-100 r=4", lap, 4)
pk = M.parsec_like()
bench("parsec r=3", pk, 3)
bench("parsec r=1", pk, 1)
bench("lap2d-200 r=1", M.laplacian2d(200), 1)
if which == "all":
    bench("lap3d-160 r=3", M.laplacian3d(160), 3, m=20, check=False)
    bench("parsec-c4 r=3", M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2), 3, m=20, check=False)
