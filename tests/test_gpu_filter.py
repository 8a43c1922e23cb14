"""GPU parity of the filter / SpMM kernels (K1, K2, K7, K11) through the C ABI.

Bar: exact mode is BIT-IDENTICAL to the reference's scalar backend (kernels.cpp:25-41 order
of operations); fast mode (FMA contraction) agrees to 1e-13 relative, the tolerance the
reference itself uses between its scalar and AVX2 backends (kernels_test.cpp:60-92).
"""
import numpy as np
import pytest

from paper_2409_15053_b200 import DeviceMatrix, FlzError, matrices as M, solver as S
from paper_2409_15053_b200 import lib

pytestmark = pytest.mark.gpu


def block(n, r, seed):
    return np.random.default_rng(seed).standard_normal((n, r))


CASES = {
    "lap2d30": lambda: M.laplacian2d(30),
    "rand400": lambda: M.random_sparse_sym(400, 0.04, 7),
    "parsec7k": lambda: M.parsec_like(radius=12.0, n_atoms=12),
    "lap3d12": lambda: M.laplacian3d(12),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("sigma", [0, 1, 64])
def test_filter_vs_golden(ctx, golden, name, sigma):
    n, rp, ci, va = CASES[name]()
    lo, hi, a, b, r, seed = golden[f"filter_{name}_meta"]
    cf = golden[f"filter_{name}_coeffs"]
    X = block(n, int(r), int(seed))
    A = DeviceMatrix(ctx, n, rp, ci, va, sigma=sigma)
    c, e = 0.5 * (lo + hi), 0.5 * (hi - lo)
    ctx.set_exact(True)
    try:
        Ye = A.filter_apply(cf, c, e, X)
    finally:
        ctx.set_exact(False)
    assert np.array_equal(Ye, golden[f"filter_{name}_scalar"])       # bit-exact
    Yf = A.filter_apply(cf, c, e, X)
    scale = np.abs(Ye).max()
    assert np.abs(Yf - golden[f"filter_{name}_scalar"]).max() <= 1e-13 * scale
    assert np.abs(Yf - golden[f"filter_{name}_avx2"]).max() <= 1e-13 * scale


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 7, 9])
def test_filter_vs_oracle_all_block_sizes(ctx, best_oracle, r):
    n, rp, ci, va = M.random_sparse_sym(333, 0.05, 21)     # n not a multiple of 32
    Ao = best_oracle.matrix_from_csr(n, rp, ci, va)
    cf, _, _, _ = best_oracle.build_filter(-12.0, 12.0, -2.0, 1.0, 40)
    X = block(n, r, 100 + r)
    Y = DeviceMatrix(ctx, n, rp, ci, va).filter_apply(cf, 0.0, 12.0, X)
    Yo = best_oracle.filter_apply(Ao, cf, -12.0, 12.0, X)
    assert np.abs(Y - Yo).max() <= 1e-13 * np.abs(Yo).max()


def test_filter_degree_edge_cases_and_counter(ctx, best_oracle):
    # filter_test.cpp:206-234: constant filter -> copy with 0 matvecs; m products otherwise
    n, rp, ci, va = M.diag_matrix([1, 2, 3, 4, 5])
    A = DeviceMatrix(ctx, n, rp, ci, va)
    X = np.ones((5, 5))
    before = lib().flz_matvec_count()
    Y0 = A.filter_apply([0.75], 3.0, 2.5, X)
    assert lib().flz_matvec_count() == before and np.array_equal(Y0, 0.75 * X)
    cf, _, _, _ = best_oracle.build_filter(0.5, 5.5, 1.5, 3.5, 48)
    Y = A.filter_apply(cf, 3.0, 2.5, X)
    assert lib().flz_matvec_count() - before == 5 * 48          # counter += r*m = 240
    for i in range(5):
        assert np.allclose(Y[i], best_oracle.clenshaw(cf, ((i + 1) - 3.0) / 2.5), atol=1e-12)
    Y1 = A.filter_apply([0.25, 0.5], 3.0, 2.5, X)               # m = 1: single (final) step
    want = 0.25 + 0.5 * (np.arange(1, 6) - 3.0) / 2.5
    assert np.allclose(Y1, want[:, None], atol=1e-15)


def test_filter_vs_dense_spectral_transform(ctx, best_oracle):
    # acceptance criterion 7 / filter_test.cpp:236-266: p(A) X == V p(L) V^T X to 1e-10
    n, rp, ci, va = M.random_sparse_sym(30, 0.35, 424242)
    Ad = M.csr_to_scipy(n, rp, ci, va).toarray()
    lam, V = np.linalg.eigh(Ad)
    lo, hi = lam[0] - 0.01, lam[-1] + 0.01
    cf, _, _, _ = best_oracle.build_filter(lo, hi, lam[9] + 1e-3, lam[20] - 1e-3, 64)
    X = np.random.default_rng(7).uniform(-1, 1, (30, 4))
    p = np.array([best_oracle.clenshaw(cf, (z - 0.5 * (lo + hi)) / (0.5 * (hi - lo))) for z in lam])
    want = V @ (p[:, None] * (V.T @ X))
    Y = DeviceMatrix(ctx, n, rp, ci, va).filter_apply(cf, 0.5 * (lo + hi), 0.5 * (hi - lo), X)
    assert np.abs(Y - want).max() <= 1e-10 * np.abs(want).max()


def test_spmm_ragged_rows_and_determinism(ctx, best_oracle):
    # kernels_test.cpp:94-138: ragged rows incl. empty rows; run-to-run bitwise determinism
    rng = np.random.default_rng(5)
    n = 257
    dense = np.zeros((n, n))
    for i in range(n):
        if i % 7 == 3:
            continue                                    # empty rows
        k = int(rng.integers(1, 40))
        cols = rng.choice(n, k, replace=False)
        dense[i, cols] = rng.uniform(-1, 1, k)
    dense = dense + dense.T
    import scipy.sparse as sp
    n, rp, ci, va = M._to_csr(sp.csr_matrix(dense))
    A = DeviceMatrix(ctx, n, rp, ci, va)
    X = block(n, 3, 9)
    ctx.set_exact(True)
    try:
        Y = A.spmm(X)
        ref_cols = [best_oracle.csr_matvec(n, rp, ci, va, X[:, j]) for j in range(3)]
        best_oracle_is_ref = best_oracle.kind == "reference"
        if best_oracle_is_ref:
            best_oracle.set_backend("scalar")
            ref_cols = [best_oracle.csr_matvec(n, rp, ci, va, X[:, j]) for j in range(3)]
            best_oracle.set_backend("avx2")
        assert np.array_equal(Y, np.stack(ref_cols, 1))      # spmm_block == per-column spmv
    finally:
        ctx.set_exact(False)
    Y1, Y2 = A.spmm(X), A.spmm(X)
    assert np.array_equal(Y1, Y2)
    assert np.abs(Y1 - dense @ X).max() < 1e-13               # sparse_test.cpp:173-187
    sym = X[:, 0] @ A.spmm(X[:, 1:2])[:, 0] - X[:, 1] @ A.spmm(X[:, 0:1])[:, 0]
    assert abs(sym) < 1e-12                                   # operator symmetry


def test_level0_seams(ctx, best_oracle):
    # kernels_test.cpp:60-92 — dot / axpy / clenshaw_combine over tail sizes
    rng = np.random.default_rng(1)
    for n in (1, 2, 3, 7, 8, 31, 32, 33, 255, 1001, 4097):
        x, y, w, z = (rng.standard_normal(n) for _ in range(4))
        assert abs(ctx.dot(x, y) - float(x @ y)) <= 1e-13 * max(1.0, np.abs(x * y).sum())
        assert np.abs(ctx.axpy(0.37, x, y) - (y + 0.37 * x)).max() <= 1e-15 * 4
        ctx.set_exact(True)
        out = ctx.clenshaw_combine(1.25, -0.5, 0.3, w, x, y, z)
        ctx.set_exact(False)
        assert np.array_equal(out, 1.25 * w + (-0.5) * x - y + 0.3 * z)


def test_dimension_errors(ctx):
    n, rp, ci, va = M.laplacian2d(6)
    A = DeviceMatrix(ctx, n, rp, ci, va)
    with pytest.raises(AssertionError):
        A.spmm(np.ones((n + 1, 2)))
    H = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    with pytest.raises(FlzError) as e:
        H.spmm_block(np.ones((n + 1, 2)))
    assert e.value.code == -2                                   # DimensionError
    with pytest.raises(FlzError):
        DeviceMatrix(ctx, 4, [0, 1, 2, 3, 4], [0, 1, 2, 9], [1.0, 1.0, 1.0, 1.0])
    with pytest.raises(FlzError):
        A.filter_apply([1.0, 0.5], 0.0, -1.0, np.ones((n, 1)))  # non-positive half width


def test_full_size_linearity_and_symmetry(ctx):
    """Size-independent properties at the C2 shape (3D Laplacian 100^3, r = 3)."""
    n, rp, ci, va = M.laplacian3d(100)
    A = DeviceMatrix(ctx, n, rp, ci, va)
    cf = S.indicator_coefficients(-0.97, -0.96, 60)
    X, Z = block(n, 3, 1), block(n, 3, 2)
    c, e = 6.0, 6.06
    FX, FZ = A.filter_apply(cf, c, e, X), A.filter_apply(cf, c, e, Z)
    F2 = A.filter_apply(cf, c, e, 2.0 * X - 0.5 * Z)
    scale = np.abs(FX).max() + np.abs(FZ).max()
    assert np.abs(F2 - (2.0 * FX - 0.5 * FZ)).max() <= 1e-12 * scale          # linearity
    assert abs(np.sum(Z * FX) - np.sum(X * FZ)) <= 1e-10 * abs(np.sum(Z * FX)) + 1e-9  # p(A) symmetric
    # against SciPy's CSR product on one plain block product
    As = M.csr_to_scipy(n, rp, ci, va)
    assert np.abs(A.spmm(X) - As @ X).max() <= 1e-13 * np.abs(X).max() * 12


def test_full_size_eigenvector_invariance(ctx):
    """C2 shape: an analytic eigenvector v of the 100^3 Laplacian satisfies p(A) v = p(lambda) v
    (the reference's eigenvector-invariance test, filter_test.cpp:268-283, at BASELINE size)."""
    g = 100
    n, rp, ci, va = M.laplacian3d(g)
    A = DeviceMatrix(ctx, n, rp, ci, va)
    idx = np.arange(1, g + 1)
    modes = ((3, 5, 7), (1, 1, 1), (40, 2, 17))
    V = np.empty((n, 3))
    lam = []
    for k, (a, b, c) in enumerate(modes):
        sx, sy, sz = (np.sin(m * np.pi * idx / (g + 1)) for m in (a, b, c))
        V[:, k] = (sz[:, None, None] * sy[None, :, None] * sx[None, None, :]).ravel()
        V[:, k] /= np.linalg.norm(V[:, k])
        lam.append(sum(2.0 * (1.0 - np.cos(m * np.pi / (g + 1))) for m in (a, b, c)))
    lo, hi = -0.05, 12.05
    cf = S.indicator_coefficients(-0.9, -0.8, 150)
    Y = A.filter_apply(cf, 0.5 * (lo + hi), 0.5 * (hi - lo), V)
    for k in range(3):
        t = (lam[k] - 0.5 * (lo + hi)) / (0.5 * (hi - lo))
        assert np.abs(Y[:, k] - S.clenshaw(cf, t) * V[:, k]).max() <= 1e-12


def test_full_size_parsec_shape_properties(ctx):
    """C3 shape (PARSEC-like, n = 113k, long ragged rows): product against SciPy, linearity and
    symmetry of p(A) — size-independent checks of the long-row kernel at BASELINE size."""
    n, rp, ci, va = M.parsec_like()
    A = DeviceMatrix(ctx, n, rp, ci, va)
    As = M.csr_to_scipy(n, rp, ci, va)
    X, Z = block(n, 3, 11), block(n, 3, 12)
    ref = As @ X
    assert np.abs(A.spmm(X) - ref).max() <= 1e-13 * np.abs(ref).max()
    cf = S.indicator_coefficients(-0.95, -0.9, 40)
    c, e = 16.0, 17.5
    FX, FZ = A.filter_apply(cf, c, e, X), A.filter_apply(cf, c, e, Z)
    F2 = A.filter_apply(cf, c, e, X + 3.0 * Z)
    scale = np.abs(FX).max() + np.abs(FZ).max()
    assert np.abs(F2 - (FX + 3.0 * FZ)).max() <= 1e-12 * scale
    assert abs(np.sum(Z * FX) - np.sum(X * FZ)) <= 1e-10 * abs(np.sum(Z * FX)) + 1e-9
    ctx.set_exact(True)
    try:
        Fe = A.filter_apply(cf, c, e, X)
    finally:
        ctx.set_exact(False)
    assert np.abs(FX - Fe).max() <= 1e-13 * np.abs(Fe).max()      # fast vs reference-order mode
