"""Pins the CPU oracles (test infrastructure) — runs without a GPU.

* the plain-C restatement oracle/flz_oracle.c against the reference's own known answers,
  the committed golden vectors (generated from the unmodified reference) and, where
  oracle/_ref exists, the reference itself bit for bit;
* the reference shim against the same known answers.
"""
import numpy as np
import pytest

import oracle
from paper_2409_15053_b200 import matrices as M


def block(n, r, seed):
    return np.random.default_rng(seed).standard_normal((n, r))


# ---- known answers held by the reference's tests --------------------------------------
def test_known_coefficients(port):
    # filter_test.cpp:27-47
    b = port.indicator_coefficients(-1.0, -0.5, 3)
    assert abs(b[0] - 1.0 / 3.0) < 1e-15
    assert abs(b[1] - (-0.5513288954217919)) < 1e-15
    assert abs(port.indicator_coefficients(0.1, 0.3, 2)[0] - 0.06510240359141833) < 1e-16


def test_known_degrees(port):
    # filter_test.cpp:96-99, acceptance_main.cpp:39-46
    assert port.select_degree(0.1, 0.3) == (48, False)
    assert port.select_degree(-1.0, -0.5) == (10, False)
    assert port.select_degree(-0.001, 0.001) == (1000, True)  # clamps at max_degree


def test_clenshaw_vs_forward(port):
    # filter_test.cpp:169-204 — backward recurrence equals the forward Chebyshev sum
    cf = port.indicator_coefficients(-0.3, 0.45, 120)
    for t in np.linspace(-1, 1, 37):
        T = np.cos(np.arange(121) * np.arccos(t))
        assert abs(port.clenshaw(cf, t) - cf @ T) < 1e-12


def test_filter_on_diagonal_matrix(port):
    # filter_test.cpp:218-234: p(A) e on diag(1..5) equals scalar p(lambda_i); r*m matvecs
    n, rp, ci, va = M.diag_matrix([1, 2, 3, 4, 5])
    A = port.matrix_from_csr(n, rp, ci, va)
    cf, _, _, _ = port.build_filter(0.5, 5.5, 1.5, 3.5, 48)
    X = np.ones((5, 5))
    before = port.matvec_count()
    Y = port.filter_apply(A, cf, 0.5, 5.5, X)
    assert port.matvec_count() - before == 5 * 48
    for i in range(5):
        want = port.clenshaw(cf, ((i + 1) - 3.0) / 2.5)
        assert np.allclose(Y[i], want, atol=1e-12)


def test_solve_analytic_laplacian(port):
    # lanczos_test.cpp:426-452 — Laplacian-900 eigenpairs vs the closed form
    n, rp, ci, va = M.laplacian2d(30)
    A = port.matrix_from_csr(n, rp, ci, va)
    res = port.solve(A, 3.0, 3.8)
    ana = M.laplacian2d_eigenvalues(30)
    ana = ana[(ana >= 3.0) & (ana <= 3.8)]
    assert res.stats["converged"] == 1
    assert len(res.eigenvalues) == len(ana)
    assert np.abs(res.eigenvalues - ana).max() < 1e-10
    assert res.residuals.max() <= 1e-10
    V = res.eigenvectors
    assert np.abs(V.T @ V - np.eye(V.shape[1])).max() < 1e-12
    # accounting identity MV = r*m*iters (lanczos_test.cpp:388-415)
    assert res.stats["mv_iteration"] == 3 * res.stats["degree"] * res.stats["block_steps"]


def test_multiplicity_three(port):
    # lanczos_test.cpp:264-272 / acceptance criterion 4
    n, rp, ci, va = M.diag_matrix([1, 2, 2, 2, 3])
    res = port.solve(port.matrix_from_csr(n, rp, ci, va), 1.5, 2.5)
    assert len(res.eigenvalues) == 3 and np.allclose(res.eigenvalues, 2.0, atol=1e-8)


def test_errors(port):
    n, rp, ci, va = M.diag_matrix([1, 2, 3, 4, 5])
    A = port.matrix_from_csr(n, rp, ci, va)
    with pytest.raises(oracle.OracleError):
        port.solve(A, 2.0, 1.0)  # alpha >= beta
    with pytest.raises(oracle.OracleError):
        port.solve(A, 50.0, 60.0)  # outside the spectrum
    with pytest.raises(oracle.OracleError):
        port.matrix_from_triplets(3, [0, 1], [1, 2], [1.0, 2.0])  # asymmetric


# ---- golden vectors generated from the unmodified reference ----------------------------
def test_port_vs_golden_scalars(port, golden):
    assert np.array_equal(port.indicator_coefficients(-1.0, -0.5, 12), golden["coef_m1_m05"])
    assert np.array_equal(port.indicator_coefficients(0.1, 0.3, 200), golden["coef_01_03"])
    degs = [port.select_degree(0.1, 0.3)[0], port.select_degree(-1.0, -0.5)[0],
            port.select_degree(-0.02, 0.02)[0], port.select_degree(0.3, 0.9, 0.1)[0]]
    assert degs == list(golden["degrees"])
    vals = [port.clenshaw(golden["coef_01_03"], t) for t in golden["clenshaw_pts"]]
    assert np.array_equal(vals, golden["clenshaw_vals"])
    Q = port.init_block(1000, 3, 20177)
    assert np.array_equal(Q, golden["init_block_1000x3_scalar"])
    assert np.abs(Q - golden["init_block_1000x3_avx2"]).max() < 1e-15


CASES = {
    "lap2d30": lambda: M.laplacian2d(30),
    "rand400": lambda: M.random_sparse_sym(400, 0.04, 7),
    "parsec7k": lambda: M.parsec_like(radius=12.0, n_atoms=12),
    "lap3d12": lambda: M.laplacian3d(12),
}


@pytest.mark.parametrize("name", list(CASES))
def test_port_filter_vs_golden(port, golden, name):
    n, rp, ci, va = CASES[name]()
    lo, hi, a, b, r, seed = golden[f"filter_{name}_meta"]
    A = port.matrix_from_csr(n, rp, ci, va)
    X = block(n, int(r), int(seed))
    Y = port.filter_apply(A, golden[f"filter_{name}_coeffs"], lo, hi, X)
    # bit-identical to the reference's scalar backend; AVX2 differs by rounding only
    assert np.array_equal(Y, golden[f"filter_{name}_scalar"])
    scale = np.abs(Y).max()
    assert np.abs(Y - golden[f"filter_{name}_avx2"]).max() <= 1e-13 * scale


def test_port_factorization_vs_golden(port, golden):
    n, rp, ci, va = M.laplacian2d(30)
    A = port.matrix_from_csr(n, rp, ci, va)
    lo, hi = port.estimate_bounds(A)
    assert np.allclose([lo, hi], golden["lap2d30_bounds"], rtol=1e-13)
    lo, hi = golden["lap2d30_bounds"]
    cf, _, _, _ = port.build_filter(lo, hi, 3.0, 3.8)
    F = port.factorization(A, port.init_block(n, 3), 300, cf, (lo, hi), (3.0, 3.8))
    assert F.expand(8) == 8
    Q, D, S, dead = F.get()
    assert np.abs(Q - golden["fact_lap2d30_Q"]).max() < 1e-12
    assert np.abs(D - golden["fact_lap2d30_D"]).max() < 1e-13
    assert np.abs(S - golden["fact_lap2d30_S"]).max() < 1e-13
    conv, vals, est, wanted, _ = F.check(3.0, 3.8)
    assert np.abs(vals - golden["fact_lap2d30_ritz"]).max() < 1e-12
    assert np.array_equal(wanted, golden["fact_lap2d30_wanted"])


SOLVES = {
    "lap2d30_r3": (lambda: M.laplacian2d(30), 3.0, 3.8, {}),
    "lap2d30_r1": (lambda: M.laplacian2d(30), 3.0, 3.8, dict(block_size=1)),
    "lap2d30_m20": (lambda: M.laplacian2d(30), 3.0, 3.8, dict(degree=20)),
    "rand400": (lambda: M.random_sparse_sym(400, 0.04, 7), -0.5, 0.5, {}),
    "diag_mult3": (lambda: M.diag_matrix([1, 2, 2, 2, 3]), 1.5, 2.5, {}),
    "diag5": (lambda: M.diag_matrix([1, 2, 3, 4, 5]), 1.5, 4.5, {}),
    "parsec7k": (lambda: M.parsec_like(radius=12.0, n_atoms=12), -0.6, 0.0, dict(degree=50)),
}


@pytest.mark.parametrize("name", list(SOLVES))
def test_port_solve_vs_golden(port, golden, name):
    gen, a, b, kw = SOLVES[name]
    n, rp, ci, va = gen()
    res = port.solve(port.matrix_from_csr(n, rp, ci, va), a, b, oracle.make_config(**kw),
                     want_vectors=False)
    eigs = golden[f"solve_{name}_eigs"]
    blocks, degree, mv, conv, norm, maxres = golden[f"solve_{name}_stats"]
    assert len(res.eigenvalues) == len(eigs)
    assert np.abs(res.eigenvalues - eigs).max() <= 1e-10 * norm
    assert res.stats["degree"] == degree and res.stats["converged"] == conv
    assert res.residuals.max() <= 1e-10


# ---- against the reference itself, where it is built ----------------------------------
def test_port_bit_exact_vs_reference_scalar(port, ref):
    ref.set_backend("scalar")
    try:
        n, rp, ci, va = M.random_sparse_sym(300, 0.05, 3)
        Ar, Ap = ref.matrix_from_csr(n, rp, ci, va), port.matrix_from_csr(n, rp, ci, va)
        assert all(np.array_equal(x, y) for x, y in zip(Ar.csr(), Ap.csr()))
        assert ref.estimate_bounds(Ar) == port.estimate_bounds(Ap)
        a = ref.solve(Ar, -0.4, 0.4, oracle.make_config(collect_diagnostics=True))
        b = port.solve(Ap, -0.4, 0.4, oracle.make_config(collect_diagnostics=True))
        assert np.array_equal(a.eigenvalues, b.eigenvalues)
        assert np.array_equal(a.eigenvectors, b.eigenvectors)
        assert np.array_equal(a.residuals, b.residuals)
        for key in ("block_steps", "degree", "mv_total", "checks", "converged", "ortho_error"):
            assert a.stats[key] == b.stats[key]
        bands = np.random.default_rng(5).uniform(-1, 1, (4, 60))
        va_, Wa = ref.sym_band_eig(bands)
        vb_, Wb = port.sym_band_eig(bands)
        assert np.array_equal(va_, vb_) and np.array_equal(Wa, Wb)
    finally:
        ref.set_backend("avx2")


def test_reference_shim_known_answers(ref):
    assert ref.kind == "reference"
    assert ref.select_degree(0.1, 0.3) == (48, False)
    assert ref.select_degree(-1.0, -0.5) == (10, False)
    assert abs(ref.indicator_coefficients(-1.0, -0.5, 1)[1] + 0.5513288954217919) < 1e-15
