"""GPU parity of the block Lanczos engine (K3-K10): factorization identities, basis
orthonormality, agreement with the reference factorization, breakdown handling."""
import numpy as np
import pytest

from paper_2409_15053_b200 import matrices as M, solver as S

pytestmark = pytest.mark.gpu


def dense_T(D, S_, k, r):
    T = np.zeros((k * r, k * r))
    for b in range(k):
        T[b * r:(b + 1) * r, b * r:(b + 1) * r] = 0.5 * (D[b] + D[b].T)
        if b + 1 < k:
            T[(b + 1) * r:(b + 2) * r, b * r:(b + 1) * r] = S_[b]
            T[b * r:(b + 1) * r, (b + 1) * r:(b + 2) * r] = S_[b].T
    return T


def test_factorization_matches_golden(golden):
    n, rp, ci, va = M.laplacian2d(30)
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    lo, hi = golden["lap2d30_bounds"]
    cf, _, _, _ = S.build_filter(lo, hi, 3.0, 3.8)
    F = S.LanczosFactorization(A, S.init_block(n, 3), 300, cf, (lo, hi), (3.0, 3.8))
    assert F.expand(8) == 8
    Q, D, S_, dead = F.get()
    assert np.abs(Q - golden["fact_lap2d30_Q"]).max() < 1e-12
    assert np.abs(D - golden["fact_lap2d30_D"]).max() < 1e-13
    assert np.abs(S_ - golden["fact_lap2d30_S"]).max() < 1e-13
    conv, vals, est, wanted, deadp = F.check(3.0, 3.8)
    assert np.abs(vals - golden["fact_lap2d30_ritz"]).max() < 1e-12
    assert np.abs(est - golden["fact_lap2d30_est"]).max() < 1e-10
    assert np.array_equal(wanted, golden["fact_lap2d30_wanted"])


def test_bounds_match_reference(golden):
    n, rp, ci, va = M.laplacian2d(30)
    lo, hi = S.estimate_spectral_bounds(S.SparseSymMatrix.from_csr(n, rp, ci, va))
    assert np.allclose([lo, hi], golden["lap2d30_bounds"], rtol=0, atol=1e-12)
    # bounds exactness on diag(1..5) incl. the 0.5 % widening (lanczos_test.cpp:42-74)
    lo, hi = S.estimate_spectral_bounds(S.SparseSymMatrix.from_csr(*M.diag_matrix([1, 2, 3, 4, 5])))
    assert abs(lo - (1 - 0.02)) < 1e-10 and abs(hi - (5 + 0.02)) < 1e-10


@pytest.mark.parametrize("filtered,r", [(True, 3), (False, 3), (True, 1), (True, 2), (False, 4)])
def test_factorization_identity(filtered, r):
    # lanczos_test.cpp:161-205: op(A) Q_k = Q_k T_k + Q_pend S_k E_k^T, Q_k^T op(A) Q_k = T_k
    n, rp, ci, va = M.random_sparse_sym(300, 0.05, 77)
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    lo, hi = -9.0, 9.0
    cf = S.build_filter(lo, hi, -1.0, 1.0, 30)[0] if filtered else None
    F = S.LanczosFactorization(A, S.init_block(n, r, 5), 120, cf, (lo, hi), (-1.0, 1.0))
    k = F.expand(12)
    assert k == 12
    Q, D, S_, dead = F.get()
    Qk, Qp = Q[:, :k * r], Q[:, k * r:]
    T = dense_T(D, S_, k, r)
    OpQ = A.filter_apply(cf, lo, hi, Qk[:, :1]) if False else None
    cols = [A.filter_apply(cf, lo, hi, Qk[:, j:j + 3]) if filtered else A.spmm_block(Qk[:, j:j + 3])
            for j in range(0, k * r, 3)]
    OpQ = np.concatenate(cols, 1)
    E = np.zeros((k * r, r))
    E[(k - 1) * r:, :] = np.eye(r)
    resid = OpQ - Qk @ T - Qp @ S_[k - 1] @ E.T
    assert np.abs(resid).max() < 1e-10
    assert np.abs(Qk.T @ OpQ - T).max() < 1e-10
    assert np.abs(Q.T @ Q - np.eye((k + 1) * r)).max() < 1e-12
    assert np.allclose(np.tril(S_[k - 1], -1), 0) and np.all(np.diag(S_[k - 1]) > 0)


def test_basis_orthonormality_sixty_vectors():
    # lanczos_test.cpp:124-132
    n, rp, ci, va = M.laplacian2d(30)
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    cf, _, _, _ = S.build_filter(-0.03, 8.03, 3.0, 3.8)
    F = S.LanczosFactorization(A, S.init_block(n, 3), 120, cf, (-0.03, 8.03), (3.0, 3.8))
    assert F.expand(20) == 20
    assert F.ortho_error() <= 1e-12
    Q = F.get()[0]
    assert np.abs(Q[:, :60].T @ Q[:, :60] - np.eye(60)).max() <= 1e-12


def test_identity_filter_breakdown_path():
    # lanczos_test.cpp:106-122: p == 1 -> Z = Q, D_1 = I, S_1 = 0, random replacements
    n, rp, ci, va = M.laplacian2d(8)
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    F = S.LanczosFactorization(A, S.init_block(n, 3), 30, [1.0], (-0.1, 8.1), (1.0, 2.0))
    assert F.expand(1) == 1
    Q, D, S_, dead = F.get()
    assert np.abs(D[0] - np.eye(3)).max() < 1e-14
    assert np.abs(S_[0]).max() < 1e-13
    assert F.flags() & 2                       # breakdown recorded
    assert not dead.any()                      # replaced by fresh directions
    assert np.abs(Q.T @ Q - np.eye(6)).max() < 1e-12


@pytest.mark.parametrize("which", [0, 1])
def test_mixed_dead_and_live_pending_block_stays_orthonormal(best_oracle, which):
    """A start block whose column `which` is an eigenvector, r = 3: that pending column dies in
    the first step (p(A) v = p(lambda) v lies in the basis) while LATER columns stay alive.  The
    replacement must be orthogonal to those later columns as well (lanczos.cpp:232-262 has it
    in place before they are processed): Q^T Q = I, the factorization identity holds, and the
    Ritz values of T_k agree with the reference's run from the same start block."""
    g = 12
    n, rp, ci, va = M.laplacian2d(g)
    idx = np.arange(1, g + 1)
    v = np.outer(np.sin(3 * np.pi * idx / (g + 1)), np.sin(5 * np.pi * idx / (g + 1))).ravel()
    q = v / np.linalg.norm(v)
    rest = np.random.default_rng(4).standard_normal((n, 2))
    rest -= np.outer(q, q @ rest)
    rest = np.linalg.qr(rest)[0]
    cols = [rest[:, 0], rest[:, 1]]
    cols.insert(which, q)                    # orthonormal start block, eigenvector at `which`
    start = np.column_stack(cols)
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    lo, hi = -0.05, 8.05
    cf = S.build_filter(lo, hi, 3.0, 4.0, 20)[0]
    F = S.LanczosFactorization(A, start, 60, cf, (lo, hi), (3.0, 4.0))
    k = F.expand(6)
    assert k == 6 and F.flags() & 2                      # breakdown recorded, run continues
    Q, D, S_, dead = F.get()
    assert not dead.any()
    assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() < 1e-12
    assert F.ortho_error() <= 1e-12
    r = 3
    Qk, Qp = Q[:, :k * r], Q[:, k * r:]
    T = dense_T(D, S_, k, r)
    OpQ = np.concatenate([A.filter_apply(cf, lo, hi, Qk[:, j:j + 3]) for j in range(0, k * r, 3)], 1)
    E = np.zeros((k * r, r))
    E[(k - 1) * r:, :] = np.eye(r)
    assert np.abs(OpQ - Qk @ T - Qp @ S_[k - 1] @ E.T).max() < 1e-10
    assert np.abs(Qk.T @ OpQ - T).max() < 1e-10
    # the reference from the same start block: same orthonormality (its replacement vectors
    # are drawn from the same stream, but it orthogonalises the other way round, so only
    # basis-independent quantities are compared)
    Ao = best_oracle.matrix_from_csr(n, rp, ci, va)
    Fo = best_oracle.factorization(Ao, start, 60, cf, (lo, hi), (3.0, 4.0))
    assert Fo.expand(6) == 6
    assert Fo.ortho_error() <= 1e-12


def test_space_exhaustion_on_tiny_matrix():
    # lanczos_test.cpp:207-224 / :297-308: the whole space gets spanned, columns go dead
    n, rp, ci, va = M.diag_matrix([1, 2, 3, 4, 5])
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    F = S.LanczosFactorization(A, S.init_block(5, 3), 12, None)
    total = 0
    for _ in range(4):
        total += F.expand(1)
    Q, D, S_, dead = F.get()
    assert F.flags() & 1 and dead.sum() >= 1
    live = Q[:, : len(dead)][:, dead == 0]
    assert live.shape[1] == 5
    assert np.abs(live.T @ live - np.eye(5)).max() < 1e-12


def test_expand_r1_recovers_spectrum():
    # lanczos_test.cpp:92-104
    A = S.SparseSymMatrix.from_csr(*M.diag_matrix([1, 2, 3, 4, 5]))
    F = S.LanczosFactorization(A, S.init_block(5, 1), 10, None)
    assert F.expand(5) == 5
    _, D, S_, _ = F.get()
    T = dense_T(D, S_, 5, 1)
    assert np.abs(np.linalg.eigvalsh(T) - np.arange(1, 6)).max() < 1e-10
