"""Host-side logic of libflz (no GPU): filter scalars, start block, projected eigenproblem,
matrix validation and Matrix Market I/O — checked against the oracle and NumPy."""
import os

import numpy as np
import pytest

import oracle
from paper_2409_15053_b200 import FlzError, matrices as M, solver as S


def test_filter_scalars_bit_equal_to_oracle(best_oracle, golden):
    for a, b, deg in [(-1.0, -0.5, 12), (0.1, 0.3, 200), (-0.37, 0.81, 64)]:
        assert np.array_equal(S.indicator_coefficients(a, b, deg),
                              best_oracle.indicator_coefficients(a, b, deg))
    assert np.array_equal(S.indicator_coefficients(0.1, 0.3, 200), golden["coef_01_03"])
    assert S.select_degree(0.1, 0.3) == (48, False)        # filter_test.cpp:96-99
    assert S.select_degree(-1.0, -0.5) == (10, False)
    assert S.select_degree(-0.001, 0.001) == (1000, True)
    for a, b, eps in [(-0.02, 0.02, 0.255), (0.3, 0.9, 0.1), (-0.9, -0.2, 0.4)]:
        assert S.select_degree(a, b, eps) == best_oracle.select_degree(a, b, eps)
    cf = golden["coef_01_03"]
    vals = [S.clenshaw(cf, t) for t in golden["clenshaw_pts"]]
    assert np.array_equal(vals, golden["clenshaw_vals"])


def test_build_filter_matches_oracle_and_errors(best_oracle):
    for args in [(-0.05, 8.05, 3.0, 3.8, 0), (-1.5, 34.0, -0.6, 0.0, 50), (0.0, 1.0, -5.0, 0.4, 0)]:
        cf, a_s, b_s, cl = S.build_filter(*args)
        cf2, a2, b2, cl2 = best_oracle.build_filter(*args)
        assert np.array_equal(cf, cf2) and (a_s, b_s, cl) == (a2, b2, cl2)
    with pytest.raises(FlzError) as e:
        S.build_filter(0.0, 1.0, 2.0, 3.0)       # interval outside the bounds
    assert e.value.code == -3                      # -> IntervalError
    with pytest.raises(FlzError):
        S.build_filter(0.0, 1.0, 0.6, 0.4)       # alpha >= beta
    with pytest.raises(FlzError):
        S.indicator_coefficients(0.5, 0.2, 4)


def test_init_block_matches_reference(golden):
    Q = S.init_block(1000, 3, 20177)
    assert np.abs(Q - golden["init_block_1000x3_scalar"]).max() < 1e-15
    assert np.abs(Q.T @ Q - np.eye(3)).max() < 1e-14
    assert np.array_equal(Q, S.init_block(1000, 3, 20177))       # deterministic per seed
    assert not np.array_equal(Q, S.init_block(1000, 3, 20178))
    with pytest.raises(FlzError):
        S.init_block(2, 3)


def band_dense(bands):
    sb, dim = bands.shape[0] - 1, bands.shape[1]
    A = np.zeros((dim, dim))
    for d in range(sb + 1):
        for i in range(dim - d):
            A[i + d, i] = A[i, i + d] = bands[d, i]
    return A


@pytest.mark.parametrize("dim,sb", [(1, 0), (2, 1), (7, 1), (40, 3), (61, 5), (30, 20), (12, 11),
                                    (200, 3)])
def test_sym_band_eig(best_oracle, dim, sb):
    rng = np.random.default_rng(dim * 31 + sb)
    bands = rng.uniform(-1, 1, (sb + 1, dim))
    A = band_dense(bands)
    vals, W = S.sym_band_eig(bands)
    assert np.abs(vals - np.linalg.eigvalsh(A)).max() < 1e-12
    assert np.abs(W.T @ W - np.eye(dim)).max() < 1e-12          # band_eig_test orthogonality
    assert np.abs(A @ W - W * vals).max() < 1e-12
    ov, _ = best_oracle.sym_band_eig(bands)
    assert np.abs(vals - ov).max() < 1e-12


@pytest.mark.parametrize("dim,sb", [(9, 1), (60, 3), (150, 1), (90, 4)])
def test_band_ritz_rows_equals_full_rows(dim, sb):
    """The cheap periodic-check path returns exactly the rows of the full eigenvector matrix."""
    bands = np.random.default_rng(dim + sb).uniform(-1, 1, (sb + 1, dim))
    vals, W = S.sym_band_eig(bands)
    rows = [dim - 1, dim - 2, 0, dim // 2]
    v2, R = S.band_ritz_rows(bands, rows)
    assert np.array_equal(vals, v2)
    assert np.array_equal(R, W[rows, :])          # same rotations -> bitwise the same rows
    v3, R3 = S.band_ritz_rows(bands, [])
    assert np.array_equal(v3, vals) and R3.shape == (0, dim)


@pytest.mark.parametrize("dim,sb", [(50, 1), (120, 3), (300, 3)])
def test_band_inverse_iteration(dim, sb):
    bands = np.random.default_rng(7 * dim + sb).uniform(-1, 1, (sb + 1, dim))
    A = band_dense(bands)
    vals, _ = S.sym_band_eig(bands, want_vectors=False)
    pick = list(range(dim - 25, dim))
    W, res, ortho = S.band_eigenvectors(bands, vals, pick)
    assert res < 1e-13 and ortho < 1e-12
    assert np.abs(A @ W - W * vals[pick]).max() < 1e-12


@pytest.mark.parametrize("dim,sb", [(260, 259), (400, 3)])
def test_host_eigensolvers_do_not_depend_on_thread_count(dim, sb, monkeypatch):
    """Recorded rotations/reflectors applied to disjoint row ranges, and independent clusters
    of the inverse iteration, on 1 or 8 host threads: bit-identical results (dense 260 x 260 is
    the recovery's V'AV problem, the band is T_k)."""
    bands = np.random.default_rng(dim + sb).uniform(-1, 1, (sb + 1, dim))
    out = {}
    for threads in ("1", "8"):
        monkeypatch.setenv("FLZ_HOST_THREADS", threads)
        vals, W = S.sym_band_eig(bands)
        pick = list(range(dim - 120, dim))
        V, res, ortho = S.band_eigenvectors(bands, vals, pick)
        out[threads] = (vals, W, V, res, ortho)
    A = band_dense(bands)
    vals, W, V, res, ortho = out["8"]
    assert np.abs(vals - np.linalg.eigvalsh(A)).max() < 1e-11
    assert np.abs(W.T @ W - np.eye(dim)).max() < 1e-12 and np.abs(A @ W - W * vals).max() < 1e-11
    assert res < 1e-12 and ortho < 1e-11
    for a, b in zip(out["1"], out["8"]):
        assert np.array_equal(a, b)


def test_band_inverse_iteration_with_multiplicities():
    # block diagonal of identical blocks -> exactly repeated eigenvalues
    dim = 90
    bands = np.zeros((3, dim))
    blk = np.random.default_rng(3).uniform(-1, 1, (3, 30))
    blk[1, 29] = blk[2, 28:] = 0.0
    for c in range(3):
        bands[:, 30 * c:30 * (c + 1)] = blk
    A = band_dense(bands)
    vals, _ = S.sym_band_eig(bands, want_vectors=False)
    pick = list(range(dim - 30, dim))
    W, res, ortho = S.band_eigenvectors(bands, vals, pick)
    assert res < 1e-12 and ortho < 1e-11
    assert np.abs(A @ W - W * vals[pick]).max() < 1e-11


def test_from_entries_semantics():
    # duplicates are summed, asymmetry / range / non-finite rejected (sparse.cpp:27-85)
    A = S.SparseSymMatrix.from_entries(3, [0, 0, 1, 2, 0, 1], [0, 0, 1, 2, 1, 0],
                                       [1.0, 0.5, 2.0, 3.0, -1.0, -1.0])
    rp, ci, va = A.csr()
    assert list(rp) == [0, 2, 4, 5] and list(ci) == [0, 1, 0, 1, 2]
    assert list(va) == [1.5, -1.0, -1.0, 2.0, 3.0]
    for rows, cols, vals in [([0, 1], [1, 2], [1.0, 2.0]), ([0, 1], [1, 0], [1.0, 1.5]),
                             ([0], [3], [1.0]), ([0], [0], [float("nan")])]:
        with pytest.raises(FlzError):
            S.SparseSymMatrix.from_entries(3, rows, cols, vals)
    n, rp, ci, va = M.laplacian2d(30)
    assert len(va) == 5 * n - 4 * 30                  # sparse_test.cpp:206-209
    assert S.SparseSymMatrix.from_csr(n, rp, ci, va).nnz == len(va)


MM_OK = """%%MatrixMarket matrix coordinate real symmetric
% comment
3 3 4
1 1 2.0
2 1 -1.0
2 2 2.0
3 3 5e-1
"""


def test_matrix_market_round_trip(tmp_path, best_oracle):
    p = tmp_path / "a.mtx"
    p.write_text(MM_OK)
    A = S.SparseSymMatrix.load_matrix_market(p)
    rp, ci, va = A.csr()
    assert list(rp) == [0, 2, 4, 5] and list(va) == [2.0, -1.0, -1.0, 2.0, 0.5]
    n, rp, ci, va = M.random_sparse_sym(60, 0.2, 5)
    B = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    q = tmp_path / "b.mtx"
    B.save_matrix_market(q)
    C2 = S.SparseSymMatrix.load_matrix_market(q)
    assert all(np.array_equal(x, y) for x, y in zip(B.csr(), C2.csr()))   # %.17g is exact
    general = tmp_path / "g.mtx"
    general.write_text("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n1 2 3\n"
                       "2 1 3.000000000000001\n")
    G = S.SparseSymMatrix.load_matrix_market(general)
    assert G.csr()[2][1] == G.csr()[2][2]             # symmetrised by averaging
    pat = tmp_path / "p.mtx"
    pat.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n2 2 2\n1 1\n2 1\n")
    assert list(S.SparseSymMatrix.load_matrix_market(pat).csr()[2]) == [1.0, 1.0, 1.0]


@pytest.mark.parametrize("text,needle", [
    ("", "empty file"),
    ("%%NotMM matrix coordinate real symmetric\n1 1 0\n", ":1:"),
    ("%%MatrixMarket matrix array real general\n1 1\n", "expected coordinate"),
    ("%%MatrixMarket matrix coordinate complex symmetric\n1 1 0\n", "complex"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n", "hermitian"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 0\n", "not square"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n", "upper-triangle"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n", "file ends after 1 of 2"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1.0\n2 2 1.0\n", "more entries"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 abc\n", ":3:"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1.0\n2 1 2.0\n", "not symmetric"),
])
def test_matrix_market_errors(tmp_path, text, needle):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(FlzError) as e:
        S.SparseSymMatrix.load_matrix_market(p)
    assert needle in str(e.value)
    with pytest.raises(FlzError):
        S.SparseSymMatrix.load_matrix_market(tmp_path / "missing.mtx")


def _write_mm(path, n, rows, cols, vals, symmetry="symmetric", shuffle=None, comments=True):
    order = np.arange(len(rows)) if shuffle is None else np.random.default_rng(shuffle).permutation(len(rows))
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate real {symmetry}\n")
        if comments:
            f.write("% a comment\n\n%another\n")
        f.write(f"{n} {n} {len(rows)}\n")
        for k in order:
            f.write(f"{rows[k] + 1} {cols[k] + 1} {vals[k]:.17g}\n")
            if comments and k % 97 == 0:
                f.write("   \n")


def test_fast_matrix_market_loader_matches_the_reference_loader(tmp_path, best_oracle, monkeypatch):
    """The multi-threaded loader (csrc/host/mmio.cpp) builds exactly the CSR arrays of the
    reference's loader (sparse.cpp:172-291): symmetric files in shuffled order with blank and
    comment lines, general files that get symmetrised, a file with duplicate entries, several
    thread counts (pieces are cut at line ends)."""
    n, rp, ci, va = M.parsec_like(radius=9.0, n_atoms=6)            # 3k rows, 250k entries
    rows = np.repeat(np.arange(n), np.diff(rp))
    low = ci <= rows
    sym = tmp_path / "sym.mtx"
    _write_mm(sym, n, rows[low], ci[low], va[low], shuffle=3)
    gen = tmp_path / "gen.mtx"
    noisy = va * (1.0 + 1e-14 * np.random.default_rng(1).standard_normal(len(va)))
    _write_mm(gen, n, rows, ci, noisy, symmetry="general", shuffle=4)
    dup = tmp_path / "dup.mtx"
    k = low.nonzero()[0]
    _write_mm(dup, n, np.concatenate([rows[k], rows[k[:50]]]), np.concatenate([ci[k], ci[k[:50]]]),
              np.concatenate([va[k], 0.25 * va[k[:50]]]), shuffle=5)
    for threads in ("1", "3", "16"):
        monkeypatch.setenv("FLZ_HOST_THREADS", threads)
        for path in (sym, gen, dup):
            got = S.SparseSymMatrix.load_matrix_market(path).csr()
            if best_oracle.kind == "reference":
                want = best_oracle.load_matrix_market(str(path))
                assert all(np.array_equal(x, y) for x, y in zip(got, want[1:])), (path, threads)
        got = S.SparseSymMatrix.load_matrix_market(sym).csr()
        assert np.array_equal(got[0], rp) and np.array_equal(got[1], ci) and np.array_equal(got[2], va)


def test_binary_csr_image_and_cache(tmp_path, monkeypatch):
    n, rp, ci, va = M.random_sparse_sym(300, 0.05, 2)
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    img = tmp_path / "a.flzcsr"
    A.save_binary(img)
    B = S.SparseSymMatrix.load_binary(img)
    assert all(np.array_equal(x, y) for x, y in zip(A.csr(), B.csr()))
    with open(img, "r+b") as f:                      # truncated image
        f.truncate(os.path.getsize(img) - 8)
    with pytest.raises(FlzError):
        S.SparseSymMatrix.load_binary(img)
    # cache of the text loader: keyed by size + mtime of the source
    mtx = tmp_path / "a.mtx"
    A.save_matrix_market(mtx)
    cache = tmp_path / "cache"
    cache.mkdir()
    monkeypatch.setenv("FLZ_MM_CACHE", str(cache))
    first = S.SparseSymMatrix.load_matrix_market(mtx).csr()
    images = list(cache.iterdir())
    assert len(images) == 1 and images[0].name.endswith(".flzcsr")
    again = S.SparseSymMatrix.load_matrix_market(mtx).csr()      # served by the image
    assert all(np.array_equal(x, y) for x, y in zip(first, again))
    # a changed source invalidates the image
    n2, rp2, ci2, va2 = M.random_sparse_sym(300, 0.05, 3)
    S.SparseSymMatrix.from_csr(n2, rp2, ci2, va2).save_matrix_market(mtx)
    os.utime(mtx, ns=(1, 10**18))
    third = S.SparseSymMatrix.load_matrix_market(mtx).csr()
    assert np.array_equal(third[2], va2)


def test_jackson_damping_is_an_opt_in_extension():
    """Default = the reference's undamped coefficients (its degrees, tau cuts and iteration
    counts depend on them); the Jackson factors are a host-side option.  Known properties of the
    kernel: g_0 = 1, strictly decreasing to ~0, and the damped indicator series stays inside
    [0, 1] (no Gibbs overshoot) while the undamped one does not."""
    m = 80
    g = S.jackson_factors(m)
    assert len(g) == m + 1 and abs(g[0] - 1.0) < 1e-15
    assert np.all(np.diff(g) < 0) and 0 <= g[-1] < 2e-3
    N = m + 1.0
    k = np.arange(m + 1)
    q = np.pi / (N + 1)
    want = ((N - k + 1) * np.cos(q * k) + np.sin(q * k) / np.tan(q)) / (N + 1)
    assert np.abs(g - want).max() < 1e-15
    cf = S.indicator_coefficients(0.1, 0.3, m)
    t = np.linspace(-1, 1, 2001)
    plain = np.array([S.clenshaw(cf, x) for x in t])
    damped = np.array([S.clenshaw(cf * g, x) for x in t])
    assert plain.min() < -0.02 and plain.max() > 1.02          # Gibbs oscillations
    assert damped.min() > -1e-12 and damped.max() < 1.0 + 1e-12
    assert S.LanczosConfig().jackson_damping == 0


@pytest.mark.parametrize("threads", ["1", "5"])
def test_symmetry_check_reports_what_the_reference_reports(threads, best_oracle):
    """The threaded cursor-per-row symmetry check (matrix.cpp) accepts and rejects the same
    matrices as the reference's binary search per upper entry (sparse.cpp:65-83), with the
    same message: the FIRST offending upper entry in row-major order.  Lower entries without
    an upper partner are not looked up by either."""
    import subprocess, sys, json
    code = r'''
import sys, json
sys.path.insert(0, %r)
import numpy as np, scipy.sparse as sp
from paper_2409_15053_b200 import FlzError, matrices as M, solver as S
n, rp, ci, va = M.laplacian2d(150)          # n = 22 500: several worker ranges
A = sp.csr_matrix((va, ci, rp), shape=(n, n)).tolil()
def attempt(edits):
    B = A.copy()
    for i, j, v in edits:
        B[i, j] = v
    B = B.tocsr(); B.eliminate_zeros(); B.sort_indices()
    try:
        S.SparseSymMatrix.from_csr(n, B.indptr.astype(np.int64), B.indices.astype(np.int32), B.data)
        return "ok"
    except FlzError as e:
        return str(e)
out = {
  "clean": attempt([]),
  "lower_only": attempt([(9000, 17, 2.5), (22499, 3, 1.0)]),        # extra LOWER entries: accepted
  "missing_mirror": attempt([(20000, 20001, 0.0)]),                  # upper (20000,20001) has no... deleted upper: lower left alone
  "structural": attempt([(20001, 20000, 0.0)]),                      # mirror of upper (20000, 20001) deleted
  "numerical": attempt([(151, 1, -1.25)]),                           # mirror of upper (1, 151) differs
  "two": attempt([(22000, 21999, 0.0), (4001, 4000, 7.0), (13000, 12999, 0.0)]),
  "far_upper": attempt([(5, 22000, 3.0)]),                           # upper entry without a mirror
}
print(json.dumps(out))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FLZ_HOST_THREADS=threads)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    got = json.loads(p.stdout.strip().splitlines()[-1])
    assert got["clean"] == "ok" and got["lower_only"] == "ok" and got["missing_mirror"] == "ok"
    assert "structurally asymmetric at (20000,20001)" in got["structural"]
    assert "numerically asymmetric at (1,151)" in got["numerical"]
    assert "numerically asymmetric at (4000,4001)" in got["two"]
    assert "structurally asymmetric at (5,22000)" in got["far_upper"]
