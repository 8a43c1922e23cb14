"""The row-partitioned device path on ONE GPU through the loopback transport (csrc/comm.cu).

A gpurun box has one GPU and NCCL refuses two ranks on one device, so the multi-rank device
code — halo packing kernels, halo slots of the planar and the interleaved blocks, interior /
boundary launches fenced by events between the compute and the communication stream, the
all-reduced coefficient blocks of the orthogonalization — is executed here with the ranks as
host threads of this process (one context, one thread per rank) and compared with the
single-context product.  Everything but the transport is the code the NCCL build runs."""
import threading

import numpy as np
import pytest

from paper_2409_15053_b200 import Basis, Context, DeviceMatrix, LoopHub, matrices as M, solver as S

pytestmark = pytest.mark.gpu


def run_ranks(nranks, body):
    """body(rank, ctx) on one thread per rank; returns the per-rank results, re-raises errors."""
    hub = LoopHub(nranks)
    out, err = [None] * nranks, [None] * nranks

    def work(r):
        try:
            ctx = Context.loopback(hub, r)
            out[r] = body(r, ctx)
            ctx.sync()
        except BaseException as e:   # noqa: BLE001 - reported below
            err[r] = e

    threads = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "a rank hangs in the loopback transport"
    for e in err:
        if e is not None:
            raise e
    return out


def slab(csr, b, e):
    n, rp, ci, va = csr
    return rp[b:e + 1] - rp[b], ci[rp[b]:rp[e]], va[rp[b]:rp[e]]


CASES = {
    "lap3d": lambda: M.laplacian3d(24),                                  # planar halo planes
    "aniso": lambda: M.laplacian3d(16, (1.0, 0.5, 0.25)),
    "parsec": lambda: M.parsec_like(radius=10.0, n_atoms=8),            # long rows, wide halo
    "random": lambda: M.random_sparse_sym(3000, 0.004, 3),              # halo from every rank
}


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("r", [1, 3, 4])
@pytest.mark.parametrize("name", list(CASES))
def test_partitioned_filter_matches_single_context(name, nranks, r):
    csr = CASES[name]()
    n, rp, ci, va = csr
    X = np.random.default_rng(5).standard_normal((n, r))
    cf = S.indicator_coefficients(-0.4, 0.1, 24)
    c, e = 3.0, 3.5
    ctx0 = Context()
    A0 = DeviceMatrix(ctx0, n, rp, ci, va)
    ctx0.set_exact(True)
    want_exact = A0.filter_apply(cf, c, e, X)
    want_spmm = A0.spmm(X, counted=False)
    ctx0.set_exact(False)
    want_fast = A0.filter_apply(cf, c, e, X)
    starts = [n * k // nranks for k in range(nranks + 1)]

    def body(rank, ctx):
        b, e_ = starts[rank], starts[rank + 1]
        lrp, lci, lva = slab(csr, b, e_)
        A = DeviceMatrix(ctx, n, lrp, lci, lva, row_begin=b, row_end=e_)
        st = A.stats()
        ctx.set_exact(True)
        ye = A.filter_apply(cf, c, e, X[b:e_])
        ze = A.spmm(X[b:e_], counted=False)
        ctx.set_exact(False)
        yf = A.filter_apply(cf, c, e, X[b:e_])
        return ye, ze, yf, st

    parts = run_ranks(nranks, body)
    got_exact = np.vstack([p[0] for p in parts])
    got_spmm = np.vstack([p[1] for p in parts])
    got_fast = np.vstack([p[2] for p in parts])
    assert sum(p[3]["halo_rows"] for p in parts) > 0 and sum(p[3]["boundary_slices"] for p in parts) > 0
    # exact mode: CSR-order sums per row, so the partitioned result is the same bit for bit
    assert np.array_equal(got_exact, want_exact)
    assert np.array_equal(got_spmm, want_spmm)
    scale = np.abs(want_fast).max()
    assert np.abs(got_fast - want_fast).max() <= 1e-13 * scale
    assert np.abs(got_fast - want_exact).max() <= 1e-12 * scale


@pytest.mark.parametrize("name", ["lap3d", "parsec"])
def test_partitioned_lanczos_steps_match_single_context(name):
    """Block Lanczos steps with full reorthogonalization on two ranks: the all-reduced
    coefficient blocks D_k, S_k and the basis agree with the single-context factorization."""
    csr = CASES[name]()
    n, rp, ci, va = csr
    r, steps = 3, 6
    start = S.init_block(n, r, 20177)
    cf = S.indicator_coefficients(-0.4, 0.1, 16)
    c, e = 3.0, 3.5
    ctx0 = Context()
    A0 = DeviceMatrix(ctx0, n, rp, ci, va)
    B0 = Basis(ctx0, A0, start, 64)
    want = [B0.step(cf, c, e) for _ in range(steps)]
    Q0 = B0.get(0, (steps + 1) * r)
    starts = [0, n // 2, n]

    def body(rank, ctx):
        b, e_ = starts[rank], starts[rank + 1]
        lrp, lci, lva = slab(csr, b, e_)
        A = DeviceMatrix(ctx, n, lrp, lci, lva, row_begin=b, row_end=e_)
        B = Basis(ctx, A, start[b:e_], 64)
        got = [B.step(cf, c, e) for _ in range(steps)]
        return got, B.get(0, (steps + 1) * r), B.ortho_error()

    parts = run_ranks(2, body)
    for k in range(steps):
        for rank in range(2):
            Dk, Sk, scale, dead = parts[rank][0][k]
            assert np.abs(Dk - want[k][0]).max() <= 1e-11 * max(1.0, np.abs(want[k][0]).max())
            assert np.abs(Sk - want[k][1]).max() <= 1e-11 * max(1.0, np.abs(want[k][1]).max())
            assert abs(scale - want[k][2]) <= 1e-12 * want[k][2] and not dead.any()
        # replicated host inputs: both ranks hold identical coefficient blocks
        assert np.array_equal(parts[0][0][k][0], parts[1][0][k][0])
        assert np.array_equal(parts[0][0][k][1], parts[1][0][k][1])
    Q = np.vstack([parts[0][1], parts[1][1]])
    assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() <= 1e-12
    assert np.abs(np.abs(np.sum(Q * Q0, axis=0)) - 1.0).max() <= 1e-9     # same basis vectors
    assert max(parts[0][2], parts[1][2]) <= 1e-12


@pytest.mark.parametrize("nranks", [2, 3])
def test_partitioned_hybrid_layout_matches_single_context(nranks):
    """Stencil + dense-block matrices keep the hybrid layout on row slabs: dense tasks of the
    local diagonal block run while the halo rows travel, the slices read the halo slots behind
    the local rows.  Filter and product agree with the single-context result (exact mode bit
    for bit; fast mode to rounding — the blocks of a slab differ from the global ones)."""
    csr = M.parsec_like(radius=17.0, n_atoms=40)
    n, rp, ci, va = csr
    r = 3
    X = np.random.default_rng(7).standard_normal((n, r))
    cf = S.indicator_coefficients(-0.4, 0.1, 24)
    c, e = 3.0, 3.5
    ctx0 = Context()
    A0 = DeviceMatrix(ctx0, n, rp, ci, va)
    assert "hybrid" in A0.k1_info(r)["kernel"]
    ctx0.set_exact(True)
    want_exact = A0.filter_apply(cf, c, e, X)
    ctx0.set_exact(False)
    want_fast = A0.filter_apply(cf, c, e, X)
    want_spmm = A0.spmm(X, counted=False)
    starts = [n * k // nranks for k in range(nranks + 1)]

    def body(rank, ctx):
        b, e_ = starts[rank], starts[rank + 1]
        lrp, lci, lva = slab(csr, b, e_)
        A = DeviceMatrix(ctx, n, lrp, lci, lva, row_begin=b, row_end=e_)
        kernel = A.k1_info(r)["kernel"]
        ctx.set_exact(True)
        ye = A.filter_apply(cf, c, e, X[b:e_])
        ctx.set_exact(False)
        yf = A.filter_apply(cf, c, e, X[b:e_])
        zf = A.spmm(X[b:e_], counted=False)
        return ye, yf, zf, kernel, A.stats()

    parts = run_ranks(nranks, body)
    # all ranks or none: the halo rows travel in the block layout of the filter workspaces, so
    # a rank whose slab has dense blocks gives the hybrid layout up when another rank's has not
    # (3 ranks here: only the last slab has them)
    kinds = ["hybrid" in p[3] for p in parts]
    assert all(kinds) if nranks == 2 else not any(kinds), [p[3] for p in parts]
    assert sum(p[4]["halo_rows"] for p in parts) > 0
    assert np.array_equal(np.vstack([p[0] for p in parts]), want_exact)
    scale = np.abs(want_fast).max()
    assert np.abs(np.vstack([p[1] for p in parts]) - want_fast).max() <= 1e-13 * scale
    assert np.abs(np.vstack([p[2] for p in parts]) - want_spmm).max() <= 1e-13 * np.abs(want_spmm).max()


SOLVES = {
    # name: (matrix, interval, config keywords, ranks)
    "lap3d": (lambda: M.laplacian3d(24), (1.0, 1.3), dict(block_size=3, degree=40), 2),
    "lap3d x3": (lambda: M.laplacian3d(24), (1.0, 1.3), dict(block_size=3, degree=40), 3),
    "lap2d r1": (lambda: M.laplacian2d(64), (2.0, 2.2), dict(block_size=1, degree=30), 2),
    "parsec": (lambda: M.parsec_like(radius=10.0, n_atoms=8), None, dict(block_size=3, degree=30), 2),
}


@pytest.mark.parametrize("name", list(SOLVES))
def test_partitioned_full_solve_matches_single_context(name):
    """The WHOLE filtered-Lanczos solve (spectral bounds, block steps with all-reduced
    coefficient blocks, replicated convergence checks, Ritz recovery, residuals) on row slabs:
    every rank reports the eigenvalues and residuals of the single-context solve — same count,
    eigenvalues within 1e-10 * ||A||, residuals <= 1e-10, local rows of the eigenvectors
    orthonormal together — and all ranks agree bit for bit (replicated host logic)."""
    gen, interval, kw, nranks = SOLVES[name]
    csr = gen()
    n, rp, ci, va = csr
    cfg = S.LanczosConfig(**kw)
    H0 = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    if interval is None:   # the lowest ~40 eigenvalues of the PARSEC-shaped matrix
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla
        A = sp.csr_matrix((va, ci, rp), shape=(n, n))
        w = np.sort(spla.eigsh(A, k=44, which="SA", return_eigenvectors=False))
        gaps = np.diff(w[30:])
        cut = 30 + int(np.argmax(gaps))
        interval = (float(w[0]) - 0.5, float(0.5 * (w[cut] + w[cut + 1])))
    a, b = interval
    want = S.filtered_lanczos(H0, a, b, cfg)
    assert want.stats["converged"] == 1 and len(want.eigenvalues) > 5
    starts = [n * k // nranks for k in range(nranks + 1)]   # Device::row_range

    def body(rank, ctx):
        ctx.adopt_for_thread()
        try:
            lo, hi = starts[rank], starts[rank + 1]
            lrp, lci, lva = slab(csr, lo, hi)
            H = S.SparseSymMatrix.from_local_rows(n, lo, hi, lrp, lci, lva)
            res = S.filtered_lanczos(H, a, b, cfg)
            return res.eigenvalues.copy(), res.residuals.copy(), np.array(res.eigenvectors), dict(res.stats)
        finally:
            ctx.release_thread()

    parts = run_ranks(nranks, body)
    norm = want.stats["norm_estimate"]
    for ev, rs, vec, st in parts:
        assert st["converged"] == 1
        assert len(ev) == len(want.eigenvalues)
        assert np.abs(ev - want.eigenvalues).max() <= 1e-10 * norm
        assert rs.max() <= 1e-10
        assert np.array_equal(ev, parts[0][0]) and np.array_equal(rs, parts[0][1])
    X = np.vstack([p[2] for p in parts])          # local rows of every rank, stacked
    assert X.shape == (n, len(want.eigenvalues))
    assert np.abs(X.T @ X - np.eye(X.shape[1])).max() <= 1e-10
    import scipy.sparse as sp
    A = sp.csr_matrix((va, ci, rp), shape=(n, n))
    R = A @ X - X * parts[0][0]
    assert np.abs(R).max() <= 1e-9 * norm
