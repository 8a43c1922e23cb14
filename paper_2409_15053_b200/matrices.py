"""Synthetic symmetric test matrices of the shapes BASELINE.json names.

All generators return ``(n, row_ptr int64, col_idx int32, values f64)`` — the CSR arrays
of speig::SparseSymMatrix (sparse.hpp:28-33) — with sorted columns and EXACT symmetry
(the reference rejects anything else, sparse.cpp:65-83).  Host-side input builders only:
nothing here is on the measured path.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _to_csr(A):
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    return (A.shape[0], A.indptr.astype(np.int64), A.indices.astype(np.int32),
            A.data.astype(np.float64))


def from_upper(n, rows, cols, vals, diag):
    """Exactly symmetric CSR from strictly-upper triplets + a diagonal."""
    U = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    U.sum_duplicates()
    A = U + U.T + sp.diags(diag, format="csr")
    return _to_csr(A)


def laplacian2d(grid: int):
    """5-point Laplacian, Dirichlet, idx = i*grid + j — same matrix as the reference's test
    oracle ``laplacian2d`` (tests/support/oracles.cpp:153-173); nnz = 5n - 4*grid."""
    g = grid
    T = sp.diags([-np.ones(g - 1), 2 * np.ones(g), -np.ones(g - 1)], [-1, 0, 1])
    I = sp.identity(g)
    return _to_csr(sp.kron(I, T) + sp.kron(T, I))


def laplacian2d_eigenvalues(grid: int):
    """Analytic spectrum (oracles.cpp:175-185), ascending."""
    t = 2.0 * (1.0 - np.cos(np.arange(1, grid + 1) * np.pi / (grid + 1)))
    return np.sort((t[:, None] + t[None, :]).ravel())


def laplacian3d(grid: int, weights=(1.0, 1.0, 1.0)):
    """7-point Laplacian on grid^3, Dirichlet, idx = i + g*j + g^2*k.
    ``weights`` de-symmetrises the stencil (anisotropic) to obtain a simple spectrum."""
    g = grid
    T = sp.diags([-np.ones(g - 1), 2 * np.ones(g), -np.ones(g - 1)], [-1, 0, 1])
    I = sp.identity(g)
    wx, wy, wz = weights
    A = (wx * sp.kron(I, sp.kron(I, T)) + wy * sp.kron(I, sp.kron(T, I)) +
         wz * sp.kron(T, sp.kron(I, I)))
    return _to_csr(A)


def laplacian3d_rows(grid: int, row_begin: int, row_end: int):
    """Rows [row_begin,row_end) of laplacian3d(grid) without forming the whole matrix
    (C5: 27M rows split over ranks).  row_ptr starts at 0, columns are global."""
    g = grid
    idx = np.arange(row_begin, row_end, dtype=np.int64)
    i, j, k = idx % g, (idx // g) % g, idx // (g * g)
    cols, vals = [], []
    for off, ok in ((-g * g, k > 0), (-g, j > 0), (-1, i > 0), (0, np.ones_like(i, bool)),
                    (1, i < g - 1), (g, j < g - 1), (g * g, k < g - 1)):
        cols.append(np.where(ok, idx + off, -1))
        vals.append(np.where(ok, 6.0 if off == 0 else -1.0, 0.0))
    cols = np.stack(cols, 1)
    vals = np.stack(vals, 1)
    mask = cols >= 0
    row_ptr = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
    return g ** 3, row_ptr, cols[mask].astype(np.int32), vals[mask]


def laplacian3d_eigenvalues_in(grid: int, lo: float, hi: float):
    """Analytic eigenvalues of laplacian3d(grid) inside [lo, hi], ascending."""
    t = 2.0 * (1.0 - np.cos(np.arange(1, grid + 1) * np.pi / (grid + 1)))
    out = []
    for a in t:
        if a > hi:
            break
        s = a + t[:, None] + t[None, :]
        out.append(s[(s >= lo) & (s <= hi)])
    return np.sort(np.concatenate(out)) if out else np.zeros(0)


def laplacian3d_lowest(grid: int, about: int):
    """(upper, count): an interval end in the widest gap near the `about` lowest eigenvalues of
    laplacian3d(grid), and the exact number of eigenvalues below it."""
    t = 2.0 * (1.0 - np.cos(np.arange(1, grid + 1) * np.pi / (grid + 1)))
    m = min(grid, 64)
    s = np.sort((t[:m, None, None] + t[None, :m, None] + t[None, None, :m]).ravel())
    gaps = np.diff(s[about - 20:about + 20])
    count = about - 20 + int(np.argmax(gaps)) + 1
    return 0.5 * (s[count - 1] + s[count]), count


def diag_matrix(values):
    n = len(values)
    return (n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
            np.asarray(values, np.float64))


def random_sparse_sym(n: int, density: float, seed: int):
    """Symmetric sparse matrix, entries in [-1,1], full diagonal (shape of the reference's
    ``random_sparse_sym`` oracle, oracles.cpp:194-209; not the same random stream)."""
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    keep = rng.random(len(iu[0])) < density
    rows, cols = iu[0][keep], iu[1][keep]
    vals = rng.uniform(-1, 1, len(rows))
    return from_upper(n, rows, cols, vals, rng.uniform(-1, 1, n))


# 12th-order central second-derivative weights (offset 0..6)
_FD12 = np.array([-5369 / 1800, 12 / 7, -15 / 56, 10 / 189, -1 / 112, 2 / 1925, -1 / 16632])


def stencil3d(grid: int, h: float = 0.567, potential=None, seed: int = 1):
    """-1/2 Laplacian with the 12th-order stencil (radius 6 per axis, 37 points) on the full
    grid^3 box (Dirichlet, x fastest) plus an optional random local potential: the kinetic
    part of a PARSEC Hamiltonian without the non-local blocks — every row has the same 37
    diagonal offsets (fewer at the faces)."""
    g = grid
    kin = -0.5 / (h * h)
    offs = np.arange(-6, 7)
    T = sp.diags([np.full(g - abs(k), kin * _FD12[abs(k)]) for k in offs], offs)
    I = sp.identity(g)
    A = sp.kron(I, sp.kron(I, T)) + sp.kron(I, sp.kron(T, I)) + sp.kron(T, sp.kron(I, I))
    if potential is not None:
        rng = np.random.default_rng(seed)
        A = A + sp.diags(rng.uniform(potential[0], potential[1], g ** 3))
    return _to_csr(A)


def parsec_like(radius: float = 30.0, h: float = 0.567, n_atoms: int = 199,
                ball_radius: float = 3.25, v_range=(-1.2, 0.3), nonlocal_strength: float = 0.35,
                seed: int = 1):
    """PARSEC-shaped real-space Hamiltonian.

    Grid points inside a sphere of ``radius`` grid units (natural x-fastest order),
    -1/2 Laplacian with a 12th-order stencil (radius 6 per axis, 37 points), a random
    local potential on the diagonal and ``n_atoms`` dense "non-local projector" blocks
    supported on balls of ``ball_radius`` grid units around random atom positions.
    Defaults give n = 113 081, ~75 nnz/row, spectrum ~[-1.2, 33] (Ge99H100-like);
    ``parsec_like(radius=40, h=0.0903, n_atoms=154, ball_radius=3.86)`` is Ga41As41H72-like.
    """
    rng = np.random.default_rng(seed)
    R = int(np.ceil(radius))
    ax = np.arange(-R, R + 1)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")  # x fastest in memory
    inside = (X * X + Y * Y + Z * Z) < radius * radius
    n = int(inside.sum())
    ident = -np.ones(inside.shape, dtype=np.int64)
    ident[inside] = np.arange(n)
    px, py, pz = X[inside], Y[inside], Z[inside]

    rows, cols, vals = [], [], []
    kin = -0.5 / (h * h)
    L = 2 * R + 1
    for axis, (dz, dy, dx) in enumerate(((0, 0, 1), (0, 1, 0), (1, 0, 0))):
        for k in range(1, 7):
            zi, yi, xi = pz + R + k * dz, py + R + k * dy, px + R + k * dx
            ok = (zi < L) & (yi < L) & (xi < L)
            nb = np.full(n, -1, dtype=np.int64)
            nb[ok] = ident[zi[ok], yi[ok], xi[ok]]
            ok = nb >= 0
            src = np.nonzero(ok)[0]
            rows.append(src)
            cols.append(nb[ok])          # neighbour in +direction has a larger id: upper part
            vals.append(np.full(len(src), kin * _FD12[k]))
    diag = np.full(n, 3 * kin * _FD12[0]) + rng.uniform(v_range[0], v_range[1], n)

    # non-local projectors: w * p p^T on a ball around each atom (upper triangle only)
    atoms = []
    while len(atoms) < n_atoms:
        p = rng.uniform(-radius, radius, 3)
        if p @ p < (radius - ball_radius) ** 2:
            atoms.append(p)
    coords = np.stack([px, py, pz], 1).astype(np.float64)
    for a in atoms:
        d2 = ((coords - a) ** 2).sum(1)
        ball = np.nonzero(d2 < ball_radius * ball_radius)[0]
        if len(ball) < 2:
            continue
        p = np.exp(-d2[ball] / (0.5 * ball_radius * ball_radius))
        p /= np.linalg.norm(p)
        w = nonlocal_strength * rng.uniform(0.5, 1.5) * (1 if rng.random() < 0.7 else -1)
        blk = w * np.outer(p, p)
        iu = np.triu_indices(len(ball), 1)
        rows.append(ball[iu[0]])
        cols.append(ball[iu[1]])
        vals.append(blk[iu])
        np.add.at(diag, ball, w * p * p)
    return from_upper(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), diag)


def csr_to_scipy(n, row_ptr, col_idx, values):
    return sp.csr_matrix((values, col_idx, row_ptr), shape=(n, n))
