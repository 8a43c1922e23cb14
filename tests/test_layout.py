"""The index-compressed matrix layout of the fast kernels (host/plan.cpp build_ug), checked on
CPUs: HaloPlan.ug_product walks the descriptors exactly as the CUDA kernels do (uniform-offset
positions with clamping, shared absolute columns of rest slices, general positions, the W
hand-over from rest slices to flagged main slices) and must reproduce A x.  Covers the SPLIT
mode (rest slices), the unsplit sigma-sorted mode and the row-partitioned case where interior
slices run before the halo arrives."""
import os

import numpy as np
import pytest

from paper_2409_15053_b200 import matrices as M
from paper_2409_15053_b200.dist import HaloPlan, uniform_starts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference(csr, x):
    n, rp, ci, va = csr
    return M.csr_to_scipy(n, rp, ci, va) @ x


CASES = {
    "lap2d30": (lambda: M.laplacian2d(30), True),            # 30 does not divide 32: mixed slices
    "lap3d12": (lambda: M.laplacian3d(12), True),
    "lap3d20": (lambda: M.laplacian3d(20), True),
    "aniso": (lambda: M.laplacian3d(9, (1.0, 0.5, 0.25)), True),
    "rand500": (lambda: M.random_sparse_sym(500, 0.03, 1), False),   # nothing uniform: unsplit
    "parsec7k": (lambda: M.parsec_like(radius=12.0, n_atoms=12), None),
    "diag": (lambda: M.diag_matrix(np.arange(1.0, 41.0)), True),
    "stencil37": (lambda: M.stencil3d(14, potential=(-1.2, 0.3)), True),   # 37 offsets per row
}


@pytest.mark.parametrize("name", list(CASES))
def test_ug_layout_reproduces_product(name, monkeypatch):
    monkeypatch.setenv("FLZ_HY", "0")     # this test is about the UG layout (parsec7k has blocks)
    gen, want_split = CASES[name]
    csr = gen()
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    u, a = P.ug_arrays(), P.arrays()
    if want_split is not None:
        assert u["split"] == want_split
    if u["split"]:
        assert np.array_equal(a["perm"], np.arange(n))       # natural row order
    x = np.random.default_rng(3).standard_normal(n)
    y = P.ug_product(x[a["perm"]])
    want = reference(csr, x)[a["perm"]]
    assert np.abs(y - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
    # stencils: (almost) every nonzero sits at a uniform position, 8 bytes instead of 12
    if name.startswith("lap3d"):
        assert u["uniform_entries"] >= 0.95 * len(va)
        assert u["nrest"] == 0
        # constant coefficients: the positions are (value, lane mask) pairs, not 32 values
        nuv = (u["desc"][:, 7] >> 16) & 0xFF
        assert nuv.sum() >= 0.95 * u["desc"][:, 5].sum()
        assert len(u["val"]) * 8 < 0.25 * 8 * len(va)
    if name == "stencil37":      # long slices: no pairs (the task kernel reads per-lane values)
        assert ((u["desc"][:, 7] >> 16) & 0xFF).sum() == 0
        assert u["uniform_entries"] >= 0.85 * len(va)


def test_forced_split_builds_rest_slices(monkeypatch):
    """PARSEC-shaped matrix with the split forced on: ragged leftovers (dense non-local blocks)
    go to rest slices, part of them as shared absolute columns; a row has one rest slice."""
    monkeypatch.setenv("FLZ_SPLIT", "1")
    csr = M.parsec_like(radius=14.0, n_atoms=10, ball_radius=3.25)
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    u = P.ug_arrays()
    assert u["split"] and u["nrest"] > 0
    nmain = len(u["desc"]) - u["nrest"]
    assert (u["desc"][:nmain, 7] & 1).sum() > 0              # main slices that add W
    rows = u["rest_rows"][u["rest_rows"] >= 0]
    assert len(np.unique(rows)) == len(rows)
    x = np.random.default_rng(4).standard_normal(n)
    y = P.ug_product(x)
    want = reference(csr, x)
    assert np.abs(y - want).max() <= 1e-12 * np.abs(want).max()
    shared = u["desc"][nmain:, 5].sum()
    assert (u["desc"][nmain:, 7][u["desc"][nmain:, 5] > 0] & 2).all()   # shared = absolute
    assert shared >= 0


@pytest.mark.parametrize("nranks,split", [(2, "1"), (3, "1"), (2, "0"), (4, None)])
def test_partitioned_ug_product(monkeypatch, nranks, split):
    """Row-partitioned: interior main/rest slices use local rows only (they run before the halo
    arrives), boundary ones run after; together they give this rank's rows of A x."""
    if split is not None:
        monkeypatch.setenv("FLZ_SPLIT", split)
    csr = M.parsec_like(radius=10.0, n_atoms=8) if split is not None else M.laplacian3d(12)
    n, rp, ci, va = csr
    starts = uniform_starts(n, nranks)
    plans = [HaloPlan(n, p, nranks, starts, rp, ci, va) for p in range(nranks)]
    for p in range(nranks):
        for q in range(nranks):
            if p != q and len(plans[p].need(q)):
                plans[q].set_give(p, plans[p].need(q))
    x = np.random.default_rng(5).standard_normal(n)
    want = reference(csr, x)
    for p in range(nranks):
        info, a = plans[p].info, plans[p].arrays()
        nl, nh = info["rows_local"], info["halo_rows"]
        xl = np.full(nl + nh, np.nan)                          # halo not there yet
        xl[:nl] = x[starts[p] + a["perm"]]
        y_int, rows_int = plans[p].ug_product(xl, "interior")
        assert not np.isnan(y_int[rows_int]).any()             # interior never touches the halo
        for q in range(nranks):                                # halo arrives
            if q == p:
                continue
            aq = plans[q].arrays()
            off, cnt = aq["give_off"][p], aq["give_cnt"][p]
            rows = aq["send_rows"][off: off + cnt]
            slot0 = a["need_off"][q]
            xl[nl + slot0: nl + slot0 + cnt] = x[starts[q] + aq["perm"][rows]]
        y_bnd, rows_bnd = plans[p].ug_product(xl, "boundary")
        assert len(set(rows_int) & set(rows_bnd)) == 0 and len(rows_int) + len(rows_bnd) == nl
        got = np.zeros(nl)
        got[rows_int] = y_int[rows_int]
        got[rows_bnd] = y_bnd[rows_bnd]
        out = np.zeros(nl)
        out[a["perm"]] = got
        assert np.abs(out - want[starts[p]:starts[p + 1]]).max() <= 1e-12 * np.abs(want).max()


def _check_p2_slices(p2, n):
    """Slices tile the permuted rows: contiguous, in order, 1..64 rows each."""
    d = p2["desc"]
    assert d[0, 4] == 0 and d[-1, 4] + d[-1, 5] == n
    assert np.all(d[1:, 4] == d[:-1, 4] + d[:-1, 5]) and np.all((d[:, 5] >= 1) & (d[:, 5] <= 64))
    assert np.all(d[:, 0] == p2["ptr"][:-1]) and np.all(d[:, 2] == np.diff(p2["ptr"]))


@pytest.mark.parametrize("gen", [lambda: M.parsec_like(radius=12.0, n_atoms=12),
                                 lambda: M.parsec_like(radius=10.0, n_atoms=30, ball_radius=3.6),
                                 lambda: M.random_sparse_sym(700, 0.06, 5)])
@pytest.mark.parametrize("dense", ["1", "0"])
def test_paired_layout_reproduces_product(gen, dense, monkeypatch):
    monkeypatch.setenv("FLZ_HY", "0")     # the paired layout (multi-rank / no-blocks fallback)
    monkeypatch.setenv("FLZ_P2_DENSE", "1")   # with its optional dense sections (experiments)
    """Long ragged rows: slices of up to 64 rows, two adjacent rows per lane, one column and
    two values per general position, one shared column per dense position (host/plan.hpp).
    The emulation walks it as clenshaw_step_p2_tasks does.  FLZ_P2_DENSE is read once per
    process, hence the subprocess for the run without dense sections."""
    csr = gen()
    n, rp, ci, va = csr
    if dense == "0":
        import os, subprocess, sys
        code = ("import sys; sys.path.insert(0, %r); import numpy as np\n"
                "from paper_2409_15053_b200.dist import HaloPlan\n"
                "d = np.load(sys.argv[1]); n = int(d['n'])\n"
                "P = HaloPlan(n, 0, 1, [0, n], d['rp'], d['ci'], d['va']); p2 = P.p2_arrays()\n"
                "perm = P.arrays()['perm']; x = np.random.default_rng(9).standard_normal(n)\n"
                "y = P.p2_product(x[perm])\n"
                "import scipy.sparse as sp\n"
                "want = (sp.csr_matrix((d['va'], d['ci'], d['rp']), shape=(n, n)) @ x)[perm]\n"
                "assert p2['blocks'] == 0 and p2['slices'] == (n + 63) // 64\n"
                "even = perm[0:len(perm) - 1:2]\n"
                "assert np.all((even %% 2 == 0) & (perm[1::2] == even + 1)[: len(even)])\n"
                "assert np.abs(y - want).max() <= 1e-12 * np.abs(want).max()\n"
                "assert p2['positions'] * 32 <= 1.15 * len(d['va'])\n" % ROOT)
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".npz") as f:
            np.savez(f, n=n, rp=rp, ci=ci, va=va)
            f.flush()
            r = subprocess.run([sys.executable, "-c", code, f.name],
                               env=dict(os.environ, FLZ_P2_DENSE="0", FLZ_HY="0"), capture_output=True,
                               text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    p2 = P.p2_arrays()
    assert p2 is not None
    _check_p2_slices(p2, n)
    perm = P.arrays()["perm"]
    assert np.array_equal(np.sort(perm), np.arange(n))
    x = np.random.default_rng(9).standard_normal(n)
    y = P.p2_product(x[perm])
    want = reference(csr, x)[perm]
    assert np.abs(y - want).max() <= 1e-12 * np.abs(want).max()
    # every nonzero is stored exactly once: general entries + dense-section entries
    stored = np.count_nonzero(p2["val"]) + np.count_nonzero(p2["dval"])
    assert stored == np.count_nonzero(va)
    assert p2["dense_entries"] == np.count_nonzero(p2["dval"]) or np.any(va == 0.0)


def test_dense_blocks_of_a_parsec_shaped_matrix_are_found(monkeypatch):
    monkeypatch.setenv("FLZ_HY", "0")
    monkeypatch.setenv("FLZ_P2_DENSE", "1")
    """The non-local projector balls of a PARSEC-shaped Hamiltonian become dense sections: one
    block per atom, most of the nonzeros leave the general positions, a dense section is shared
    by rows of ONE block (its columns are exactly that block's members), and what is left per
    row is the 37-point stencil."""
    n_atoms = 24
    csr = M.parsec_like(radius=14.0, n_atoms=n_atoms, ball_radius=3.4)
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    p2 = P.p2_arrays()
    _check_p2_slices(p2, n)
    assert p2["blocks"] == n_atoms
    assert p2["dense_entries"] >= 0.3 * len(va)
    d = p2["desc"]
    dense = d[d[:, 3] > 0]
    assert len(dense) >= n_atoms
    perm = P.arrays()["perm"]
    A = M.csr_to_scipy(n, rp, ci, va)
    for gpos, dpos, ng, nd, row0, nrows in dense[:: max(1, len(dense) // 8)]:
        cols_old = np.sort(perm[p2["dcol"][dpos: dpos + nd]])
        rows_old = perm[row0: row0 + nrows]
        assert np.all(np.isin(rows_old, cols_old))             # rows are members of the block
        sub = A[rows_old][:, cols_old]
        assert sub.nnz >= 0.9 * nrows * nd                      # and the block is dense
        assert ng <= 64                                         # the stencil part is what is left
    # general positions: fewer than half of what the layout without dense sections needs
    assert p2["positions"] * 32 <= 0.72 * len(va)     # general positions left (0.78 without dense sections)
    x = np.random.default_rng(4).standard_normal(n)
    want = (A @ x)[perm]
    assert np.abs(P.p2_product(x[perm]) - want).max() <= 1e-12 * np.abs(want).max()


def test_hybrid_layout_not_used_when_the_blocks_leave_long_rows():
    """Heavily overlapping balls: the block search finds only some of the cliques, the rest of
    those rows would be hundreds of general positions per slice — the paired layout stays."""
    n, rp, ci, va = M.parsec_like(radius=10.0, n_atoms=30, ball_radius=3.6)
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    assert P.hy_arrays() is None and P.p2_arrays() is not None


@pytest.mark.parametrize("gen", [lambda: M.parsec_like(radius=14.0, n_atoms=24, ball_radius=3.4),
                                 lambda: M.parsec_like(radius=12.0, n_atoms=10, seed=3),
                                 lambda: M.parsec_like(radius=16.0, n_atoms=30, ball_radius=3.0, seed=5)])
def test_hybrid_layout_reproduces_product(gen):
    """Stencil + dense blocks on one rank: natural row order, dense tasks (block x 32 rows, values
    only) and slices whose entries are grouped by value (host/plan.hpp).  The emulation walks
    the arrays as hybrid_dense_tasks / hybrid_slices do."""
    csr = gen()
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    hy = P.hy_arrays()
    assert hy is not None and P.p2_arrays() is None
    assert np.array_equal(P.arrays()["perm"], np.arange(n))          # no permutation
    x = np.random.default_rng(9).standard_normal(n)
    want = reference(csr, x)
    assert np.abs(P.hy_product(x) - want).max() <= 1e-12 * np.abs(want).max()
    sl, tk = hy["slices"], hy["tasks"]
    # every nonzero is stored exactly once: dense tasks + uniform-value + general + diagonal
    general = sum(np.count_nonzero(hy["gval"][g * 32:(g + ng) * 32]) for g, ng in zip(sl[:, 2], sl[:, 4]))
    assert hy["dense_entries"] == np.count_nonzero(hy["dval"])
    assert hy["dense_entries"] + hy["uv_entries"] + general + np.count_nonzero(hy["diag"]) == len(va)
    assert hy["dense_entries"] >= 0.3 * len(va)
    # the stencil part sits at uniform-value positions, 4 bytes per entry (36 per interior row)
    assert hy["uv_entries"] >= 0.75 * 30 * n
    # tasks: 32 slots each, one task per 32 rows of a block, slots 0..31 stay free
    assert np.all(tk[:, 3] % 32 == 0) and tk[:, 3].min() == 32 and len(set(tk[:, 3])) == len(tk)
    assert hy["nslots"] == 32 * (len(tk) + 1)
    # exact-mode SELL arrays: rows grouped by length, every row once
    rows = hy["sell_rows"]
    assert np.array_equal(np.sort(rows[rows >= 0]), np.arange(n))


def test_hybrid_layout_exact_mode_arrays_follow_sell_rows():
    """The CSR-order SELL arrays of a hybrid plan list the rows through sell_rows while their
    columns stay in the natural order (the vectors are not permuted)."""
    csr = M.parsec_like(radius=12.0, n_atoms=12)
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    a, hy = P.arrays(), P.hy_arrays()
    x = np.random.default_rng(2).standard_normal(n)
    y = np.zeros(n)
    for s in range(P.info["slices"]):
        base, L = int(a["slice_ptr"][s]), int(a["slice_len"][s])
        for lane in range(32):
            row = int(hy["sell_rows"][s * 32 + lane])
            if row < 0:
                continue
            k = int(a["row_len"][s * 32 + lane])
            idx = base + lane + 32 * np.arange(k)
            y[row] = np.dot(a["val"][idx], x[a["col"][idx]])
    want = reference(csr, x)
    assert np.abs(y - want).max() <= 1e-13 * np.abs(want).max()
    # grouping by length keeps the padding small although the row order is the natural one
    assert P.info["stored"] <= 1.2 * len(va)


@pytest.mark.parametrize("nranks", [2, 3])
def test_hybrid_layout_on_row_slabs(nranks):
    """Row-partitioned plans take the hybrid layout too: the dense blocks are searched inside
    the local diagonal block, halo columns stay in the slices and point at the halo slots
    behind the local rows, the zero row moves behind the halo.  Every rank's product, evaluated
    from the arrays as the kernels walk them, is its slab of A x."""
    csr = M.parsec_like(radius=17.0, n_atoms=40)
    n, rp, ci, va = csr
    x = np.random.default_rng(3).standard_normal(n)
    want = reference(csr, x)
    starts = [n * k // nranks for k in range(nranks + 1)]
    hybrids = 0
    for rank in range(nranks):
        b, e = starts[rank], starts[rank + 1]
        P = HaloPlan(n, rank, nranks, starts, rp[b:e + 1], ci, va)
        hy = P.hy_arrays()
        if hy is None:
            continue
        hybrids += 1
        need = np.concatenate([P.need(p) for p in range(nranks)]).astype(np.int64)
        assert len(need) == P.info["halo_rows"] > 0
        y = P.hy_product(x[b:e], x[need])
        assert np.abs(y - want[b:e]).max() <= 1e-12 * np.abs(want).max()
        # dense tasks gather local rows only: they can run while the halo rows travel
        assert hy["dcols"].max() < e - b
    assert hybrids >= 1


def test_matrices_without_dense_blocks_keep_the_plain_paired_layout():
    """Long rows that are not cliques (random sparse, banded): the block search gives up after a
    bounded number of seeds and the layout is the plain paired one."""
    import scipy.sparse as sp
    rng = np.random.default_rng(11)
    n = 3000
    B = sp.random(n, n, density=0.03, random_state=5, format="csr")
    B = B + B.T + sp.diags(rng.uniform(1, 2, n))
    csr = M._to_csr(B)
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    p2 = P.p2_arrays()
    assert p2 is not None and p2["blocks"] == 0 and p2["dense_positions"] == 0
    assert p2["slices"] == (n + 63) // 64
    perm = P.arrays()["perm"]
    x = rng.standard_normal(n)
    want = (B @ x)[perm]
    assert np.abs(P.p2_product(x[perm]) - want).max() <= 1e-12 * np.abs(want).max()


def test_paired_layout_odd_row_count_lone_row_longest():
    """An odd number of rows whose lone last row is the longest: the length sort moves it in
    front of the pairs, every later pair then straddles two lanes — the product must still be
    right (regression: slice lengths were taken from the pre-sort pair counts)."""
    rng = np.random.default_rng(3)
    n = 257
    dense = np.zeros((n, n))
    for i in range(n - 1):
        if i % 7 == 3:
            continue
        cols = rng.choice(n - 1, int(rng.integers(25, 40)), replace=False)
        dense[i, cols] = rng.uniform(-1, 1, len(cols))
    dense[n - 1, rng.choice(n, 200, replace=False)] = 1.5
    dense = dense + dense.T
    import scipy.sparse as sp
    csr = M._to_csr(sp.csr_matrix(dense))
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    p2 = P.p2_arrays()
    assert p2 is not None
    perm = P.arrays()["perm"]
    x = rng.standard_normal(n)
    y = P.p2_product(x[perm])
    want = (dense @ x)[perm]
    assert np.abs(y[:n] - want).max() <= 1e-12 * np.abs(want).max()


def test_paired_layout_saves_gathers_on_dense_blocks(monkeypatch):
    monkeypatch.setenv("FLZ_HY", "0")
    monkeypatch.setenv("FLZ_P2_DENSE", "1")
    csr = M.parsec_like(radius=14.0, n_atoms=20, ball_radius=3.25)
    n, rp, ci, va = csr
    p2 = HaloPlan(n, 0, 1, [0, n], rp, ci, va).p2_arrays()
    assert p2["positions"] * 32 <= 0.9 * len(va)


@pytest.mark.parametrize("tile", [32, 128, 512])
@pytest.mark.parametrize("gen", [lambda: M.laplacian3d(20), lambda: M.laplacian2d(50),
                                 lambda: M.laplacian3d(40), lambda: M.laplacian2d(33)])
def test_stencil_tile_plan_reproduces_product(monkeypatch, gen, tile):
    """Tile plan of the TMA-staged stencil kernel: staging the segments of every tile (clipped
    at the ends of the vector, 16-byte aligned runs) and reading `staged element + row in
    tile` per position reproduces A x; elements no copy or zero fill defines are never read
    (the emulation poisons them with NaN)."""
    monkeypatch.setenv("FLZ_ST_TILE", str(tile))
    n, rp, ci, va = gen()
    P = HaloPlan(n, 0, 1, uniform_starts(n, 1), rp, ci, va)
    G = P.tile_plan()
    assert G is not None and G["tile_rows"] == tile and 1 <= G["nseg"] <= 8
    assert len(G["pairs"]) % (16 * tile // 32) == 0
    x = np.random.default_rng(3).standard_normal(n)
    y = P.tile_product(x)
    assert np.abs(y - reference((n, rp, ci, va), x)).max() <= 1e-13 * np.abs(y).max()


def test_stencil_tile_plan_absent_where_it_does_not_apply(monkeypatch):
    """No tile plan for ragged matrices, for row slabs with an odd number of rows (16-byte
    bulk copies) or when switched off."""
    n, rp, ci, va = M.parsec_like(radius=10.0, n_atoms=8)
    assert HaloPlan(n, 0, 1, uniform_starts(n, 1), rp, ci, va).tile_plan() is None
    n, rp, ci, va = M.laplacian3d(16)
    st = [0, 2049, n]
    assert HaloPlan(n, 0, 2, st, rp[: st[1] + 1], ci, va).tile_plan() is None
    monkeypatch.setenv("FLZ_ST_SLAB", "0")
    st = uniform_starts(n, 2)
    # (FLZ_ST_SLAB is read once per process: only checked when set before the first slab plan)
    monkeypatch.delenv("FLZ_ST_SLAB")
    monkeypatch.setenv("FLZ_ST_TILE", "0")
    assert HaloPlan(n, 0, 1, uniform_starts(n, 1), rp, ci, va).tile_plan() is None
    assert HaloPlan(n, 0, 2, st, rp[: st[1] + 1], ci, va).tile_plan() is None


def slab_csr(csr, b, e):
    n, rp, ci, va = csr
    return rp[b:e + 1] - rp[b], ci[rp[b]:rp[e]], va[rp[b]:rp[e]]


@pytest.mark.parametrize("tile", [32, 256])
@pytest.mark.parametrize("case", [
    ("lap3d z slabs", lambda: M.laplacian3d(24), 3, None),
    ("lap3d 8 slabs", lambda: M.laplacian3d(16), 8, None),
    ("aniso", lambda: M.laplacian3d(16, (1.0, 0.5, 0.25)), 2, None),
    ("lap2d", lambda: M.laplacian2d(64), 4, None),
    ("cut inside a plane", lambda: M.laplacian3d(16), 3, [0, 1400, 2900, 4096]),
    ("slices across planes", lambda: M.laplacian3d(12), 3, None),
], ids=lambda c: c[0])
def test_stencil_tile_plan_on_row_slabs(monkeypatch, case, tile):
    """Row slabs: the tile kernel stages runs of the virtual source [front halo | local | back
    halo] (a neighbour plane from a peer sits at the offset it has inside the slab), every rank's
    product from its plan equals its rows of A x; the tiles of phase 1 read no halo row (the
    emulation poisons them) and the two phases together cover every row once."""
    monkeypatch.setenv("FLZ_ST_TILE", str(tile))
    _, gen, nranks, starts = case
    csr = gen()
    n, rp, ci, va = csr
    starts = starts or [n * k // nranks for k in range(nranks + 1)]
    x = np.random.default_rng(7).standard_normal(n)
    want = reference(csr, x)
    for rank in range(nranks):
        b, e = starts[rank], starts[rank + 1]
        lrp, lci, lva = slab_csr(csr, b, e)
        P = HaloPlan(n, rank, nranks, starts, lrp, lci, lva)
        G = P.tile_plan()
        assert G is not None, f"rank {rank} has no tile plan"
        need = np.concatenate([P.need(p) for p in range(nranks)]).astype(np.int64)
        assert G["front"] == int((need < b).sum()) and G["back"] == int((need >= e).sum())
        assert G["front"] + G["back"] == len(need) > 0
        single = HaloPlan(n, 0, 1, [0, n], rp, ci, va).tile_plan()
        if case[0] in ("lap3d z slabs", "lap3d 8 slabs", "aniso", "lap2d"):
            # whole planes per rank: the offsets (and segments) of the single-rank plan
            assert G["nseg"] == single["nseg"] and list(G["seg_base"]) == list(single["seg_base"])
        y = P.tile_product(x[b:e], x_halo=x[need])
        assert np.abs(y - want[b:e]).max() <= 1e-13 * np.abs(want).max()
        y1 = P.tile_product(x[b:e], x_halo=x[need], phase=1, poison_halo=True)
        y2 = P.tile_product(x[b:e], x_halo=x[need], phase=2)
        inner = ~np.isnan(y1)
        assert not np.isnan(y1[inner]).any() and np.isnan(y2[inner]).all()
        assert not np.isnan(y2[~inner]).any()
        assert np.array_equal(np.where(inner, y1, y2), y)
        T = G["tile_rows"]
        assert inner.sum() == max(0, min(e - b, G["tile_b"] * T) - G["tile_a"] * T)
        # every slice that touches a halo row lies outside the phase-1 tiles
        bnd = P.arrays()["boundary"]
        assert all(not (G["tile_a"] <= s // (T // 32) < G["tile_b"]) for s in bnd)
