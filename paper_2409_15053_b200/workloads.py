"""The BASELINE.json configurations as named workloads (shared by bench.py, the full-size
parity tests and tests/golden/make_golden_fullsize.py so that all three use the same matrix,
interval and solver options).  Host-side input builders only; nothing here is measured.

Keys of a workload: ``desc`` text, ``gen()`` -> (n, row_ptr, col_idx, values), ``interval``,
``cfg`` (LanczosConfig keyword arguments, identical for the reference and this build),
``expect`` (eigenvalue count in the interval — analytic for the Laplacians, from the compiled
reference's own solve for the PARSEC shapes: tests/golden/fullsize_*.npz) and, for the
row-partitioned case, ``gen_rows(b, e)`` / ``n``.
"""
from __future__ import annotations

from . import matrices as M


def workloads():
    c5_hi, c5_count = M.laplacian3d_lowest(300, 285)
    return {
        # BASELINE.json configs[0]: the reference's own CPU-runnable case
        "c1": dict(desc="2D Laplacian 5-point 200x200 (n=40k), [1.00,1.02], degree 50, block 1",
                   gen=lambda: M.laplacian2d(200), interval=(1.00, 1.02),
                   cfg=dict(block_size=1, degree=50), expect=80),
        # configs[1]
        "c2": dict(desc="3D Laplacian 7-point 100^3 (n=1M), [0.10,0.11] (82 eigenpairs), block 3, "
                        "auto degree (clamps at 1000)",
                   gen=lambda: M.laplacian3d(100), interval=(0.10, 0.11), cfg=dict(block_size=3),
                   expect=82),
        # configs[2]: PARSEC-shaped Ge99H100-like Hamiltonian — the configuration north_star's
        # 1-GPU targets are quoted on.  ball_radius 3.384 gives Ge99H100's nonzero count
        # (8 444 471 vs 8 451 395); the interval ends sit in the two widest gaps around the
        # lowest ~250 eigenvalues (scripts/explore_c3.py).
        "c3": dict(desc="synthetic PARSEC-shaped Hamiltonian (Ge99H100-like, n~113k, 8.44M nnz, "
                        "74.8 nnz/row), lowest 247 eigenpairs, degree 50, block 3",
                   gen=lambda: M.parsec_like(ball_radius=3.384), interval=(-0.65, -0.0034),
                   cfg=dict(block_size=3, degree=50), expect=247),
        # configs[3]: Ga41As41H72-shaped
        "c4": dict(desc="synthetic Ga41As41H72-shaped Hamiltonian (n~268k, ~65 nnz/row, spectrum "
                        "[-0.06, 1300]), [3.0,10.0] (208 eigenpairs), degree 200, block 3",
                   gen=lambda: M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86,
                                             seed=2),
                   interval=(3.0, 10.0), cfg=dict(block_size=3, degree=200), expect=208),
        # configs[4]: row-partitioned 27M-row Laplacian (2/4/8 GPUs; does not fit one GPU:
        # 216 MB per basis vector).  RE-SCOPED against BASELINE.json's "500 eigenpairs": max_dim
        # is fixed so that the 2-GPU basis fits (97 GB/GPU) and is identical at every GPU count.
        # With 900 basis vectors and the reference's degree cap (1000) an interior interval of
        # this matrix cannot converge (its filter would need degree ~23000), and 500
        # pairs need ~1400 vectors; the workload is therefore the LOWEST 284 eigenpairs.
        "c5": dict(desc="RE-SCOPED (BASELINE says 500 eigenpairs): 3D Laplacian 7-point 300^3 "
                        "(n=27M) row-partitioned, lowest 284 eigenpairs ([-0.001, %.6f]), block 3, "
                        "auto degree (clamps at 1000), max_dim 900" % c5_hi,
                   gen=lambda: M.laplacian3d(300),
                   gen_rows=lambda b, e: M.laplacian3d_rows(300, b, e),
                   n=27000000, interval=(-0.001, c5_hi),
                   cfg=dict(block_size=3, max_dim=900), expect=c5_count),
        # BASELINE.json's stated C5 variant: lowest ~500 eigenpairs, for 4/8 GPUs only
        # (1500 basis vectors = 81 GB/GPU at 4 GPUs).
        "c5-500": dict(desc="3D Laplacian 7-point 300^3 (n=27M) row-partitioned, lowest ~500 "
                            "eigenpairs, block 3, auto degree (clamps at 1000), max_dim 1500 "
                            "(needs >= 4 GPUs)",
                       gen=lambda: M.laplacian3d(300),
                       gen_rows=lambda b, e: M.laplacian3d_rows(300, b, e),
                       n=27000000, interval=(-0.001, M.laplacian3d_lowest(300, 500)[0]),
                       cfg=dict(block_size=3, max_dim=1500),
                       expect=M.laplacian3d_lowest(300, 500)[1]),
        # small smoke-sized case
        "tiny": dict(desc="2D Laplacian 30x30, [3.0,3.8]", gen=lambda: M.laplacian2d(30),
                     interval=(3.0, 3.8), cfg=dict(), expect=124),
    }


def step_bytes(n, nnz, r):
    """Algorithmic bytes of one fused Clenshaw step."""
    return 12 * nnz + 4 * (n + 1) + 32 * n * r
