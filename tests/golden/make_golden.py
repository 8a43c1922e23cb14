"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libspeig_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

The vectors pin (a) the plain-C restatement oracle/flz_oracle.c and (b) the CUDA path on the
GPU box, where /root/reference does not exist.  Inputs are regenerated from seeds by
paper_2409_15053_b200.matrices (deterministic NumPy generators), outputs are the reference's.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2409_15053_b200 import matrices as M  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ref = oracle.load("ref")
assert ref.kind == "reference"


def block(n, r, seed):
    return np.random.default_rng(seed).standard_normal((n, r))


def main():
    g = {}
    # ---- filter scalars (reference KATs: filter_test.cpp:27-47, :96-99)
    g["coef_m1_m05"] = ref.indicator_coefficients(-1.0, -0.5, 12)
    g["coef_01_03"] = ref.indicator_coefficients(0.1, 0.3, 200)
    g["degrees"] = np.array([ref.select_degree(0.1, 0.3)[0], ref.select_degree(-1.0, -0.5)[0],
                             ref.select_degree(-0.02, 0.02)[0], ref.select_degree(0.3, 0.9, 0.1)[0]])
    g["clenshaw_pts"] = np.linspace(-1, 1, 41)
    g["clenshaw_vals"] = np.array([ref.clenshaw(g["coef_01_03"], t) for t in g["clenshaw_pts"]])
    # ---- start block / bounds
    for backend in ("scalar", "avx2"):
        ref.set_backend(backend)
        g[f"init_block_1000x3_{backend}"] = ref.init_block(1000, 3, 20177)
    # ---- filter apply, both backends, several shapes
    cases = {
        "lap2d30": (M.laplacian2d(30), (-0.02, 8.02), (3.0, 3.8), 0, 3, 11),
        "rand400": (M.random_sparse_sym(400, 0.04, 7), (-12.0, 12.0), (-1.0, 1.0), 64, 4, 12),
        "parsec7k": (M.parsec_like(radius=12.0, n_atoms=12), (-1.5, 34.0), (-0.6, 0.0), 50, 3, 13),
        "lap3d12": (M.laplacian3d(12), (-0.05, 12.05), (2.0, 2.6), 0, 5, 14),
    }
    for name, (csr, (lo, hi), (a, b), deg, r, seed) in cases.items():
        n, rp, ci, va = csr
        A = ref.matrix_from_csr(n, rp, ci, va)
        cf, _, _, _ = ref.build_filter(lo, hi, a, b, deg)
        X = block(n, r, seed)
        for backend in ("scalar", "avx2"):
            ref.set_backend(backend)
            g[f"filter_{name}_{backend}"] = ref.filter_apply(A, cf, lo, hi, X)
        g[f"filter_{name}_coeffs"] = cf
        g[f"filter_{name}_meta"] = np.array([lo, hi, a, b, r, seed], dtype=np.float64)
    ref.set_backend("avx2")
    # ---- factorization: 8 filtered block steps on lap2d(30), r = 3
    n, rp, ci, va = M.laplacian2d(30)
    A = ref.matrix_from_csr(n, rp, ci, va)
    lo, hi = ref.estimate_bounds(A)
    g["lap2d30_bounds"] = np.array([lo, hi])
    cf, _, _, _ = ref.build_filter(lo, hi, 3.0, 3.8)
    F = ref.factorization(A, ref.init_block(n, 3), 300, cf, (lo, hi), (3.0, 3.8))
    F.expand(8)
    Q, D, S, dead = F.get()
    g["fact_lap2d30_Q"], g["fact_lap2d30_D"], g["fact_lap2d30_S"] = Q, D, S
    conv, vals, est, wanted, deadp = F.check(3.0, 3.8)
    g["fact_lap2d30_ritz"], g["fact_lap2d30_est"], g["fact_lap2d30_wanted"] = vals, est, wanted
    # ---- full solves (eigenvalues + residual bound + stats that must agree)
    solves = {
        "lap2d30_r3": (M.laplacian2d(30), 3.0, 3.8, dict()),
        "lap2d30_r1": (M.laplacian2d(30), 3.0, 3.8, dict(block_size=1)),
        "lap2d30_m20": (M.laplacian2d(30), 3.0, 3.8, dict(degree=20)),
        "rand400": (M.random_sparse_sym(400, 0.04, 7), -0.5, 0.5, dict()),
        "lap3d20": (M.laplacian3d(20), 1.0, 1.2, dict()),
        "diag_mult3": (M.diag_matrix([1, 2, 2, 2, 3]), 1.5, 2.5, dict()),
        "diag5": (M.diag_matrix([1, 2, 3, 4, 5]), 1.5, 4.5, dict()),
        "parsec7k": (M.parsec_like(radius=12.0, n_atoms=12), -0.6, 0.0, dict(degree=50)),
    }
    for name, (csr, a, b, kw) in solves.items():
        n, rp, ci, va = csr
        A = ref.matrix_from_csr(n, rp, ci, va)
        res = ref.solve(A, a, b, oracle.make_config(**kw), want_vectors=False)
        g[f"solve_{name}_eigs"] = res.eigenvalues
        g[f"solve_{name}_stats"] = np.array([res.stats["block_steps"], res.stats["degree"],
                                             res.stats["mv_iteration"], res.stats["converged"],
                                             res.stats["norm_estimate"], res.residuals.max()])
        print(name, len(res.eigenvalues), res.stats["block_steps"], res.stats["degree"])
    np.savez_compressed(os.path.join(OUT, "reference_vectors.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_vectors.npz"),
          os.path.getsize(os.path.join(OUT, "reference_vectors.npz")) >> 10, "KiB")


if __name__ == "__main__":
    main()
