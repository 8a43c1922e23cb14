"""Finds an interval of the C4-shaped synthetic Hamiltonian that holds ~200 eigenvalues."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import matrices as M, solver as S
n, rp, ci, va = M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2)
H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=False)
lo, hi = S.estimate_spectral_bounds(H)
print("bounds", lo, hi, flush=True)
for a, b, m in ((3.0, 9.0, 200), (3.0, 10.0, 200), (3.0, 10.0, 400)):
    t = time.time()
    res = S.filtered_lanczos(H, a, b, S.LanczosConfig(block_size=3, degree=m), want_vectors=False)
    print(f"[{a},{b}] m={m}: {len(res.eigenvalues)} eigs conv={res.stats['converged']} blocks={res.stats['block_steps']} "
          f"t={time.time()-t:.2f}s first {res.eigenvalues[:3]} last {res.eigenvalues[-3:]}", flush=True)
