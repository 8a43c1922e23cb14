"""Finds an interval of the C3-shaped synthetic Hamiltonian (ball_radius tuned to the Ge99H100
nonzero count, 8.44M) that holds ~250 eigenvalues, with both ends at gap midpoints."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import matrices as M, solver as S
br = float(sys.argv[1]) if len(sys.argv) > 1 else 3.384
n, rp, ci, va = M.parsec_like(ball_radius=br)
print("n", n, "nnz", len(ci), flush=True)
H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=False)
lo, hi = S.estimate_spectral_bounds(H)
print("bounds", lo, hi, flush=True)
t = time.time()
res = S.filtered_lanczos(H, -1.0, 0.15, S.LanczosConfig(block_size=3, degree=50), want_vectors=False)
ev = np.sort(res.eigenvalues)
print(f"{len(ev)} eigs conv={res.stats['converged']} blocks={res.stats['block_steps']} t={time.time()-t:.2f}s")
np.save("gpurun_out/c3_eigs.npy", ev)
gaps = np.diff(ev)
# widest gaps near the 250-eigenvalue mark from a low start
for start in range(0, 6):
    a = ev[start] - 0.5 * (ev[start] - (ev[start - 1] if start else ev[0] - 0.02))
    for cnt in range(240, 262):
        j = start + cnt
        if j < len(ev):
            print(start, cnt, f"a={a:.6f} b={0.5 * (ev[j - 1] + ev[j]):.6f} gap_b={gaps[j - 1]:.2e} "
                  f"gap_a={(ev[start] - ev[start - 1]) if start else 0:.2e}")
