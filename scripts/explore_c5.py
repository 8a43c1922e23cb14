"""Scale model of the C5 choice: lowest ~500 eigenpairs of the 7-point Laplacian (end interval),
degree chosen so that the filter is as blunt relative to the interval as degree 1000 is on the
300^3 grid.  Reports convergence, block steps and time on one GPU."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import matrices as M, solver as S
g = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n, rp, ci, va = M.laplacian3d(g)
H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=False)
t = 2.0 * (1.0 - np.cos(np.arange(1, g + 1) * np.pi / (g + 1)))
s = np.sort((t[:40, None, None] + t[None, :40, None] + t[None, None, :40]).ravel())
def gap_count(k):
    gaps = np.diff(s[k - 20:k + 20]); j = int(np.argmax(gaps)); return k - 20 + j + 1
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 333
for count, degree in ((gap_count(330), deg),):
    hi = 0.5 * (s[count - 1] + s[count])
    t0 = time.time()
    res = S.filtered_lanczos(H, -0.01, hi, S.LanczosConfig(block_size=3, degree=degree, max_dim=900), want_vectors=bool(os.environ.get("WANT_VECTORS")))
    st = res.stats
    ok = len(res.eigenvalues) == count and np.abs(res.eigenvalues - s[:count]).max() < 1e-9
    print(f"g={g} [-0.01,{hi:.5f}] want {count} degree {degree}: got {len(res.eigenvalues)} conv={st['converged']} "
          f"blocks={st['block_steps']} ok={ok} t={time.time()-t0:.1f}s mv={st['time_mv_s']:.1f} orth={st['time_orth_s']:.1f} rec={st['time_recover_s']:.1f}", flush=True)
