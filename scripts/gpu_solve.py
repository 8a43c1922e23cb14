"""End-to-end GPU solves vs the reference oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2409_15053_b200 import matrices as M, solver as S

ref = oracle.best()
print("oracle:", ref.kind)

def compare(name, csr, alpha, beta, run_ref=True, **cfgkw):
    n, rp, ci, va = csr
    A = S.SparseSymMatrix.from_csr(n, rp, ci, va)
    t = time.time(); res = S.filtered_lanczos(A, alpha, beta, S.LanczosConfig(**cfgkw)); tg = time.time() - t
    st = res.stats
    print(f"{name}: GPU {len(res.eigenvalues)} eigs conv={st['converged']} blocks={st['block_steps']} m={st['degree']} "
          f"maxres={res.residuals.max() if len(res.residuals) else 0:.2e} wall={tg:.3f}s total={st['time_total_s']:.3f} mv={st['time_mv_s']:.3f} orth={st['time_orth_s']:.3f} "
          f"pre={st['time_preproc_s']:.3f} check={st['time_check_s']:.3f} rec={st['time_recover_s']:.3f} up={st['time_upload_s']:.3f} launches={st['gpu_launches']}")
    if run_ref:
        Ar = ref.matrix_from_csr(n, rp, ci, va)
        t = time.time(); rr = ref.solve(Ar, alpha, beta, oracle.make_config(**cfgkw), want_vectors=False); tr = time.time() - t
        same = len(rr.eigenvalues) == len(res.eigenvalues)
        dev = np.abs(rr.eigenvalues - res.eigenvalues).max() / rr.stats['norm_estimate'] if same and len(rr.eigenvalues) else float('nan')
        print(f"   REF {len(rr.eigenvalues)} eigs conv={rr.stats['converged']} blocks={rr.stats['block_steps']} wall={tr:.3f}s  count-match={same} rel-dev={dev:.2e}  speedup={tr/tg:.1f}x")
    # check eigenvectors
    if res.eigenvectors is not None and len(res.eigenvalues):
        import scipy.sparse as sp
        As = M.csr_to_scipy(n, rp, ci, va)
        V = res.eigenvectors
        R = As @ V - V * res.eigenvalues
        print("   true resid max", np.linalg.norm(R, axis=0).max() / st['norm_estimate'], " ortho", np.abs(V.T @ V - np.eye(V.shape[1])).max())
    return res

compare("diag1..5 r=3", M.diag_matrix([1, 2, 3, 4, 5]), 1.5, 4.5)
compare("diag mult3", M.diag_matrix([1, 2, 2, 2, 3]), 1.5, 2.5)
compare("lap2d30 r=3", M.laplacian2d(30), 3.0, 3.8)
compare("lap2d30 r=1", M.laplacian2d(30), 3.0, 3.8, block_size=1)
compare("rand400", M.random_sparse_sym(400, 0.04, 7), -0.5, 0.5)
compare("lap3d-20 r=3", M.laplacian3d(20), 1.0, 1.2)
res = compare("lap2d-100 [1,1.05] m=50 r=3", M.laplacian2d(100), 1.0, 1.05, degree=50)
ana = M.laplacian2d_eigenvalues(100); ana = ana[(ana >= 1.0) & (ana <= 1.05)]
print("   analytic count", len(ana), "dev", np.abs(ana - res.eigenvalues).max() if len(ana) == len(res.eigenvalues) else None)
res = compare("C1 lap2d-200 [1,1.02] m=50 r=1", M.laplacian2d(200), 1.0, 1.02, run_ref=False, degree=50, block_size=1)
ana = M.laplacian2d_eigenvalues(200); ana = ana[(ana >= 1.0) & (ana <= 1.02)]
print("   analytic count", len(ana), "dev", np.abs(ana - res.eigenvalues).max() if len(ana) == len(res.eigenvalues) else None)
pk = M.parsec_like()
res = compare("parsec [-0.65,-0.3] m=50", pk, -0.65, -0.30, run_ref=False, degree=50)
print("  eigs", res.eigenvalues[:5], "...", res.eigenvalues[-5:])
