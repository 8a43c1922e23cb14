"""Small driver for ncu captures: one solve of a bench workload (optionally degree-capped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2409_15053_b200 import solver as S

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
max_dim = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = bench.workloads()[name]
n, rp, ci, va = wl["gen"]()
H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=False)
cfg = S.LanczosConfig(max_dim=max_dim, **wl["cfg"])
res = S.filtered_lanczos(H, *wl["interval"], cfg, want_vectors=False)
print(name, len(res.eigenvalues), res.stats["block_steps"], res.stats["converged"], res.stats["time_total_s"])
