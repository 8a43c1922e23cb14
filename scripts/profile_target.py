"""Small driver for ncu captures: one solve of a bench workload (optionally degree-capped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_15053_b200.workloads import workloads
from paper_2409_15053_b200 import solver as S

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
max_dim = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = workloads()[name]
n, rp, ci, va = wl["gen"]()
H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=False)
cfg = S.LanczosConfig(max_dim=max_dim, **wl["cfg"])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
want = len(sys.argv) > 4 and sys.argv[4] == "vectors"
for rep in range(reps):
    print(f"--- solve {rep}", file=sys.stderr, flush=True)
    res = S.filtered_lanczos(H, *wl["interval"], cfg, want_vectors=want)
print(name, len(res.eigenvalues), res.stats["block_steps"], res.stats["converged"], res.stats["time_total_s"])
