"""One end-to-end iteration of bench.py's e2e arm with FLZ_TRACE phase timings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200.workloads import workloads
from paper_2409_15053_b200 import solver as S, Context
ctx = Context.default()
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = workloads()[name]
n, rp, ci, va = wl["gen"]()
cfg = S.LanczosConfig(**wl["cfg"])
for rep in range(3):
    ctx.flush_l2(); ctx.sync()
    print(f"--- e2e iteration {rep}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=True)
    t1 = time.perf_counter()
    res = S.filtered_lanczos(H, *wl["interval"], cfg, want_vectors=True)
    _ = float(res.eigenvalues.sum())
    ctx.sync()
    t2 = time.perf_counter()
    del H
    t3 = time.perf_counter()
    print(f"{name} rep{rep}: from_csr {1e3*(t1-t0):.0f} ms, solve call {1e3*(t2-t1):.0f} ms (stats total {1e3*res.stats['time_total_s']:.0f}, upload {1e3*res.stats['time_upload_s']:.0f}), del {1e3*(t3-t2):.0f} ms", flush=True)
