"""Where the end-to-end overhead goes: host-side matrix construction and upload, phase by phase
(FLZ_TRACE=1 prints the plan phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200.workloads import workloads
from paper_2409_15053_b200 import solver as S, Context
ctx = Context.default()
for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    wl = workloads()[name]
    n, rp, ci, va = wl["gen"]()
    for rep in range(2):
        t0 = time.perf_counter()
        H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=True)
        t1 = time.perf_counter()
        lay = H.layout()          # forces plan + upload
        ctx.sync()
        t2 = time.perf_counter()
        print(f"{name} rep{rep}: from_csr(check) {1e3*(t1-t0):.1f} ms, plan+upload {1e3*(t2-t1):.1f} ms", flush=True)
        del H
