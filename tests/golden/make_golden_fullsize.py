"""Full-size golden solves of the BASELINE.json configurations by the UNMODIFIED reference
(oracle/_ref/libspeig_ref.so = /root/reference/proj/src compiled by oracle/Makefile):

    python tests/golden/make_golden_fullsize.py c1 c2 c3 c4        (one process per name)

Each run calls the reference's ``speig::filtered_lanczos`` (lanczos.cpp:659 -> run_solve
:573-655) once on the workload of paper_2409_15053_b200/workloads.py with the same
LanczosConfig the GPU build gets, and writes tests/golden/fullsize_<name>.npz: eigenvalues,
residuals, SolveStats (block steps, degree, matvec counts, time split) and the wall time on
this container's host (one core: the reference is serial).  CPU cost in this container:
c1 ~10 min, c3 ~12 min, c4 ~40 min, c2 ~45 min; c2 needs 24 GB (the reference zero-fills its
whole basis, lanczos.cpp:111).

The `-m gpu` tests tests/test_gpu_fullsize.py compare the CUDA path with these files on the
GPU box, where /root/reference does not exist.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2409_15053_b200.workloads import workloads  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main(names):
    ref = oracle.load("ref")
    assert ref.kind == "reference"
    W = workloads()
    for name in names:
        wl = W[name]
        n, rp, ci, va = wl["gen"]()
        A = ref.matrix_from_csr(n, rp, ci, va)
        a, b = wl["interval"]
        t0 = time.perf_counter()
        res = ref.solve(A, a, b, oracle.make_config(**wl["cfg"]), want_vectors=False)
        wall = time.perf_counter() - t0
        st = res.stats
        keys = sorted(st)
        np.savez_compressed(
            os.path.join(OUT, f"fullsize_{name}.npz"),
            eigenvalues=res.eigenvalues, residuals=res.residuals,
            stat_keys=np.array(keys), stat_values=np.array([float(st[k]) for k in keys]),
            wall_s=np.array([wall]), n=np.array([n]), nnz=np.array([len(va)]),
            interval=np.array([a, b]), backend=np.array([ref.backend()]),
            csr_checksum=np.array([float(np.abs(va).sum()), float(ci.astype(np.int64).sum())]))
        print(name, "eigs", len(res.eigenvalues), "blocks", st["block_steps"], "degree",
              st["degree"], "converged", st["converged"], "max_res",
              float(res.residuals.max()) if len(res.residuals) else 0.0,
              f"wall {wall:.1f} s (mv {st['time_mv_s']:.1f} orth {st['time_orth_s']:.1f})",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3"])
