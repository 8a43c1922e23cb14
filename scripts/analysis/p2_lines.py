"""L1 cost model of the paired (P2) layout: distinct 128-byte lines touched by each warp-level
gather of 32-byte block rows (4 rows per line), summed with the matrix-stream wavefronts.
cost(position) = 2.07 * lines + 5 cycles (B300_MICROARCH.md: 2.07 cycles per wavefront inside
one LDG; 4 lines of values + 1 of columns streamed per position)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2409_15053_b200 import matrices as M
from paper_2409_15053_b200.dist import HaloPlan


def model(csr, label):
    n, rp, ci, va = csr
    P = HaloPlan(n, 0, 1, [0, n], rp, ci, va)
    p2 = P.p2_arrays()
    col = p2["col"].reshape(-1, 32)
    lines = np.sort(col // 4, axis=1)
    nl = 1 + (np.diff(lines, axis=1) != 0).sum(1)
    L = np.diff(p2["ptr"])
    cyc = (2.07 * nl + 5).sum()
    print(f"{label}: slices {len(L)} positions {len(nl)} lane-entries/nnz {len(nl) * 32 / len(va):.3f} "
          f"mean lines {nl.mean():.2f} model {cyc / 148 / 1.92e3:.1f} us (perfect balance, 148 SMs)")
    return nl, L


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "c3"
    if which == "c3":
        model(M.parsec_like(ball_radius=3.384), "c3 8.44M")
    elif which == "c3old":
        model(M.parsec_like(), "c3 7.41M")
    else:
        model(M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2), "c4")
