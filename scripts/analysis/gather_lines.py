"""Host-side model of K1's L1 wavefronts: distinct 128-byte lines touched per warp-level
gather of the interleaved block (row stride S doubles), for several matrix layouts.
No GPU needed.  Usage: python scripts/analysis/gather_lines.py [c3|c4|c2]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2409_15053_b200 import matrices as M

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
if name == "c3":
    n, rp, ci, va = M.parsec_like()
elif name == "c4":
    n, rp, ci, va = M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2)
else:
    n, rp, ci, va = M.laplacian3d(100)
S = 4 if name != "c2" else 3
ROWS_PER_LINE = 16 // S if S == 4 else None
length = np.diff(rp).astype(np.int64)
nnz = len(ci)
print(f"{name}: n={n} nnz={nnz} nnz/row={nnz/n:.1f} min/max len {length.min()}/{length.max()}")

def line_of(col):
    return (col.astype(np.int64) * S * 8) // 128

def sigma_perm(sigma):
    perm = np.arange(n)
    if sigma > 1:
        for w0 in range(0, n, sigma):
            w1 = min(n, w0 + sigma)
            order = np.argsort(-length[w0:w1], kind="stable")
            perm[w0:w1] = w0 + order
    return perm

def sell_lines(perm, reorder=None, label=""):
    """lane = row; returns total distinct lines summed over (slice, p) and warp-steps."""
    iperm = np.empty(n, np.int64); iperm[perm] = np.arange(n)
    total_lines = 0; steps = 0; stored = 0
    ns = (n + 31) // 32
    for s in range(ns):
        rows = perm[s * 32:(s + 1) * 32]
        L = length[rows].max()
        stored += L * 32
        mat = np.full((len(rows), L), -1, np.int64)
        for l, r in enumerate(rows):
            c = iperm[ci[rp[r]:rp[r + 1]]]
            if reorder is not None:
                c = reorder(iperm[r], c)
            mat[l, :len(c)] = c
        ln = np.where(mat >= 0, (mat * S * 8) // 128, -1)
        for p in range(L):
            u = np.unique(ln[:, p]); total_lines += len(u) - (u[0] == -1)
        steps += L
    print(f"  {label:40s} warp-steps {steps:8d} gather lines {total_lines:9d}  per step {total_lines/steps:5.1f}  "
          f"fill {stored/nnz:.3f}  wavefronts/SM (gather+3/step) {(total_lines+3*steps)/148:8.0f}")
    return total_lines, steps

def csr_vector_lines():
    total = 0; steps = 0
    for r in range(n):
        c = ci[rp[r]:rp[r + 1]]
        ln = line_of(c)
        for q in range(0, len(c), 32):
            total += len(np.unique(ln[q:q + 32])); steps += 1
    print(f"  {'CSR-vector (warp per row), natural order':40s} warp-steps {steps:8d} gather lines {total:9d}  per step {total/steps:5.1f}  "
          f"wavefronts/SM {(total+3*steps)/148:8.0f}")

best_sigma = 4096 if name != "c2" else 1
perm = sigma_perm(best_sigma)
sell_lines(perm, label=f"SELL-32 sigma={best_sigma}, CSR order")
if name != "c2":
    sell_lines(np.arange(n), label="SELL-32 sigma=1 (natural), CSR order")
    # entries ordered by diagonal offset instead of column
    sell_lines(perm, reorder=lambda r, c: c[np.argsort(c - r, kind="stable")], label="sigma sorted, offset order (same as col order)")
    csr_vector_lines()
