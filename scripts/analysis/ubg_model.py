"""Prototype of the SELL-32 'UBG' layout: per slice (<= 32 consecutive rows),
positions are
  U: every lane's column = its row + d        (one int32 per position),
  B: every lane reads the same column         (one int32 per position),
  G: general                                   (one int32 per lane and position).
Main slices are cut adaptively in natural row order where the offset pattern changes; entries
that neither fit U nor a balanced G section spill to a 'rest' matrix whose rows are regrouped
by column extent so that B positions appear.  Reports HBM bytes per Clenshaw step and
modelled L1 wavefronts.  No GPU needed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from collections import Counter
from paper_2409_15053_b200 import matrices as M

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
TU = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5     # U position needs >= TU*h lanes
TB = float(sys.argv[3]) if len(sys.argv) > 3 else 0.6     # B position needs >= TB*h lanes
if name == "c3":
    n, rp, ci, va = M.parsec_like()
elif name == "c4":
    n, rp, ci, va = M.parsec_like(radius=40.0, h=0.0903, n_atoms=154, ball_radius=3.86, seed=2)
elif name == "c2":
    n, rp, ci, va = M.laplacian3d(100)
elif name == "rand":
    n, rp, ci, va = M.random_sparse_sym(4000, 0.01, 3)
else:
    n, rp, ci, va = M.laplacian2d(200)
S = 4
nnz = len(ci)
ci64 = ci.astype(np.int64)

def nlines(cols):
    return len(set((int(c) * S * 8) // 128 for c in cols))

def sectors(h):      # 32-byte sectors of one position's value (or G index) row with h lanes
    return (h + 3) // 4

class Acc:
    def __init__(s): s.bytes = 0; s.steps = 0; s.wave = 0; s.vals = 0; s.slices = 0; s.U = s.B = s.G = 0
A = Acc()

def emit(rows, U, B, G, offsets_of):
    """account one slice. rows: row ids; U: offsets; B: columns; G: per-lane leftover arrays"""
    h = len(rows)
    gmax = max((len(g) for g in G), default=0)
    L = len(U) + len(B) + gmax
    A.slices += 1; A.steps += L; A.vals += L * h
    A.U += len(U); A.B += len(B); A.G += gmax
    A.bytes += L * sectors(h) * 32 + 4 * (len(U) + len(B)) + gmax * ((h * 4 + 31) // 32) * 32 + 32
    w = 0
    for d in U:
        w += max(nlines([r + d for r in rows if d in offsets_of[r]]), 1)
    w += len(B)
    for p in range(gmax):
        w += nlines([g[p] for g in G if p < len(g)])
    w += L * (1 if h <= 16 else 2) + gmax        # value stream (+ index stream for G)
    A.wave += w

# ---- main slices: adaptive cut in natural order
spill = {}
i = 0
while i < n:
    rows = [i]
    base = set((ci64[rp[i]:rp[i + 1]] - i).tolist())
    cnt = Counter(base)
    j = i + 1
    while j < n and len(rows) < 32:
        offs = set((ci64[rp[j]:rp[j + 1]] - j).tolist())
        common = len(offs & base)
        if common < 0.5 * max(len(offs), 1) and common < 0.5 * len(base):
            break
        cnt.update(offs); rows.append(j); j += 1
    h = len(rows)
    offsets_of = {r: set((ci64[rp[r]:rp[r + 1]] - r).tolist()) for r in rows}
    U = sorted(d for d, k in cnt.items() if k >= max(TU * h, 1))
    Uarr = np.array(U, np.int64)
    G = []
    for r in rows:
        c = ci64[rp[r]:rp[r + 1]]
        G.append(c[~np.isin(c - r, Uarr)])
    gmax = max(len(g) for g in G); gsum = sum(len(g) for g in G)
    if gmax > 0 and (gsum < 0.75 * gmax * h and gmax > 2):      # unbalanced leftovers: spill
        for r, g in zip(rows, G):
            if len(g): spill[r] = g
        G = [g[:0] for g in G]
    emit(rows, U, [], G, offsets_of)
    i = j
main = (A.slices, A.steps, A.vals, A.bytes, A.wave, A.U, A.G)
print(f"{name}: n={n} nnz={nnz}")
print(f" main: slices {A.slices} (avg height {n/A.slices:.1f}) positions U {A.U} G {A.G}; stored {A.vals}; "
      f"spilled rows {len(spill)} entries {sum(len(g) for g in spill.values())}")

# ---- rest: group rows by column extent, then length (desc); slices break when the key changes
keys = sorted(spill.items(), key=lambda kv: (int(kv[1][0]), int(kv[1][-1]), -len(kv[1]), kv[0]))
i = 0
r0 = A.slices
while i < len(keys):
    k0 = (int(keys[i][1][0]), int(keys[i][1][-1]))
    grp = [keys[i]]; j = i + 1
    while j < len(keys) and len(grp) < 32:
        kj = (int(keys[j][1][0]), int(keys[j][1][-1]))
        if kj != k0 and len(grp) >= 8: break
        grp.append(keys[j]); j += 1
    i = j
    rows = [r for r, _ in grp]; ents = [g for _, g in grp]
    h = len(rows)
    colc = Counter()
    for c in ents: colc.update(c.tolist())
    B = sorted(c for c, k in colc.items() if k >= max(TB * h, 2))
    Barr = np.array(B, np.int64)
    G = [c[~np.isin(c, Barr)] for c in ents]
    emit(rows, [], B, G, None)
print(f" rest: slices {A.slices - r0} positions B {A.B} G {A.G - main[6]}; stored {A.vals - main[2]}")
r = 3
vec = 32 * n * r
formula = 12 * nnz + 4 * (n + 1) + vec
print(f" total stored values {A.vals} (fill {A.vals/nnz:.3f}); matrix bytes {A.bytes/1e6:.1f} MB (CSR formula {12*nnz/1e6:.1f}); "
      f"step bytes {(A.bytes+vec)/1e6:.1f} MB vs formula {formula/1e6:.1f} MB  -> {100*(A.bytes+vec)/formula:.0f}%")
print(f" warp-steps {A.steps}; modelled L1 wavefronts/SM {A.wave/148:.0f}  ({A.wave/148/1.9e3:.1f} us at 1/clk)")
