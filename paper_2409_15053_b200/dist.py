"""Row-partition helpers for the multi-GPU path (one process per GPU).

``HaloPlan`` wraps the host-only ``flz_plan_*`` entry points: the code flz_matrix_upload runs
before it touches the GPU (SELL-32-sigma layout of the local rows, halo slots, per-peer need /
give lists, interior / boundary slices).  It exists so that the N>1 logic is testable on CPUs
(tests/test_dist_plan.py, gloo) — it performs no arithmetic of the hot path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib


def uniform_starts(n: int, nranks: int) -> np.ndarray:
    """Contiguous row blocks: rank p owns [n*p//P, n*(p+1)//P) — the split the C++ facade uses."""
    return np.array([n * p // nranks for p in range(nranks + 1)], dtype=np.int64)


class HaloPlan:
    INFO = ("rows_local", "halo_rows", "slices", "stored", "interior_slices", "boundary_slices",
            "send_rows", "sigma", "nnz_local", "short_rows")

    def __init__(self, n_global, rank, nranks, starts, row_ptr, col_idx, values, sigma=0):
        """row_ptr/col_idx/values: the GLOBAL CSR arrays or this rank's slab with absolute
        offsets (row_ptr[i] indexes col_idx/values directly); col_idx are global ids."""
        self.rank, self.nranks = rank, nranks
        starts = np.ascontiguousarray(starts, np.int64)
        rp = np.ascontiguousarray(row_ptr, np.int64)
        if len(rp) == n_global + 1 and nranks > 1:      # global array given: view of our rows
            rp = np.ascontiguousarray(rp[starts[rank]:starts[rank + 1] + 1])
        self._keep = (rp, np.ascontiguousarray(col_idx, np.int32),
                      np.ascontiguousarray(values, np.float64))
        h = C.c_void_p()
        check(lib().flz_plan_create(n_global, rank, nranks, starts, *self._keep, sigma,
                                    C.byref(h)))
        self.handle = h
        self._refresh()

    def _refresh(self):
        info = np.zeros(10, np.int64)
        check(lib().flz_plan_info(self.handle, info))
        self.info = dict(zip(self.INFO, (int(v) for v in info)))

    def need(self, peer: int) -> np.ndarray:
        cnt = lib().flz_plan_need(self.handle, peer, None)
        out = np.zeros(max(cnt, 1), np.int64)
        lib().flz_plan_need(self.handle, peer, out.ctypes.data_as(C.c_void_p))
        return out[:cnt]

    def set_give(self, peer: int, rows):
        rows = np.ascontiguousarray(rows, np.int64)
        check(lib().flz_plan_set_give(self.handle, peer, len(rows), rows))
        self._refresh()

    def arrays(self):
        i, P = self.info, self.nranks
        a = dict(perm=np.zeros(max(i["rows_local"], 1), np.int32),
                 slice_ptr=np.zeros(i["slices"] + 1, np.int64),
                 slice_len=np.zeros(max(i["slices"], 1), np.int32),
                 row_len=np.zeros(max(i["slices"] * 32, 1), np.int32),
                 col=np.zeros(max(i["stored"], 1), np.int32),
                 val=np.zeros(max(i["stored"], 1), np.float64),
                 interior=np.zeros(max(i["interior_slices"], 1), np.int32),
                 boundary=np.zeros(max(i["boundary_slices"], 1), np.int32),
                 send_rows=np.zeros(max(i["send_rows"], 1), np.int32),
                 give_off=np.zeros(P, np.int64), give_cnt=np.zeros(P, np.int64),
                 need_off=np.zeros(P, np.int64))
        order = ("perm", "slice_ptr", "slice_len", "row_len", "col", "val", "interior", "boundary",
                 "send_rows", "give_off", "give_cnt", "need_off")
        check(lib().flz_plan_arrays(self.handle, *[a[k].ctypes.data_as(C.c_void_p) for k in order]))
        a["perm"] = a["perm"][: i["rows_local"]]
        a["interior"] = a["interior"][: i["interior_slices"]]
        a["boundary"] = a["boundary"][: i["boundary_slices"]]
        a["send_rows"] = a["send_rows"][: i["send_rows"]]
        a["col"], a["val"] = a["col"][: i["stored"]], a["val"][: i["stored"]]
        return a

    def ug_arrays(self):
        """Index-compressed layout (descriptors, values, general columns, uniform offsets,
        rest rows); main slices come first, rest slices (SPLIT mode) after them."""
        sizes = np.zeros(8, np.int64)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        check(lib().flz_plan_ug(self.handle, vp(sizes), None, None, None, None, None))
        desc = np.zeros((max(int(sizes[0]), 1), 16), np.int32)
        val = np.zeros(max(int(sizes[1]), 1), np.float64)
        col = np.zeros(max(int(sizes[2]), 1), np.int32)
        uoff = np.zeros(max(int(sizes[3]), 1), np.int32)
        rest_rows = np.zeros(max(int(sizes[5]) * 32, 1), np.int32)
        check(lib().flz_plan_ug(self.handle, vp(sizes), vp(desc), vp(val), vp(col), vp(uoff),
                                vp(rest_rows)))
        return dict(desc=desc[: int(sizes[0])], val=val, col=col, uoff=uoff,
                    uniform_entries=int(sizes[4]), nrest=int(sizes[5]), split=bool(sizes[6]),
                    rest_interior=int(sizes[7]),
                    rest_rows=rest_rows[: int(sizes[5]) * 32].reshape(-1, 32))

    def ug_product(self, x, which="all"):
        """y = A x evaluated from the index-compressed layout exactly as the fast kernels walk
        it (host-side check of the layout; x is indexed by permuted local row / halo slot).
        which: "all", or ("interior" | "boundary") to evaluate only those main slices together
        with the rest slices that must precede them; returns (y, rows computed)."""
        u = self.ug_arrays()
        a = self.arrays()
        nl = self.info["rows_local"]
        ncols = nl + self.info["halo_rows"]
        nmain = len(u["desc"]) - u["nrest"]
        lanes = np.arange(32)

        def slice_sum(s, rows):
            d = u["desc"][s]
            val_ptr = int(np.array(d[0:2]).view(np.int64)[0])
            col_ptr = int(np.array(d[2:4]).view(np.int64)[0])
            uoff_ptr, nu, ng = int(d[4]), int(d[5]), int(d[6])
            base = 0 if int(d[7]) & 2 else rows       # flag bit 1: absolute shared columns
            nuv = (int(d[7]) >> 16) & 0xff            # uniform-value positions come first
            hdr = (2 * nuv + 15) // 16 * 16 if nu + ng - nuv > 0 else 2 * nuv
            lane_rows = val_ptr + hdr                 # per-lane value rows start here
            acc = np.zeros(32)
            for p in range(nu):
                off = int(u["uoff"][uoff_ptr + p])
                if p < 8:
                    assert off == int(d[8 + p])
                c = np.clip(base + off, 0, ncols - 1)
                if p < nuv:                           # one (value, lane mask) pair
                    value = u["val"][val_ptr + 2 * p]
                    mask = int(u["val"][val_ptr + 2 * p + 1: val_ptr + 2 * p + 2].view(np.uint64)[0])
                    v = np.where((mask >> lanes) & 1, value, 0.0)
                else:
                    q = lane_rows + (p - nuv) * 32
                    v = u["val"][q: q + 32]
                acc += v * x[c]
            for q in range(ng):
                c = u["col"][col_ptr + q * 32: col_ptr + q * 32 + 32]
                k = lane_rows + (nu - nuv + q) * 32
                acc += u["val"][k: k + 32] * x[c]
            return acc

        W = np.zeros(nl + 32)
        if which == "all":
            rest_ids = range(u["nrest"])
            main_ids = range(nmain)
        else:
            ri = u["rest_interior"]
            rest_ids = range(ri) if which == "interior" else range(ri, u["nrest"])
            main_ids = a[which]
        for t in rest_ids:
            rows = u["rest_rows"][t]
            acc = slice_sum(nmain + t, np.where(rows < 0, nl, rows))
            assert not np.any(W[rows[rows >= 0]] != 0)      # a row sits in one rest slice only
            W[rows[rows >= 0]] = acc[rows >= 0]
        y = np.zeros(nmain * 32)
        done = []
        for s in main_ids:
            rows = s * 32 + lanes
            acc = slice_sum(s, rows)
            if u["desc"][s][7] & 1:
                acc += W[np.minimum(rows, nl + 31)]
            y[rows] = acc
            done.extend(r for r in rows if r < nl)
        self._w_rows_used = W
        return (y[:nl], np.array(done, np.int64)) if which != "all" else y[:nl]

    def p2_arrays(self):
        """Paired layout (slices of up to 64 rows, two rows per lane, optional dense section
        per slice), or None when the plan has none."""
        sizes = np.zeros(8, np.int64)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        check(lib().flz_plan_p2(self.handle, vp(sizes), None, None, None, None, None, None))
        if not sizes[0]:
            return None
        ns, npos, nd = int(sizes[1]), int(sizes[2]), int(sizes[4])
        ptr = np.zeros(ns + 1, np.int64)
        col = np.zeros(max(npos * 32, 1), np.int32)
        val = np.zeros(max(npos * 64, 2), np.float64)
        desc = np.zeros((max(ns, 1), 6), np.int64)
        dcol = np.zeros(max(nd, 1), np.int32)
        dval = np.zeros(max(nd * 64, 2), np.float64)
        check(lib().flz_plan_p2(self.handle, vp(sizes), vp(ptr), vp(col), vp(val), vp(desc),
                                vp(dcol), vp(dval)))
        return dict(ptr=ptr, col=col, val=val, slices=ns, positions=npos, interior=int(sizes[3]),
                    desc=desc[:ns], dcol=dcol[:nd], dval=dval[:nd * 64], dense_positions=nd,
                    blocks=int(sizes[5]), dense_entries=int(sizes[6]))

    def hy_arrays(self):
        """Hybrid layout (dense tasks + value-grouped slices, natural row order), or None."""
        sizes = np.zeros(12, np.int64)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        check(lib().flz_plan_hy(self.handle, vp(sizes), *([None] * 9)))
        if not sizes[0]:
            return None
        ns, nt = int(sizes[1]), int(sizes[2])
        nl = self.info["rows_local"]
        slices = np.zeros((max(ns, 1), 6), np.int64)
        tasks = np.zeros((max(nt, 1), 5), np.int64)
        cols = np.zeros(max(int(sizes[3]), 1), np.int32)
        uvval = np.zeros(max(int(sizes[4]), 1), np.float64)
        gval = np.zeros(max(int(sizes[5]), 1), np.float64)
        diag = np.zeros(max(nl, 1), np.float64)
        dcols = np.zeros(max(int(sizes[6]), 1), np.int32)
        dval = np.zeros(max(int(sizes[7]), 1), np.float64)
        sell_rows = np.zeros(max(self.info["slices"] * 32, 1), np.int32)
        check(lib().flz_plan_hy(self.handle, vp(sizes), vp(slices), vp(cols), vp(uvval), vp(gval),
                                vp(diag), vp(tasks), vp(dcols), vp(dval), vp(sell_rows)))
        return dict(slices=slices[:ns], tasks=tasks[:nt], cols=cols, uvval=uvval, gval=gval,
                    diag=diag[:nl], dcols=dcols, dval=dval, nslots=int(sizes[8]),
                    blocks=int(sizes[9]), dense_entries=int(sizes[10]),
                    uv_entries=int(sizes[11]), sell_rows=sell_rows)

    def hy_product(self, x, x_halo=None):
        """y = A x evaluated from the hybrid layout as hybrid_dense_tasks / hybrid_slices walk
        it: the dense tasks leave partial sums in slots, a slice adds its uniform-value
        positions ([position / 4][lane][4] columns), its general positions, the partial slots
        of its rows and the diagonal.  The gather source is [local rows | halo rows | zero row];
        x_halo: the values of the halo rows (order of need()), for row-partitioned plans."""
        hy = self.hy_arrays()
        nl = self.info["rows_local"]
        halo = np.zeros(0) if x_halo is None else np.asarray(x_halo, np.float64)
        assert len(halo) == self.info["halo_rows"]
        xz = np.concatenate([np.asarray(x, np.float64), halo, [0.0]])
        P = np.zeros(hy["nslots"])
        for val_off, col_off, ncols, slot_base, nrows in hy["tasks"]:
            v = hy["dval"][val_off * 32:(val_off + ncols) * 32].reshape(ncols, 32)
            g = xz[hy["dcols"][col_off:col_off + ncols]]
            assert np.all(P[slot_base:slot_base + 32] == 0) and 0 < nrows <= 32
            assert not v[:, nrows:].any()
            P[slot_base:slot_base + 32] = g @ v
        assert not P[:32].any()
        y = np.zeros(nl)
        for s, (col_off, uv_off, g_off, nuv, ng, npart) in enumerate(hy["slices"]):
            assert nuv % 4 == 0 and uv_off % 2 == 0
            acc = np.zeros(32)
            base = col_off * 32
            c = hy["cols"][base:base + nuv * 32].reshape(nuv // 4, 32, 4)
            for p in range(nuv):
                acc += hy["uvval"][uv_off + p] * xz[c[p // 4, :, p % 4]]
            base += nuv * 32
            for p in range(ng):
                acc += hy["gval"][(g_off + p) * 32:(g_off + p + 1) * 32] * xz[hy["cols"][base:base + 32]]
                base += 32
            for p in range(npart):
                acc += P[hy["cols"][base:base + 32]]
                base += 32
            rows = np.arange(s * 32, min(nl, s * 32 + 32))
            y[rows] = acc[:len(rows)] + hy["diag"][rows] * xz[rows]
        return y

    def tile_plan(self):
        """Tile plan of the TMA-staged stencil kernel (flz_plan_tiles), or None."""
        info = np.zeros(30, np.int64)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        check(lib().flz_plan_tiles(self.handle, vp(info), None))
        if not info[1]:
            return None
        pairs = np.zeros(int(info[28]), np.float64)
        check(lib().flz_plan_tiles(self.handle, vp(info), vp(pairs)))
        ns = int(info[1])
        slab = np.zeros(4, np.int64)
        check(lib().flz_plan_tile_slab(self.handle, vp(slab)))
        return dict(tile_rows=int(info[0]), nseg=ns, seg_base=info[2:2 + ns].copy(),
                    seg_len=info[10:10 + ns].copy(), seg_start=info[18:18 + ns].copy(),
                    y1_elems=int(info[26]), own_e=int(info[27]), pairs=pairs,
                    front=int(slab[0]), back=int(slab[1]), tile_a=int(slab[2]),
                    tile_b=int(slab[3]))

    def tile_product(self, x, y_rows=None, x_halo=None, phase=0, poison_halo=False):
        """y = A x evaluated tile by tile as clenshaw_step_stencil_tma does: the runs of x a
        tile's segments reach are staged (clipped to [0, y_rows), zero filled), every position
        reads staged element + row-in-tile, masked by its lane bit.  Row slabs: x_halo holds the
        halo rows in slot order; the runs are pieces of the stored source [local | halo] that
        make up the virtual source [front halo | local | back halo].  phase 1 / 2: only the
        tiles that stage local rows / the others (rows of the other tiles stay NaN);
        poison_halo: the halo rows are NaN (phase 1 must not read them)."""
        G = self.tile_plan()
        u = self.ug_arrays()
        nl = self.info["rows_local"]
        T = G["tile_rows"]
        nh = 0 if x_halo is None else len(x_halo)
        front = G["front"]
        assert front + G["back"] == nh
        y_rows = y_rows or (nl + nh + 31) // 32 * 32
        xs = np.zeros(y_rows)
        xs[:nl] = x
        if nh:
            xs[nl:nl + nh] = np.nan if poison_halo else x_halo
        lo, split, hi = -front, (nl if front > 0 else y_rows), y_rows - front
        words = G["pairs"].view(np.uint64)
        ntiles = len(G["pairs"]) // 16 // (T // 32)
        y = np.full(ntiles * T, np.nan)
        lanes = np.arange(32)
        for t in range(ntiles):
            inner = G["tile_a"] <= t < G["tile_b"]
            if (phase == 1 and not inner) or (phase == 2 and inner):
                continue
            r0 = t * T
            stage = np.full(G["y1_elems"], np.nan)     # unfilled elements must never be read
            for j in range(G["nseg"]):
                g0 = r0 + int(G["seg_base"][j]); g1 = g0 + int(G["seg_len"][j])
                seg = np.zeros(g1 - g0)
                pieces = [(max(g0, 0), min(g1, split), 0),               # local rows
                          (max(g0, lo), min(g1, 0), split - lo),         # front halo rows
                          (max(g0, split), min(g1, hi), front)]          # back halo rows
                for a0, a1, shift in pieces:
                    if a1 > a0:
                        assert a0 % 2 == 0 and a1 % 2 == 0 and (a0 + shift) % 2 == 0
                        seg[a0 - g0:a1 - g0] = xs[a0 + shift:a1 + shift]
                assert g0 % 2 == 0 and len(seg) % 2 == 0 and int(G["seg_start"][j]) % 2 == 0
                stage[int(G["seg_start"][j]):int(G["seg_start"][j]) + len(seg)] = seg
            for w in range(T // 32):
                s = t * (T // 32) + w
                nuv = int(words[s * 16 + 1] >> np.uint64(52)) & 0xf
                acc = np.zeros(32)
                for p in range(8):
                    value = G["pairs"][s * 16 + 2 * p]
                    word = int(words[s * 16 + 2 * p + 1])
                    if p >= nuv:
                        assert value == 0.0 and (word & 0xffffffff) == 0
                    e = ((word >> 32) & 0xfffff) // 8
                    on = ((word & 0xffffffff) >> lanes) & 1
                    acc += np.where(on == 1, value, 0.0) * stage[e + w * 32 + lanes]
                if (int(words[s * 16 + 1]) >> 56) & 1:   # per-lane positions, from "global" x
                    d = u["desc"][s]
                    val_ptr = int(np.array(d[0:2]).view(np.int64)[0])
                    col_ptr = int(np.array(d[2:4]).view(np.int64)[0])
                    nu, ng = int(d[5]), int(d[6])
                    assert nuv == (int(d[7]) >> 16) & 0xff and nu <= 8
                    lane_rows = val_ptr + (2 * nuv + 15) // 16 * 16
                    rows = s * 32 + lanes
                    for p in range(nuv, nu):
                        c = np.clip(rows + int(d[8 + p]), 0, nl + nh - 1)
                        q = lane_rows + (p - nuv) * 32
                        acc += u["val"][q: q + 32] * xs[c]
                    for q in range(ng):
                        c = u["col"][col_ptr + q * 32: col_ptr + q * 32 + 32]
                        k = lane_rows + (nu - nuv + q) * 32
                        acc += u["val"][k: k + 32] * xs[c]
                elif s < len(u["desc"]):
                    d = u["desc"][s]
                    assert int(d[6]) == 0 and int(d[5]) == nuv
                y[s * 32 + lanes] = acc
        return y[:nl]

    def p2_product(self, x):
        """y = A x evaluated from the paired layout as clenshaw_step_p2_tasks walks it: the
        general positions of a slice (one column, two values per lane), then its dense section
        (one shared column per position, two values per lane)."""
        p2 = self.p2_arrays()
        nl = self.info["rows_local"]
        y = np.full(nl, np.nan)
        lanes = np.arange(32)
        for s in range(p2["slices"]):
            gpos, dpos, ng, nd, row0, nrows = (int(v) for v in p2["desc"][s])
            assert gpos == int(p2["ptr"][s]) and 0 < nrows <= 64
            accA, accB = np.zeros(32), np.zeros(32)
            for p in range(gpos, gpos + ng):
                g = x[p2["col"][p * 32: p * 32 + 32]]
                v = p2["val"][p * 64: p * 64 + 64].reshape(32, 2)
                accA += v[:, 0] * g
                accB += v[:, 1] * g
            for p in range(dpos, dpos + nd):
                v = p2["dval"][p * 64: p * 64 + 64].reshape(32, 2)
                g = x[p2["dcol"][p]]
                accA += v[:, 0] * g
                accB += v[:, 1] * g
            ra, rb = row0 + 2 * lanes, row0 + 2 * lanes + 1
            assert np.all(np.isnan(y[ra[ra < row0 + nrows]]))     # every row in one slice only
            y[ra[ra < row0 + nrows]] = accA[ra < row0 + nrows]
            y[rb[rb < row0 + nrows]] = accB[rb < row0 + nrows]
        assert not np.isnan(y).any()
        return y

    def __del__(self):
        try:
            lib().flz_plan_destroy(self.handle)
        except Exception:
            pass
