"""Multi-GPU host logic on CPUs (no GPU): row partition, halo slots, need/give lists and the
interior/boundary split of flz_matrix_upload, exercised (a) with all ranks simulated in one
process and (b) across two real processes talking over torch.distributed/gloo — the halo
exchange a Clenshaw step performs, with NumPy standing in for the device kernel."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2409_15053_b200 import matrices as M
from paper_2409_15053_b200.dist import HaloPlan, uniform_starts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sell_rows_product(arr, info, slices, y1, R):
    """out[new_row, :] = sum_p val * y1[col] over the given slices (NumPy stand-in for K1)."""
    nl = info["rows_local"]
    out = {}
    for s in slices:
        base, L = arr["slice_ptr"][s], arr["slice_len"][s]
        for lane in range(32):
            row = s * 32 + lane
            if row >= nl:
                continue
            acc = np.zeros(R)
            for p in range(arr["row_len"][row]):
                e = base + p * 32 + lane
                acc += arr["val"][e] * y1[arr["col"][e]]
            assert arr["row_len"][row] <= L
            out[row] = acc
    return out


def run_partitioned_spmv(csr, nranks, R=3, sigma=0, exchange=None):
    """Simulates every rank in this process; returns max |A X - reference|."""
    n, rp, ci, va = csr
    starts = uniform_starts(n, nranks)
    plans = [HaloPlan(n, p, nranks, starts, rp, ci, va, sigma) for p in range(nranks)]
    for p in range(nranks):                                   # need lists -> give lists
        for q in range(nranks):
            if p != q:
                need = plans[p].need(q)
                assert np.all((need >= starts[q]) & (need < starts[q + 1]))
                assert np.all(np.diff(need) > 0)              # sorted unique
                if len(need):
                    plans[q].set_give(p, need)
    X = np.random.default_rng(1).standard_normal((n, R))
    want = M.csr_to_scipy(n, rp, ci, va) @ X
    worst = 0.0
    for p in range(nranks):
        info, arr = plans[p].info, plans[p].arrays()
        nl, nh = info["rows_local"], info["halo_rows"]
        y1 = np.zeros((nl + nh, R))
        y1[:nl] = X[starts[p] + arr["perm"]]                  # device order = permuted rows
        # interior slices must not touch halo slots: they run before the halo arrives
        interior = sell_rows_product(arr, info, arr["interior"], y1, R)
        for s in arr["interior"]:
            L = arr["slice_len"][s]
            cols = arr["col"][arr["slice_ptr"][s]: arr["slice_ptr"][s] + 32 * L]
            assert cols.max(initial=0) < nl
        # halo exchange: every peer packs the rows we asked for, in our need order
        for q in range(nranks):
            if q == p:
                continue
            aq = plans[q].arrays()
            off, cnt = aq["give_off"][p], aq["give_cnt"][p]
            assert cnt == len(plans[p].need(q))
            rows = aq["send_rows"][off: off + cnt]            # permuted local ids on q
            packed = X[starts[q] + aq["perm"][rows]]
            slot0 = arr["need_off"][q]
            y1[nl + slot0: nl + slot0 + cnt] = packed
        boundary = sell_rows_product(arr, info, arr["boundary"], y1, R)
        assert set(interior).isdisjoint(boundary) and len(interior) + len(boundary) == nl
        got = np.zeros((nl, R))
        for row, acc in {**interior, **boundary}.items():
            got[arr["perm"][row]] = acc
        worst = max(worst, np.abs(got - want[starts[p]:starts[p + 1]]).max())
    return worst, plans


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_partitioned_spmv_laplacian3d(nranks):
    csr = M.laplacian3d(12)                                    # z-slab partition, plane halos
    worst, plans = run_partitioned_spmv(csr, nranks)
    assert worst < 1e-12
    if nranks > 1:
        inner = plans[1].info
        assert inner["halo_rows"] == (144 if nranks == 2 else 288) or nranks > 4
        assert inner["boundary_slices"] > 0 and (inner["interior_slices"] > 0 or nranks > 4)


@pytest.mark.parametrize("nranks,sigma", [(2, 0), (3, 64), (4, 1)])
def test_partitioned_spmv_parsec_like(nranks, sigma):
    csr = M.parsec_like(radius=9.0, n_atoms=8)                 # long rows -> sigma sorting
    worst, plans = run_partitioned_spmv(csr, nranks, R=2, sigma=sigma)
    assert worst < 1e-12
    assert sum(p.info["nnz_local"] for p in plans) == len(csr[3])


def test_partition_edge_cases():
    csr = M.random_sparse_sym(50, 0.2, 3)
    worst, plans = run_partitioned_spmv(csr, 7, R=1)           # ragged: 50 rows over 7 ranks
    assert worst < 1e-12
    n, rp, ci, va = M.diag_matrix(np.arange(1.0, 11.0))        # no coupling: no halo at all
    worst, plans = run_partitioned_spmv((n, rp, ci, va), 3, R=1)
    assert worst == 0.0 and all(p.info["halo_rows"] == 0 for p in plans)
    from paper_2409_15053_b200 import FlzError
    with pytest.raises(FlzError):
        HaloPlan(n, 0, 2, [0, 7, 9], rp, ci, va)               # ranges do not cover [0, n)
    p0 = HaloPlan(n, 0, 2, [0, 5, 10], rp, ci, va)
    with pytest.raises(FlzError):
        p0.set_give(1, [7])                                    # row 7 is not ours


WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np
import torch.distributed as dist
from paper_2409_15053_b200 import matrices as M
from paper_2409_15053_b200.dist import HaloPlan, uniform_starts

dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]),
                        world_size=2)
rank, world = dist.get_rank(), dist.get_world_size()
n, rp, ci, va = M.laplacian3d(10)
starts = uniform_starts(n, world)
b, e = starts[rank], starts[rank + 1]
plan = HaloPlan(n, rank, world, starts, rp, ci, va)
# 1. need lists travel to the owners (the NCCL send/recv of flz_matrix_upload)
needs = [None] * world
dist.all_gather_object(needs, [plan.need(q) for q in range(world)])
for q in range(world):
    if q != rank and len(needs[q][rank]):
        plan.set_give(q, needs[q][rank])
info, arr = plan.info, plan.arrays()
nl, nh, R = info["rows_local"], info["halo_rows"], 3
# 2. three Clenshaw-like steps y <- A y, each with a halo exchange of the interleaved block
X = np.random.default_rng(5).standard_normal((n, R))
y_loc = X[b + arr["perm"]].copy()
ref = X.copy()
A = M.csr_to_scipy(n, rp, ci, va)
for step in range(3):
    y1 = np.zeros((nl + nh, R))
    y1[:nl] = y_loc
    send = [None] * world
    for q in range(world):
        if q != rank:
            off, cnt = arr["give_off"][q], arr["give_cnt"][q]
            send[q] = y_loc[arr["send_rows"][off: off + cnt]]       # pack_rows_kernel
    gathered = [None] * world
    dist.all_gather_object(gathered, send)
    for q in range(world):
        if q != rank:
            blk = gathered[q][rank]
            y1[nl + arr["need_off"][q]: nl + arr["need_off"][q] + len(blk)] = blk
    out = np.zeros((nl, R))
    for s in list(arr["interior"]) + list(arr["boundary"]):
        base = arr["slice_ptr"][s]
        for lane in range(32):
            row = s * 32 + lane
            if row < nl:
                for p in range(arr["row_len"][row]):
                    idx = base + p * 32 + lane
                    out[row] += arr["val"][idx] * y1[arr["col"][idx]]
    y_loc = out
    ref = A @ ref
got = np.zeros((nl, R)); got[arr["perm"]] = y_loc
err = np.abs(got - ref[b:e]).max() / np.abs(ref).max()
# 3. the all-reduced dot products of the orthogonalization: local partial sums add up
part = np.array([np.sum(got * ref[b:e])])
import torch
t = torch.from_numpy(part); dist.all_reduce(t)
tot = float(np.sum(ref * ref))
assert err < 1e-13, err
assert abs(t.item() - tot) <= 1e-12 * tot
assert info["halo_rows"] == 100 and info["boundary_slices"] > 0
print("rank", rank, "ok", err)
dist.destroy_process_group()
"""


def test_two_process_gloo_halo_exchange(tmp_path):
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT, port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{out}"
        assert f"rank {r} ok" in out
