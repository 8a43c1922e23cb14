"""Row-slab K1 on ONE GPU through the loopback transport: time per Clenshaw step of the
100^3 Laplacian split into `nranks` z slabs whose ranks share the device (threads of this
process), tile kernel (default) against the one-warp-per-slice kernel (FLZ_ST_SLAB=0).
The ranks' kernels run side by side on the one GPU, so the figure is the time of the WHOLE
matrix per step with the halo exchange and the phase split in place — comparable with the
single-context 16.4 us, not a per-rank time of a multi-GPU run.

SLAB_SKEW=1: rank 0 owns all planes but two per other rank, so that the other ranks' kernels
are negligible and rank 0's time is that of one rank of a multi-GPU run (halo exchange, phase
split) whose peers answer at once.

  python scripts/slab_k1_bench.py [nranks] [grid] [degree]"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2409_15053_b200 import Context, DeviceMatrix, LoopHub, matrices as M, solver as S


def main():
    nranks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    m = int(sys.argv[3]) if len(sys.argv) > 3 else 400
    n, rp, ci, va = M.laplacian3d(g)
    plane = g * g
    starts = [(g * k // nranks) * plane for k in range(nranks + 1)]
    if os.environ.get("SLAB_SKEW"):     # rank 0 owns all but 2 planes per other rank: its time is
        # the time of ONE rank of a multi-GPU run whose peers answer at once
        starts = [0] + [(g - 2 * (nranks - k)) * plane for k in range(1, nranks)] + [n]
    X = np.random.default_rng(1).standard_normal((n, 3))
    degrees = (m, 3 * m)
    cfs = [S.indicator_coefficients(-0.3, 0.25, d) for d in degrees]
    hub = LoopHub(nranks)
    out = [None] * nranks
    gate = threading.Barrier(nranks)

    def timed(A, ctx, Xl, cf, sync):
        # device time of 3 back-to-back filter applications (CUDA events on the rank's stream)
        best = 1e9
        for _ in range(3):
            sync()
            ms, _ = A.filter_bench(cf, 4.0, 4.5, Xl, reps=3, flush_l2=False)
            sync()
            best = min(best, ms * 1e-3 / 3)
        return best

    def work(rank):
        ctx = Context.loopback(hub, rank)
        b, e = starts[rank], starts[rank + 1]
        A = DeviceMatrix(ctx, n, rp[b:e + 1] - rp[b], ci[rp[b]:rp[e]], va[rp[b]:rp[e]],
                         row_begin=b, row_end=e)
        Xl = np.ascontiguousarray(X[b:e])
        A.filter_apply(cfs[0], 4.0, 4.5, Xl)
        ctx.sync()
        out[rank] = (A.k1_info(3)["kernel"], [timed(A, ctx, Xl, cf, gate.wait) for cf in cfs])

    th = [threading.Thread(target=work, args=(k,)) for k in range(nranks)]
    [t.start() for t in th]
    [t.join() for t in th]
    # one context for comparison
    ctx0 = Context(0)
    A0 = DeviceMatrix(ctx0, n, rp, ci, va)
    A0.filter_apply(cfs[0], 4.0, 4.5, X)
    t1 = [timed(A0, ctx0, X, cf, lambda: None) for cf in cfs]
    # slope between the two degrees: the per-step time without the fixed cost of a call
    # (upload and download of the block, Python)
    slope = lambda t: (t[1] - t[0]) / (degrees[1] - degrees[0]) * 1e6
    print(json.dumps({"nranks": nranks, "grid": g, "degrees": degrees, "kernel": out[0][0],
                      "rank_us_per_step": [round(slope(o[1]), 2) for o in out],
                      "rows": [starts[k + 1] - starts[k] for k in range(nranks)],
                      "one_context_kernel": A0.k1_info(3)["kernel"],
                      "one_context_us_per_step": round(slope(t1), 2),
                      "FLZ_ST_SLAB": os.environ.get("FLZ_ST_SLAB", ""),
                      "FLZ_HALO_DRY": os.environ.get("FLZ_HALO_DRY", "")}))


if __name__ == "__main__":
    main()
