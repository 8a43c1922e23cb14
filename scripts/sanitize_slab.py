"""compute-sanitizer target: the TMA-staged stencil kernel on ROW SLABS through the loopback
transport (2 and 3 ranks as threads): runs cut into halo / local pieces, tiles behind the
hole, fused halo pack, all column counts; products checked against scipy."""
import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, LoopHub, matrices as M, solver as S

for gen, nranks in ((lambda: M.laplacian3d(24), 3), (lambda: M.laplacian2d(64), 2),
                    (lambda: M.laplacian3d(12), 3)):
    n, rp, ci, va = gen()
    As = M.csr_to_scipy(n, rp, ci, va)
    starts = [n * k // nranks // 2 * 2 for k in range(nranks + 1)]
    cf = S.indicator_coefficients(-0.3, 0.25, 6)
    hub = LoopHub(nranks)
    err = [None] * nranks

    def work(rank):
        try:
            ctx = Context.loopback(hub, rank)
            b, e = starts[rank], starts[rank + 1]
            A = DeviceMatrix(ctx, n, rp[b:e + 1] - rp[b], ci[rp[b]:rp[e]], va[rp[b]:rp[e]],
                             row_begin=b, row_end=e)
            assert A.k1_info(3)["kernel"] == "clenshaw_step_stencil_tma"
            for r in (1, 2, 3, 4):
                X = np.random.default_rng(r).standard_normal((n, r))
                Y = A.filter_apply(cf, 4.0, 4.5, X[b:e])
                Z = A.spmm(X[b:e], counted=False)
                assert np.abs(Z - (As @ X)[b:e]).max() < 1e-12
                assert np.isfinite(Y).all()
            ctx.sync()
        except BaseException as ex:
            err[rank] = ex

    th = [threading.Thread(target=work, args=(k,)) for k in range(nranks)]
    [t.start() for t in th]
    [t.join() for t in th]
    for ex in err:
        if ex is not None:
            raise ex
print("ok")
