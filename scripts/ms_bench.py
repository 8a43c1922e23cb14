"""Several Clenshaw steps per launch (clenshaw_multistep_stencil) against one launch per step on
2-D Laplacians: us per Clenshaw step (CUDA events around 4 filter applications of degree 50).
Run once per setting of FLZ_MS / FLZ_MS_K / FLZ_MS_CORE (read once per process)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S

ctx = Context()
out = {k: os.environ.get(k, "") for k in ("FLZ_MS", "FLZ_MS_K", "FLZ_MS_CORE")}
cases = ((200, 1), (200, 3), (500, 1), (500, 3), (1000, 3), (2000, 3))
if len(sys.argv) > 1:
    cases = tuple(tuple(int(v) for v in a.split("x")) for a in sys.argv[1:])
for g, r in cases:
    n, rp, ci, va = M.laplacian2d(g)
    A = DeviceMatrix(ctx, n, rp, ci, va)
    cf = S.indicator_coefficients(-0.3, 0.25, 50)
    X = np.random.default_rng(0).standard_normal((n, r))
    A.filter_bench(cf, 4.0, 4.5, X, reps=1)
    ms, _ = A.filter_bench(cf, 4.0, 4.5, X, reps=4)
    out["lap2d-%d r=%d" % (g, r)] = round(ms / 4 / 50 * 1e3, 2)
print(json.dumps(out))
