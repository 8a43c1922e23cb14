"""One short filter application on a bench shape (ncu target): python scripts/k1_one.py c3|c4|c2 [degree]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, solver as S
from paper_2409_15053_b200.workloads import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n, rp, ci, va = workloads()[name]["gen"]()
ctx = Context()
A = DeviceMatrix(ctx, n, rp, ci, va)
cf = S.indicator_coefficients(-0.3, -0.25, m)
X = np.random.default_rng(0).standard_normal((n, 3))
A.filter_bench(cf, 1.0, 2.0, X, reps=2)          # warm-up: lazy allocations, clocks
reps = 20
ms, _ = A.filter_bench(cf, 1.0, 2.0, X, reps=reps, flush_l2=False)
print(name, os.environ.get("FLZ_LIB", "default"), "us/step %.2f" % (ms / reps / m * 1e3))
