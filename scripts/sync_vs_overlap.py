"""The overlapped convergence check must not change any result: same solve with
FLZ_SYNC_CHECK=1 (sequential, as the reference) and without, compared bit for bit."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200.workloads import workloads
from paper_2409_15053_b200 import solver as S
out = {}
for name in sys.argv[1:]:
    wl = workloads()[name]
    n, rp, ci, va = wl["gen"]()
    H = S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=False)
    cfg = S.LanczosConfig(**wl["cfg"])
    res = S.filtered_lanczos(H, *wl["interval"], cfg, want_vectors=True)
    st = res.stats
    out[name] = dict(count=len(res.eigenvalues), ev=hashlib.sha1(res.eigenvalues.tobytes()).hexdigest(),
                     vec=hashlib.sha1(np.ascontiguousarray(res.eigenvectors).tobytes()).hexdigest(),
                     blocks=st["block_steps"], mv=st["mv_iteration"], checks=st["checks"],
                     total=round(st["time_total_s"], 3), check_s=round(st["time_check_s"], 3))
print(json.dumps(out))
''' % ROOT
names = sys.argv[1:] or ["tiny", "c1", "c3"]
res = {}
for mode in ("sync", "overlap"):
    env = dict(os.environ)
    if mode == "sync":
        env["FLZ_SYNC_CHECK"] = "1"
    else:
        env.pop("FLZ_SYNC_CHECK", None)
    p = subprocess.run([sys.executable, "-c", CODE] + names, env=env, capture_output=True, text=True)
    if p.returncode:
        print(p.stderr[-2000:]); sys.exit(1)
    res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    print(mode, res[mode])
ok = all(all(res["sync"][n][k] == res["overlap"][n][k] for k in ("count", "ev", "vec", "blocks", "mv", "checks")) for n in names)
print("IDENTICAL" if ok else "MISMATCH")
sys.exit(0 if ok else 2)
