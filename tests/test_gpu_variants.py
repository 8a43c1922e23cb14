"""GPU coverage of the code paths the automatic choices rarely take: the SPLIT layout with
rest slices (forced), the planar block layout (forced), and the pipelined convergence checks
against the sequential order.  Each variant runs in a fresh process because the switches are
read once per process."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def run(code, env_extra, args=()):
    env = dict(os.environ)
    for k in ("FLZ_SPLIT", "FLZ_K1_LAYOUT", "FLZ_SYNC_CHECK", "FLZ_K1_PDL", "FLZ_P2_DENSE",
              "FLZ_ST_TILE", "FLZ_ST_STAGES", "FLZ_ST_CTAS",
              "FLZ_ST_PRODUCERS", "FLZ_HY", "FLZ_HY_OVERLAP", "FLZ_SPECULATE", "FLZ_ORTH_FUSED",
              "FLZ_TS_UPDATE", "FLZ_PLAN_AHEAD", "FLZ_ST_SLAB", "FLZ_SLAB_PACK", "FLZ_SLAB_PDL",
              "FLZ_MS", "FLZ_MS_K", "FLZ_MS_CORE", "FLZ_MS_ROWS"):
        env.pop(k, None)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", code, *args], env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("env", [{"FLZ_SPLIT": "1"}, {"FLZ_SPLIT": "0"}, {"FLZ_K1_LAYOUT": "planar"},
                                 {"FLZ_SPLIT": "1", "FLZ_K1_LAYOUT": "planar"},
                                 {"FLZ_K1_PDL": "0"},          # plain stream-ordered launches
                                 {"FLZ_P2_DENSE": "1", "FLZ_HY": "0"},   # paired layout with dense sections
                                 {"FLZ_HY": "0"},              # plain paired layout for block matrices
                                 {"FLZ_ST_TILE": "0"},         # stencils: one-warp-per-slice kernel
                                 {"FLZ_HY_OVERLAP": "1"},      # hybrid layout: gather + finish launches
                                 {"FLZ_HY_OVERLAP": "0"},
                                 {"FLZ_ST_TILE": "64", "FLZ_ST_STAGES": "2", "FLZ_ST_CTAS": "3"},
                                 {"FLZ_ST_TILE": "256", "FLZ_ST_STAGES": "4", "FLZ_ST_CTAS": "1"},
                                 {"FLZ_ST_TILE": "512", "FLZ_K1_LAYOUT": "planar"}])
def test_filter_variants_vs_oracle(env, best_oracle):
    """p(A) X through the forced layouts agrees with the reference (oracle) to 1e-13."""
    code = r'''
import sys, json
sys.path.insert(0, %r)
import numpy as np
import oracle
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M
orc = oracle.best()
ctx = Context(0)
out = {}
for name, gen in (("parsec7k", lambda: M.parsec_like(radius=12.0, n_atoms=12)),
                  ("parsec_overlap", lambda: M.parsec_like(radius=10.0, n_atoms=30, ball_radius=3.6)),
                  ("lap2d30", lambda: M.laplacian2d(30)), ("lap3d12", lambda: M.laplacian3d(12)),
                  ("rand400", lambda: M.random_sparse_sym(400, 0.04, 7))):
    n, rp, ci, va = gen()
    for r in (1, 3, 4):
        X = np.random.default_rng(r).standard_normal((n, r))
        cf, _, _, _ = orc.build_filter(-1.0, 9.0, 2.0, 3.0, 30)
        Yo = orc.filter_apply(orc.matrix_from_csr(n, rp, ci, va), cf, -1.0, 9.0, X)
        A = DeviceMatrix(ctx, n, rp, ci, va)
        Y = A.filter_apply(cf, 4.0, 5.0, X)
        out["%%s_r%%d" %% (name, r)] = float(np.abs(Y - Yo).max() / np.abs(Yo).max())
print(json.dumps(out))
''' % ROOT
    errs = run(code, env)
    assert max(errs.values()) <= 1e-13, errs


SOLVE_CODE = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200 import matrices as M, solver as S
out = {}
for name, gen, a, b, kw in (("lap2d30", lambda: M.laplacian2d(30), 3.0, 3.8, {}),
                            ("lap2d30_r1", lambda: M.laplacian2d(30), 3.0, 3.8, dict(block_size=1, degree=20)),
                            ("rand400", lambda: M.random_sparse_sym(400, 0.04, 7), -0.5, 0.5, {}),
                            ("diag5", lambda: M.diag_matrix([1, 2, 3, 4, 5]), 1.5, 4.5, {}),
                            ("parsec7k", lambda: M.parsec_like(radius=12.0, n_atoms=12), -0.6, 0.0, dict(degree=50))):
    res = S.filtered_lanczos(S.SparseSymMatrix.from_csr(*gen()), a, b, S.LanczosConfig(**kw))
    st = res.stats
    out[name] = dict(ev=hashlib.sha1(res.eigenvalues.tobytes()).hexdigest(),
                     vec=hashlib.sha1(np.ascontiguousarray(res.eigenvectors).tobytes()).hexdigest(),
                     count=len(res.eigenvalues), blocks=st["block_steps"], mv=st["mv_iteration"],
                     checks=st["checks"], conv=st["converged"])
print(json.dumps(out))
''' % ROOT


def test_pipelined_checks_equal_sequential_order():
    """Snapshots + rollback: the overlapped convergence checks give bit-identical eigenpairs,
    block counts, matvec counts and check counts to the reference's sequential order."""
    seq = run(SOLVE_CODE, {"FLZ_SYNC_CHECK": "1"})
    par = run(SOLVE_CODE, {})
    assert seq == par
    assert all(v["conv"] == 1 for v in par.values())


TILE_CODE = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S
ctx = Context(0)
out = {}
for name, gen in (("lap3d33", lambda: M.laplacian3d(33)), ("lap2d77", lambda: M.laplacian2d(77)),
                  ("lap3d12", lambda: M.laplacian3d(12)), ("lap3d64", lambda: M.laplacian3d(64))):
    n, rp, ci, va = gen()
    A = DeviceMatrix(ctx, n, rp, ci, va)
    cf = S.indicator_coefficients(-0.3, 0.25, 40)
    for r in (1, 3, 6):
        X = np.random.default_rng(r).standard_normal((n, r))
        Y = A.filter_apply(cf, 4.0, 4.5, X)
        Z = A.spmm(X) if hasattr(A, "spmm") else Y
        out["%%s_r%%d" %% (name, r)] = [hashlib.sha1(np.ascontiguousarray(Y).tobytes()).hexdigest(),
                                      hashlib.sha1(np.ascontiguousarray(Z).tobytes()).hexdigest()]
print(json.dumps(out))
''' % ROOT


def test_tile_kernel_bit_identical_to_warp_kernel():
    """The TMA-staged stencil kernel adds the positions of a row in the same order as the
    one-warp-per-slice kernel: filter outputs and plain products are bit-identical, for every
    tile size / ring depth (boundary tiles: clipped runs, slices with per-lane positions)."""
    warp = run(TILE_CODE, {"FLZ_ST_TILE": "0", "FLZ_K1_LAYOUT": "planar"})
    for env in ({"FLZ_K1_LAYOUT": "planar"},                       # one launch per Clenshaw step
                {"FLZ_ST_TILE": "64", "FLZ_ST_PRODUCERS": "2", "FLZ_K1_LAYOUT": "planar"},
                {"FLZ_ST_TILE": "32", "FLZ_ST_STAGES": "2", "FLZ_K1_LAYOUT": "planar"},
                {"FLZ_ST_TILE": "256", "FLZ_ST_STAGES": "5", "FLZ_ST_CTAS": "1", "FLZ_K1_LAYOUT": "planar"}):
        assert run(TILE_CODE, env) == warp, env


SLAB_CODE = r'''
import sys, json, hashlib, threading
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, LoopHub, matrices as M, solver as S
out = {}
cf = S.indicator_coefficients(-0.3, 0.25, 24)
for name, gen, nranks in (("lap3d24x3", lambda: M.laplacian3d(24), 3),
                          ("lap3d32x2", lambda: M.laplacian3d(32), 2),
                          ("lap3d16x8", lambda: M.laplacian3d(16), 8),
                          ("lap3d12x3", lambda: M.laplacian3d(12), 3),      # slices across planes
                          ("lap2d96x4", lambda: M.laplacian2d(96), 4),
                          ("lap3d40x2", lambda: M.laplacian3d(40), 2)):
    n, rp, ci, va = gen()
    starts = [n * k // nranks // 2 * 2 for k in range(nranks + 1)]
    hub = LoopHub(nranks)
    res, err = [None] * nranks, [None] * nranks
    def work(rank):
        try:
            ctx = Context.loopback(hub, rank)
            b, e = starts[rank], starts[rank + 1]
            A = DeviceMatrix(ctx, n, rp[b:e + 1] - rp[b], ci[rp[b]:rp[e]], va[rp[b]:rp[e]],
                             row_begin=b, row_end=e)
            got = {"kernel": A.k1_info(3)["kernel"]}
            for r in (1, 3, 4):
                X = np.random.default_rng(r).standard_normal((n, r))
                Y = A.filter_apply(cf, 4.0, 4.5, X[b:e])
                Z = A.spmm(X[b:e], counted=False)
                got[r] = (Y, Z)
            ctx.sync()
            res[rank] = got
        except BaseException as ex:
            err[rank] = ex
    th = [threading.Thread(target=work, args=(k,)) for k in range(nranks)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not any(t.is_alive() for t in th), "a rank hangs"
    for ex in err:
        if ex is not None:
            raise ex
    out[name + "_kernel"] = sorted(set(p["kernel"] for p in res))
    ctx0 = Context(0)
    A0 = DeviceMatrix(ctx0, n, rp, ci, va)
    for r in (1, 3, 4):
        Y = np.vstack([p[r][0] for p in res]); Z = np.vstack([p[r][1] for p in res])
        X = np.random.default_rng(r).standard_normal((n, r))
        Y0 = A0.filter_apply(cf, 4.0, 4.5, X); Z0 = A0.spmm(X, counted=False)
        out["%%s_r%%d" %% (name, r)] = [hashlib.sha1(np.ascontiguousarray(Y).tobytes()).hexdigest(),
                                      hashlib.sha1(np.ascontiguousarray(Z).tobytes()).hexdigest()]
        out["%%s_r%%d_dev" %% (name, r)] = max(float(np.abs(Y - Y0).max() / np.abs(Y0).max()),
                                             float(np.abs(Z - Z0).max() / np.abs(Z0).max()))
print(json.dumps(out))
''' % ROOT


def test_tile_kernel_on_row_slabs_bit_identical_to_warp_kernel():
    """Row slabs through the loopback transport: the TMA-staged tile kernel (runs of the
    virtual source [front halo | local | back halo], tiles without halo rows launched while
    the halo travels) against the one-warp-per-slice kernel on the same slabs — same order of
    additions, bit-identical filter outputs and products; both within 1e-13 of one context."""
    tile = run(SLAB_CODE, {})
    warp = run(SLAB_CODE, {"FLZ_ST_SLAB": "0"})
    small = run(SLAB_CODE, {"FLZ_ST_TILE": "64", "FLZ_ST_STAGES": "2"})
    plain = run(SLAB_CODE, {"FLZ_SLAB_PACK": "0", "FLZ_SLAB_PDL": "0"})   # pack launch, no PDL
    for k, v in tile.items():
        if k.endswith("_kernel"):
            assert v == ["clenshaw_step_stencil_tma"], (k, v)
            assert warp[k] == ["clenshaw_step_ug_warp"], (k, warp[k])
        elif k.endswith("_dev"):
            assert v <= 1e-13 and warp[k] <= 1e-13, (k, v, warp[k])
        else:
            assert v == warp[k], k
            assert v == small[k], k
            assert v == plain[k], k


MS_CODE = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S
ctx = Context(0)
out = {}
for name, gen in (("lap2d200", lambda: M.laplacian2d(200)), ("lap2d77", lambda: M.laplacian2d(77)),
                  ("lap2d33", lambda: M.laplacian2d(33)), ("lap2d300", lambda: M.laplacian2d(300)),
                  ("lap3d12", lambda: M.laplacian3d(12))):
    n, rp, ci, va = gen()
    A = DeviceMatrix(ctx, n, rp, ci, va)
    for m in (1, 2, 3, 4, 5, 6, 9, 10, 50):
        cf = S.indicator_coefficients(-0.3, 0.25, m)
        for r in (1, 3, 4, 6):
            X = np.random.default_rng(r + m).standard_normal((n, r))
            Y = A.filter_apply(cf, 4.0, 4.5, X)
            out["%%s_m%%d_r%%d" %% (name, m, r)] = hashlib.sha1(np.ascontiguousarray(Y).tobytes()).hexdigest()
out["launches"] = ctx.launches
print(json.dumps(out))
''' % ROOT


def test_multistep_stencil_launches_bit_identical_to_single_steps():
    """clenshaw_multistep_stencil (K Clenshaw steps of a short-reach stencil per launch, halo
    rows recomputed per CTA) against one launch per step: bit-identical filter outputs for every
    degree (leftover steps, m < K), column count, K and core size; fewer launches."""
    one = run(MS_CODE, {"FLZ_MS": "0"})
    for env in ({}, {"FLZ_MS": "1"}, {"FLZ_MS": "1", "FLZ_MS_K": "2"}, {"FLZ_MS": "1", "FLZ_MS_K": "8"},
                {"FLZ_MS": "1", "FLZ_MS_K": "3", "FLZ_MS_CORE": "1024"}):
        got = run(MS_CODE, env)
        assert got["launches"] < one["launches"], env
        for k, v in one.items():
            if k != "launches":
                assert got[k] == v, (env, k)


HY_CODE = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S
ctx = Context(0)
out = {}
for name, gen in (("parsec7k", lambda: M.parsec_like(radius=12.0, n_atoms=12)),
                  ("parsec_overlap", lambda: M.parsec_like(radius=10.0, n_atoms=30, ball_radius=3.6)),
                  ("parsec20k", lambda: M.parsec_like(radius=17.0, n_atoms=40))):
    n, rp, ci, va = gen()
    A = DeviceMatrix(ctx, n, rp, ci, va)
    out[name + "_kernel"] = A.k1_info(3)["kernel"] if hasattr(A, "k1_info") else ""
    cf = S.indicator_coefficients(-0.3, 0.25, 25)
    for r in (1, 2, 3, 4, 7):
        X = np.random.default_rng(r).standard_normal((n, r))
        Y = A.filter_apply(cf, 4.0, 4.5, X)
        Z = A.spmm(X)
        out["%%s_r%%d" %% (name, r)] = [hashlib.sha1(np.ascontiguousarray(Y).tobytes()).hexdigest(),
                                      hashlib.sha1(np.ascontiguousarray(Z).tobytes()).hexdigest()]
print(json.dumps(out))
''' % ROOT


def test_hybrid_overlapped_variant_bit_identical():
    """hybrid_gather + hybrid_finish (dense tasks and slices in one launch, sums combined by a
    second one) add in the same order as hybrid_dense_tasks + hybrid_slices."""
    two = run(HY_CODE, {"FLZ_HY_OVERLAP": "0"})
    one = run(HY_CODE, {"FLZ_HY_OVERLAP": "1"})
    assert any("hybrid_gather" in v for k, v in one.items() if k.endswith("_kernel")), one
    assert all("hybrid_gather" not in v for k, v in two.items() if k.endswith("_kernel"))
    strip = lambda d: {k: v for k, v in d.items() if not k.endswith("_kernel")}
    assert strip(one) == strip(two)


def test_speculative_application_changes_nothing():
    """The operator application queued ahead of the host's wait (flz_lanczos_step) is the
    application the next step would have run: eigenpairs, block counts, matvec counts and check
    counts are bit-identical with FLZ_SPECULATE=0, with the pipelined and the sequential
    checks (rollbacks drop a queued application), and with the layout planned at the first
    product instead of inside from_csr."""
    base = run(SOLVE_CODE, {"FLZ_SPECULATE": "0"})
    assert run(SOLVE_CODE, {}) == base
    assert run(SOLVE_CODE, {"FLZ_SYNC_CHECK": "1", "FLZ_SPECULATE": "0"}) == base
    assert run(SOLVE_CODE, {"FLZ_PLAN_AHEAD": "0"}) == base
    assert all(v["conv"] == 1 for v in base.values())


ORTH_CODE = r'''
import sys, json
sys.path.insert(0, %r)
import numpy as np
from paper_2409_15053_b200 import Context, DeviceMatrix, matrices as M, solver as S
from paper_2409_15053_b200.device import Basis
ctx = Context(0)
out = {}
for name, gen in (("lap3d20", lambda: M.laplacian3d(20)), ("parsec7k", lambda: M.parsec_like(radius=12.0, n_atoms=12))):
    n, rp, ci, va = gen()
    A = DeviceMatrix(ctx, n, rp, ci, va)
    cf = S.indicator_coefficients(-0.4, 0.1, 12)
    for r in (1, 2, 3, 4, 5, 8):
        start = S.init_block(n, r, 20177)
        B = Basis(ctx, A, start, 10 * r)
        res = [B.step(cf, 3.0, 3.5) for _ in range(8)]
        out["%%s_r%%d" %% (name, r)] = dict(
            D=[x[0].tolist() for x in res], S=[x[1].tolist() for x in res],
            scale=[x[2] for x in res], dead=[x[3].tolist() for x in res],
            ortho=B.ortho_error(), Q=B.get(0, 9 * r).tolist() if r <= 2 and n < 9000 else None)
        B.close()
print(json.dumps(out))
''' % ROOT


def test_fused_orthogonalization_agrees_with_the_multi_launch_path():
    """One rank: [Q Z]^T Z in one sweep, the tall-skinny update kernel and the cooperative block
    QR (r <= 4: block_qr_kernel<4>, r = 5, 8: <16>) against the multi-launch path of the
    row-partitioned runs — same D_k, S_k, op_scale and dead flags to rounding, basis
    orthonormal to 1e-13 either way."""
    fused = run(ORTH_CODE, {})
    plain = run(ORTH_CODE, {"FLZ_ORTH_FUSED": "0"})
    old_update = run(ORTH_CODE, {"FLZ_TS_UPDATE": "0"})
    for other in (plain, old_update):
        for key, a in fused.items():
            b = other[key]
            assert a["ortho"] <= 1e-13 and b["ortho"] <= 1e-13, key
            assert a["dead"] == b["dead"], key
            for k in range(len(a["D"])):
                Da, Db = np.array(a["D"][k]), np.array(b["D"][k])
                Sa, Sb = np.array(a["S"][k]), np.array(b["S"][k])
                tol = 1e-10 * max(1.0, np.abs(Da).max(), np.abs(Sa).max())
                assert np.abs(Da - Db).max() <= tol and np.abs(Sa - Sb).max() <= tol, (key, k)
                assert abs(a["scale"][k] - b["scale"][k]) <= 1e-12 * a["scale"][k]
