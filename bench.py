#!/usr/bin/env python
"""bench.py — filtered-Lanczos time-to-solution + filter-SpMV roofline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl flz|reference]

One "step" = one full filtered-Lanczos solve of the named workload (BASELINE.json configs,
paper_2409_15053_b200/workloads.py).  Prints ONE JSON line (rank 0).

Headline workload at N = 1: **c3**, the PARSEC-shaped Ge99H100-like Hamiltonian — the
configuration north_star's 1-GPU targets (>= 70 % of HBM bandwidth for the filter SpMV, >= 15x
the host-CPU reference time-to-solution) are quoted on, and the one the CPU reference can
solve completely inside the reference arm's time budget (~4 min on one core).  The other
single-GPU configurations (c1, c2, c4) are measured in the same run and reported under
``workloads`` (3 timed solves each, same keys).  N > 1: c5 (row-partitioned 27M-row
Laplacian, strong scaling), see workloads.py for its re-scope.

Keys follow the driver contract:
  value      seconds per solve with the matrix already resident in HBM (CUDA events on the
             library's stream bracket each solve; host logic in between is included)
  e2e        seconds per solve through the reference-facing API (flz_solve ==
             speig::filtered_lanczos) from HOST CSR buffers: host validation, layout
             construction, H2D, solve, D2H of the eigenvectors, all inside the timed region
  roofline   the dominant kernel (fused Clenshaw-step SpMM, K1).  Two byte counts per launch:
             ``bytes_algorithmic`` = 12*nnz + 4*(n+1) + 32*n*r (CSR stream +
             four block streams) and ``bytes_streamed`` = what this build's layout actually
             has to move (compressed matrix stream + block streams).  ``achieved``/``frac``
             use the SMALLER of the two, so a format that needs fewer bytes than CSR is not
             credited with bandwidth it never used; ``frac_csr_equivalent`` keeps the §8d
             figure and ``frac_streamed`` the layout's own.  Time = CUDA events around
             every filter application of the timed solves / number of Clenshaw steps.
             ``traffic`` is the committed ncu DRAM figure of the same kernel and workload
             (profiles/k1_traffic.json, bytes per launch), not measured in this run.
  cpu_baseline  the reference CPU library (oracle/_ref, one core: it is serial) on a bounded
             sample of the headline workload, scaled to a full solve and labelled as such;
             the real full-solve measurement is the reference arm.
`--impl reference` runs ONE complete ``speig::filtered_lanczos`` of the same workload on the
host (oracle/_ref) when its projected time fits the budget, and says so (``steps_run``).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "filtered_lanczos_time_to_solution"
UNIT = "s"
L2_NOTE = ("a 256 MB buffer is written between timed solves (L2 flush); inside a solve the "
           "Clenshaw steps re-read the matrix back to back as the algorithm does, so "
           "workloads whose per-step streams fit the 126 MB L2 (c1: 3.8 MB, c3: ~100 MB) "
           "run partly from L2")


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.tmp,
                stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.tmp.flush()
        rows = [ln.strip().split(", ") for ln in open(self.tmp.name) if ln.strip()]
        os.unlink(self.tmp.name)
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                power.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for name, flag in zip(names, r[3:7]):
                if flag.strip().lower() == "active":
                    reasons.add(name)
        # idle samples (between solves, during host-side matrix generation) are excluded from
        # the median: "under load" = above the idle clock floor
        loaded = [x for x in sm if x >= 0.5 * max(smax)] if sm else []
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return float(json.load(open(path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(name):
    prof = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(prof):
        return json.load(open(prof)).get(name)
    return None


# ------------------------------------------------------------------------ CPU reference
def _oracle():
    import oracle
    return oracle.best()


def cpu_filter_sample(orc, A, n, r, degree, budget_s):
    """Seconds per Clenshaw step of the reference's ChebyshevFilter::apply (filter.cpp:122-155)
    on one n x r block, from a run of about `budget_s` seconds."""
    lo, hi = -0.1, 1.0  # any bounds: the arithmetic per step does not depend on them
    X = np.random.default_rng(0).standard_normal((n, r))
    t0 = time.perf_counter()
    orc.filter_apply(A, np.ones(3), lo, hi, X)  # 2 steps: estimate the per-step cost
    per_step = (time.perf_counter() - t0) / 2
    m_s = int(max(2, min(degree, budget_s / max(per_step, 1e-9))))
    t0 = time.perf_counter()
    orc.filter_apply(A, np.ones(m_s + 1), lo, hi, X)
    elapsed = time.perf_counter() - t0
    return elapsed / m_s, m_s, elapsed


def cpu_baseline_sample(csr, cfg, block_steps, degree, budget_s=12.0):
    """Bounded CPU sample for the flz arm's `cpu_baseline`: the reference's filter on one
    block for ~budget_s seconds, scaled by degree x block_steps.  Orthogonalization, checks and
    recovery of the reference are NOT included: a lower bound, labelled extrapolated."""
    orc = _oracle()
    n, rp, ci, va = csr
    r = cfg.get("block_size", 3)
    A = orc.matrix_from_csr(n, rp, ci, va)
    per_step, m_s, elapsed = cpu_filter_sample(orc, A, n, r, degree, budget_s)
    return {"value": per_step * degree * block_steps, "unit": UNIT, "cores": 1, "kind": orc.kind,
            "extrapolated": True,
            "sample": (f"reference ChebyshevFilter::apply on one n x {r} block, {m_s} of {degree} "
                       f"Clenshaw steps ({elapsed:.1f} s on 1 host core, {per_step * 1e3:.2f} ms/step, "
                       f"backend {orc.backend()}); scaled x{degree}/{m_s} x {block_steps} block steps; "
                       "reference orthogonalization/check/recovery time not included (lower "
                       "bound); the measured full solve is the --impl reference arm"),
            "host_cores_available": os.cpu_count(), "ms_per_clenshaw_step": per_step * 1e3}


def golden_stats(name):
    """SolveStats of the reference's own full solve of this workload, generated in the build
    container (tests/golden/make_golden_fullsize.py) — informational."""
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    st = dict(zip([str(k) for k in g["stat_keys"]], [float(v) for v in g["stat_values"]]))
    st["wall_s"] = float(g["wall_s"][0])
    st["eigenpairs"] = int(len(g["eigenvalues"]))
    return st


def run_reference(args, wl):
    """Reference arm: the reference's own CPU implementation (oracle/_ref: the unmodified
    library compiled by oracle/Makefile; else the plain-C port) on this box's host cores, same
    workload / config / metric.  It runs ONE complete speig::filtered_lanczos (lanczos.cpp:
    573-655) when the projected time (filter sample x degree x block steps of the committed
    golden run, x1.5 for orthogonalization and checks) fits --ref-budget; the reference is
    serial, so `cores` = 1 and one solve is all the budget holds (steps_run = 1, no warm-up:
    a 4-minute CPU solve has no cold-start effect worth a second run).  Otherwise the sample
    is scaled and the line says "extrapolated": true."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    name = args.workload
    orc = _oracle()
    gold = golden_stats(name)
    if "gen_rows" in wl and wl.get("n", 0) > 5_000_000:
        # c5: the 27M-row matrix cannot be solved by the reference; sample a slab
        from paper_2409_15053_b200 import matrices as M
        n, rp, ci, va = M.laplacian3d(120)
        scale_rows = wl["n"] / n
    else:
        n, rp, ci, va = wl["gen"]()
        scale_rows = 1.0
    nnz = int(len(va))
    r = wl["cfg"].get("block_size", 3)
    A = orc.matrix_from_csr(n, rp, ci, va)
    degree = int(gold["degree"]) if gold else (wl["cfg"].get("degree") or 1000)
    block_steps = int(gold["block_steps"]) if gold else 100
    per_step, m_s, elapsed = cpu_filter_sample(orc, A, n, r, degree, 4.0)
    projected = per_step * degree * block_steps * 1.5 * scale_rows
    a, b = wl["interval"]
    base = {"unit": UNIT, "cores": 1, "kind": orc.kind, "host_cores_available": os.cpu_count(),
            "ms_per_clenshaw_step": per_step * 1e3, "backend": orc.backend()}
    config = {"workload": f"{name}: {wl['desc']}", "n": int(n * scale_rows), "nnz": int(nnz * scale_rows),
              "interval": [a, b], "block_size": r, "degree": degree,
              "expected_eigenpairs": wl["expect"], "l2": "n/a (CPU)"}
    if scale_rows == 1.0 and projected <= args.ref_budget:
        import oracle
        t0 = time.perf_counter()
        res = orc.solve(A, a, b, oracle.make_config(**wl["cfg"]), want_vectors=True)
        wall = time.perf_counter() - t0
        st = res.stats
        value = wall
        steps_run, extrapolated = 1, False
        config.update(degree=int(st["degree"]), degree_clamped=bool(st["degree_clamped"]),
                      block_steps=int(st["block_steps"]), basis_vectors=int(st["basis_vectors"]),
                      eigenpairs=int(len(res.eigenvalues)),
                      count_ok=len(res.eigenvalues) == wl["expect"], converged=bool(st["converged"]),
                      max_residual=float(res.residuals.max()) if len(res.residuals) else 0.0)
        base.update(value=value, sample=(
            f"ONE complete speig::filtered_lanczos of the workload on 1 host core: {wall:.1f} s wall "
            f"(reference SolveStats: total {st['time_total_s']:.1f} s, MV {st['time_mv_s']:.1f} s, "
            f"ORTH {st['time_orth_s']:.1f} s, PREPROC {st['time_preproc_s']:.2f} s; "
            f"{st['mv_total']} matvecs); --steps/--warmup do not multiply a serial 4-minute solve"))
        breakdown = {"filter_mv": st["time_mv_s"], "orth": st["time_orth_s"],
                     "preproc": st["time_preproc_s"], "total": st["time_total_s"]}
    else:
        value = per_step * degree * block_steps * scale_rows
        steps_run, extrapolated = 0, True
        config.update(block_steps=block_steps)
        base.update(value=value, sample=(
            f"EXTRAPOLATED: reference ChebyshevFilter::apply on one n x {r} block, {m_s} Clenshaw "
            f"steps ({elapsed:.1f} s), scaled x {degree} x {block_steps} block steps"
            + (f" x {scale_rows:.2f} rows (slab of the same stencil)" if scale_rows != 1.0 else "")
            + f"; a full solve is projected at {projected:.0f} s > budget {args.ref_budget:.0f} s; "
              "orthogonalization/check/recovery not included (lower bound)"))
        breakdown = None
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "steps_run": steps_run, "warmup_run": 0,
            "extrapolated": extrapolated, "ms_per_step": value * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config, "cpu_baseline": base,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    if breakdown:
        line["breakdown_s"] = breakdown
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ flz arm
class Dist:
    """torch.distributed plumbing of the N > 1 runs (rendezvous, barrier, max over ranks)."""

    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local_rank)
            dist.init_process_group("nccl")
            self.pg = dist

    def context(self):
        from paper_2409_15053_b200 import Context
        if self.world == 1:
            return Context.default()
        uid = [Context.nccl_unique_id() if self.rank == 0 else None]
        self.pg.broadcast_object_list(uid, src=0)
        ctx = Context(self.local_rank, self.rank, self.world, uid[0])
        ctx.adopt_as_default()
        return ctx

    def barrier(self, ctx):
        ctx.sync()
        if self.pg is not None:
            self.pg.barrier()

    def max(self, x):
        if self.pg is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum_int(self, x):
        if self.pg is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.int64, device="cuda")
        self.pg.all_reduce(t)
        return int(t.item())


def measure(D, ctx, name, wl, steps, warmup, e2e_steps):
    """W warm-up + K timed solves with the matrix resident, then e2e_steps end-to-end solves
    from host CSR.  Returns (record, last result, csr)."""
    from paper_2409_15053_b200 import solver as S
    from paper_2409_15053_b200.workloads import step_bytes

    a, b = wl["interval"]
    cfg = S.LanczosConfig(**wl["cfg"])
    r = cfg.block_size
    slab = D.world > 1 and "gen_rows" in wl
    if slab:  # every rank builds only its own rows
        n = wl["n"]
        rb, re_ = n * D.rank // D.world, n * (D.rank + 1) // D.world
        _, rp, ci, va = wl["gen_rows"](rb, re_)
        csr = None
        nnz = D.sum_int(int(len(va)))
    else:
        csr = wl["gen"]()
        n, rp, ci, va = csr
        nnz = int(len(va))

    def make_matrix(check):
        if slab:
            return S.SparseSymMatrix.from_local_rows(n, rb, re_, rp, ci, va)
        return S.SparseSymMatrix.from_csr(n, rp, ci, va, check_symmetry=check)

    want_vectors = D.world == 1  # distributed results hold local rows inside the library

    # ---- resident arm
    H = make_matrix(False)
    res = None
    for _ in range(warmup):
        res = S.filtered_lanczos(H, a, b, cfg, want_vectors=want_vectors)
    times, mv_s, orth_s, chk_s, rec_s, launches, filter_steps = [], 0.0, 0.0, 0.0, 0.0, 0, 0
    for _ in range(steps):
        ctx.flush_l2()
        D.barrier(ctx)
        ctx.timer_start(0)
        res = S.filtered_lanczos(H, a, b, cfg, want_vectors=want_vectors)
        ms = ctx.timer_stop(0)
        D.barrier(ctx)
        times.append(D.max(ms * 1e-3))
        st = res.stats
        mv_s += st["time_mv_s"]
        orth_s += st["time_orth_s"]
        chk_s += st["time_check_s"]
        rec_s += st["time_recover_s"]
        launches += st["gpu_launches"]
        filter_steps += st["degree"] * st["block_steps"]
    value = sum(times) / len(times)
    st = res.stats

    # ---- e2e arm: host CSR -> validated SparseSymMatrix -> solve -> eigenvectors on the host
    e2e_times = []
    h2d = (12 * nnz + 8 * (n + 1) + 8 * n * r + 8 * n) // D.world   # per rank
    d2h = 8 * n * len(res.eigenvalues) // D.world
    for i in range(1 + e2e_steps):
        ctx.flush_l2()
        D.barrier(ctx)
        t0 = time.perf_counter()
        H2 = make_matrix(True)
        r2 = S.filtered_lanczos(H2, a, b, cfg, want_vectors=want_vectors)
        _ = float(r2.eigenvalues.sum()) if len(r2.eigenvalues) else 0.0
        ctx.sync()
        dt = time.perf_counter() - t0
        del H2
        if i > 0:  # first pass is the warm-up of this arm
            e2e_times.append(D.max(dt))
    e2e = sum(e2e_times) / len(e2e_times)

    peak, peak_src = measured_peak_gbs()
    b_alg = step_bytes(n, nnz, r)
    lay = H.layout() if D.world == 1 else None
    b_str = lay["step_bytes"][min(r, 4) - 1] if lay else None
    t_step = mv_s / max(filter_steps, 1)
    gbs = lambda nbytes: nbytes / t_step / 1e9 if (nbytes and t_step > 0) else None
    b_used = min(b_alg, b_str) if b_str else b_alg
    traffic = committed_traffic(name)
    ok = len(res.eigenvalues) == wl["expect"] if wl["expect"] is not None else True
    rec = {
        "value": value, "unit": UNIT, "steps": steps, "warmup": warmup,
        "config": {"workload": f"{name}: {wl['desc']}", "n": n, "nnz": nnz,
                   "interval": [a, b], "block_size": r, "degree": st["degree"],
                   "degree_clamped": bool(st["degree_clamped"]), "block_steps": st["block_steps"],
                   "basis_vectors": st["basis_vectors"], "eigenpairs": int(len(res.eigenvalues)),
                   "expected_eigenpairs": wl["expect"], "count_ok": ok,
                   "converged": bool(st["converged"]),
                   "max_residual": float(res.residuals.max()) if len(res.residuals) else 0.0,
                   "l2": L2_NOTE},
        "breakdown_s": {"filter_mv": mv_s / steps, "orth": orth_s / steps,
                        "host_check": chk_s / steps, "recover": rec_s / steps,
                        "preproc": st["time_preproc_s"]},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": {"kernel": (lay["kernel"] if lay else "clenshaw_step_ug_warp")
                     + " (fused Clenshaw-step SpMM, K1)", "bound": "hbm",
                     "achieved": gbs(b_used), "peak": peak, "unit": "GB/s",
                     "frac": gbs(b_used) / peak if gbs(b_used) else None,
                     "peak_source": peak_src, "bytes_per_launch": b_used,
                     "bytes_algorithmic": b_alg, "bytes_streamed": b_str,
                     "frac_csr_equivalent": gbs(b_alg) / peak if gbs(b_alg) else None,
                     "frac_streamed": gbs(b_str) / peak if gbs(b_str) else None,
                     "launches_timed": int(filter_steps), "avg_launch_us": t_step * 1e6,
                     "traffic": traffic,
                     "traffic_source": "committed ncu capture (profiles/k1_traffic.json), "
                                       "not measured in this run" if traffic else None,
                     "note": "achieved = min(algorithmic, streamed) bytes per launch / CUDA-event "
                             "time of the filter launches; algorithmic = 12*nnz + 4*(n+1) + 32*n*r "
                             "(SURVEY 8d), streamed = the layout's matrix stream + block streams"},
    }
    return rec, res, csr


def run_flz(args, wl):
    D = Dist()
    if D.world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={D.world}")
    ctx = D.context()
    sampler = (ClockSampler(D.local_rank)
               if D.rank == 0 and not os.environ.get("FLZ_BENCH_NO_SAMPLER") else None)
    head, res, csr = measure(D, ctx, args.workload, wl, args.steps, args.warmup, args.steps)
    extras = {}
    if D.world == 1 and args.extra:
        from paper_2409_15053_b200.workloads import workloads
        W = workloads()
        for name in args.extra.split(","):
            if name and name != args.workload and name in W:
                extras[name], _, _ = measure(D, ctx, name, W[name], 3, 3, 3)
    clocks = sampler.stop() if sampler else None
    if D.rank != 0:
        return
    cpu = None
    if D.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(csr, wl["cfg"], head["config"]["block_steps"],
                                  head["config"]["degree"])
        gold = golden_stats(args.workload)
        if gold:
            cpu["reference_full_solve_build_container"] = {
                "wall_s": gold["wall_s"], "time_mv_s": gold["time_mv_s"],
                "time_orth_s": gold["time_orth_s"], "block_steps": int(gold["block_steps"]),
                "eigenpairs": gold["eigenpairs"],
                "note": "one run of the compiled reference in the build container "
                        "(tests/golden/make_golden_fullsize.py), not on this box"}
    line = {"metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": D.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["value"] * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": head["config"], "breakdown_s": head["breakdown_s"],
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"] + sum(x["gpu_launches"] for x in extras.values()),
            "gpu_launches_headline": head["gpu_launches"],
            "roofline": head["roofline"], "clocks": clocks}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if extras:
        line["workloads"] = extras
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`python bench.py --gpus N` without a launcher: start N ranks with torch.distributed.run
    on this node and relay rank 0's JSON line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None)
    ap.add_argument("--impl", default="flz", choices=["flz", "reference"])
    ap.add_argument("--extra", default="c1,c2,c4",
                    help="further single-GPU workloads reported under `workloads` ('' = none)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=1200.0,
                    help="seconds the reference arm may spend on one complete CPU solve")
    args = ap.parse_args()
    from paper_2409_15053_b200.workloads import workloads
    if args.workload is None:  # PARSEC-shaped config on one GPU, configs[4] row-partitioned
        args.workload = "c3" if args.gpus == 1 else "c5"
    wl = workloads()[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    else:
        run_flz(args, wl)


if __name__ == "__main__":
    main()
