"""Python handles over the device layer of libflz (include/flz.h).

These are thin RAII wrappers used by the tests, bench.py and smoke(): every method is one
C-ABI call.  Dense blocks are NumPy arrays with column-major semantics (Fortran order),
as speig::DenseBlock (dense_block.hpp:11-40).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib


def _fcol(X, dtype=np.float64):
    """n x r array -> contiguous column-major buffer (1-D view) + shape."""
    X = np.asarray(X, dtype=dtype)
    if X.ndim == 1:
        X = X[:, None]
    flat = np.ascontiguousarray(X.T).ravel()  # column j contiguous
    return flat, X.shape


def _from_fcol(flat, n, r):
    return flat.reshape(r, n).T  # Fortran-ordered view n x r


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class LoopHub:
    """Shared state of the loopback transport (tests only; flz_loop_hub_create)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        check(lib().flz_loop_hub_create(nranks, C.byref(h)))
        self.handle, self.nranks = h, nranks

    def close(self):
        if getattr(self, "handle", None):
            lib().flz_loop_hub_destroy(self.handle)
            self.handle = None


class Context:
    """flz_ctx: one GPU, one stream (+ NCCL communicator when nranks > 1)."""

    def __init__(self, device: int = -1, rank: int = 0, nranks: int = 1, nccl_uid: bytes = b""):
        h = C.c_void_p()
        if nranks > 1:
            buf = C.create_string_buffer(nccl_uid, 128)
            check(lib().flz_ctx_create_dist(device, rank, nranks, buf, C.byref(h)))
        else:
            check(lib().flz_ctx_create(device, C.byref(h)))
        self.handle = h
        self.rank, self.nranks = rank, nranks

    @classmethod
    def loopback(cls, hub: "LoopHub", rank: int, device: int = -1) -> "Context":
        """TESTS ONLY: rank `rank` of a row-partitioned run whose ranks are threads of this
        process sharing one GPU (csrc/comm.cu).  Call the library from one thread per rank."""
        h = C.c_void_p()
        check(lib().flz_ctx_create_loopback(device, rank, hub.nranks, hub.handle, C.byref(h)))
        self = cls.__new__(cls)
        self.handle, self.rank, self.nranks, self._hub = h, rank, hub.nranks, hub
        return self

    @classmethod
    def default(cls) -> "Context":
        """Non-owning view of the context the host solver layer uses (flz_default_ctx)."""
        h = C.c_void_p()
        check(lib().flz_default_ctx(C.byref(h)))
        self = cls.__new__(cls)
        self.handle, self.rank, self.nranks = h, int(lib().flz_ctx_rank(h)), int(lib().flz_ctx_nranks(h))
        self.close = lambda: None
        return self

    def adopt_as_default(self):
        """Make the host solver layer (filtered_lanczos & co.) run on this context."""
        check(lib().flz_set_default_ctx(self.handle))

    def adopt_for_thread(self):
        """TESTS ONLY: the calling thread's host-layer calls run on this context (the ranks of
        a loopback run are threads of one process)."""
        check(lib().flz_set_thread_ctx(self.handle))

    @staticmethod
    def release_thread():
        check(lib().flz_set_thread_ctx(None))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().flz_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self.handle:
            lib().flz_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib().flz_ctx_sync(self.handle))

    def set_exact(self, exact: bool):
        check(lib().flz_ctx_set_exact(self.handle, int(exact)))

    def set_tuning(self, slices_per_cta=0, tasks_per_cta=0, batch=0):
        """Launch-shape knobs of the fused Clenshaw-step kernels (0 = default)."""
        check(lib().flz_ctx_set_tuning(self.handle, int(slices_per_cta), int(tasks_per_cta),
                                       int(batch)))

    @property
    def launches(self) -> int:
        return int(lib().flz_ctx_launch_count(self.handle))

    def timer_start(self, slot=0):
        check(lib().flz_timer_start(self.handle, slot))

    def timer_stop(self, slot=0) -> float:
        ms = C.c_double()
        check(lib().flz_timer_stop(self.handle, slot, C.byref(ms)))
        return ms.value

    def flush_l2(self, nbytes=256 << 20):
        check(lib().flz_flush_l2(self.handle, nbytes))

    def mem_info(self):
        f, t = C.c_size_t(), C.c_size_t()
        check(lib().flz_mem_info(self.handle, C.byref(f), C.byref(t)))
        return f.value, t.value

    # ---- L0 seams (kernels.hpp:29-49)
    def dot(self, x, y) -> float:
        out = C.c_double()
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        check(lib().flz_dot(self.handle, x, y, len(x), C.byref(out)))
        return out.value

    def axpy(self, a, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.array(y, dtype=np.float64, order="C")
        check(lib().flz_axpy(self.handle, a, x, y, len(x)))
        return y

    def clenshaw_combine(self, s1, s2, b, w, y1, y2, x):
        arrs = [np.ascontiguousarray(a, np.float64) for a in (w, y1, y2, x)]
        out = np.empty_like(arrs[0])
        check(lib().flz_clenshaw_combine(self.handle, len(out), s1, s2, b, *arrs, out))
        return out


class DeviceMatrix:
    """flz_matrix: SELL-32-sigma matrix resident in HBM (CSR in, like sparse.hpp:28-33)."""

    def __init__(self, ctx: Context, n, row_ptr, col_idx, values, sigma=0, row_begin=0,
                 row_end=None):
        self.ctx = ctx
        self.n = int(n)
        row_end = self.n if row_end is None else row_end
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col_idx, np.int32)
        va = np.ascontiguousarray(values, np.float64)
        h = C.c_void_p()
        check(lib().flz_matrix_upload(ctx.handle, self.n, row_begin, row_end, rp, ci, va, sigma,
                                      C.byref(h)))
        self.handle = h
        self.nl = int(lib().flz_matrix_rows_local(h))
        self.nnz = int(lib().flz_matrix_nnz_local(h))

    def stats(self):
        a, b, c, e = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        sigma = lib().flz_matrix_stats(self.handle, C.byref(a), C.byref(b), C.byref(c), C.byref(e))
        mb, ue = C.c_int64(), C.c_int64()
        check(lib().flz_matrix_layout(self.handle, C.byref(mb), C.byref(ue)))
        return {"stored": a.value, "slices": b.value, "halo_rows": c.value,
                "boundary_slices": e.value, "sigma": sigma, "nnz": self.nnz,
                "fill": a.value / max(self.nnz, 1), "matrix_bytes": mb.value,
                "uniform_entries": ue.value}

    def k1_info(self, r=3):
        """Kernel a fused Clenshaw step of r columns runs and the bytes it streams."""
        info = (C.c_int64 * 4)()
        name = C.create_string_buffer(96)
        check(lib().flz_matrix_k1_info(self.handle, r, info, name, 96))
        return {"kernel": name.value.decode(), "step_bytes": int(info[0]),
                "dense_blocks": int(info[1]), "dense_entries": int(info[2])}

    def close(self):
        if getattr(self, "handle", None):
            lib().flz_matrix_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def spmm(self, X, counted=True):
        flat, (n, r) = _fcol(X)
        assert n == self.nl, "block rows do not match matrix dimension"
        out = np.empty_like(flat)
        check(lib().flz_spmm(self.ctx.handle, self.handle, _ptr(flat), r, _ptr(out), int(counted)))
        return _from_fcol(out, n, r)

    def filter_apply(self, coeffs, c, e, X):
        flat, (n, r) = _fcol(X)
        assert n == self.nl, "block rows do not match matrix dimension"
        cf = np.ascontiguousarray(coeffs, np.float64)
        out = np.empty_like(flat)
        check(lib().flz_filter_apply(self.ctx.handle, self.handle, cf, len(cf) - 1, c, e,
                                     _ptr(flat), r, _ptr(out)))
        return _from_fcol(out, n, r)

    def filter_bench(self, coeffs, c, e, X, reps=1, flush_l2=True, want_output=False):
        flat, (n, r) = _fcol(X)
        cf = np.ascontiguousarray(coeffs, np.float64)
        ms = C.c_double()
        out = np.empty_like(flat) if want_output else None
        check(lib().flz_filter_bench(self.ctx.handle, self.handle, cf, len(cf) - 1, c, e,
                                     _ptr(flat), r, reps, int(flush_l2), C.byref(ms),
                                     _ptr(out) if want_output else None))
        return ms.value, (_from_fcol(out, n, r) if want_output else None)

    def bounds_lanczos(self, q0, steps):
        q0 = np.ascontiguousarray(q0, np.float64)
        dd, ee = np.zeros(steps), np.zeros(max(steps, 1))
        beta, done = C.c_double(), C.c_int()
        check(lib().flz_bounds_lanczos(self.ctx.handle, self.handle, steps, q0, dd, ee,
                                       C.byref(beta), C.byref(done)))
        k = done.value
        return dd[:k], ee[: max(k - 1, 0)], beta.value


class Basis:
    """flz_basis: device-resident block Lanczos factorization (lanczos.hpp:71-113)."""

    def __init__(self, ctx: Context, A: DeviceMatrix, start, max_cols: int):
        flat, (n, r) = _fcol(start)
        self.ctx, self.A, self.n, self.r, self.max_cols = ctx, A, n, r, max_cols
        h = C.c_void_p()
        check(lib().flz_basis_create(ctx.handle, A.handle, max_cols, r, flat, C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().flz_basis_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def blocks(self) -> int:
        return int(lib().flz_basis_blocks(self.handle))

    def step(self, coeffs=None, c=0.0, e=1.0):
        r = self.r
        Dk, Sk = np.zeros(r * r), np.zeros(r * r)
        dead = np.zeros(r, np.uint8)
        scale = C.c_double()
        if coeffs is None:
            cf, m = None, -1
        else:
            cfa = np.ascontiguousarray(coeffs, np.float64)
            cf, m = _ptr(cfa), len(cfa) - 1
        check(lib().flz_lanczos_step(self.ctx.handle, self.A.handle, self.handle, cf, m, c, e, Dk,
                                     Sk, C.byref(scale), dead))
        return Dk.reshape(r, r), Sk.reshape(r, r), scale.value, dead

    def get(self, j0, count):
        out = np.empty(self.n * count)
        check(lib().flz_basis_get(self.ctx.handle, self.handle, j0, count, out))
        return _from_fcol(out, self.n, count)

    def set(self, j, col):
        check(lib().flz_basis_set(self.ctx.handle, self.handle, j,
                                  np.ascontiguousarray(col, np.float64)))

    def ortho_error(self, dead=None) -> float:
        out = C.c_double()
        dp = None if dead is None else _ptr(np.ascontiguousarray(dead, np.uint8))
        check(lib().flz_basis_ortho_error(self.ctx.handle, self.handle, dp, C.byref(out)))
        return out.value

    def times(self):
        a, b = C.c_double(), C.c_double()
        check(lib().flz_basis_times(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    def ritz_lift(self, W):
        flat, (dim, w) = _fcol(W)
        vnorm, keep = np.zeros(max(w, 1)), np.zeros(max(w, 1), np.uint8)
        wk = C.c_int()
        Bm = np.zeros(max(w * w, 1))
        check(lib().flz_ritz_lift(self.ctx.handle, self.A.handle, self.handle, dim, flat, w, vnorm,
                                  keep, C.byref(wk), Bm))
        k = wk.value
        return vnorm[:w], keep[:w], Bm[: k * k].reshape(k, k).T

    def ritz_rotate(self, U, lam, scale=1.0, want_vectors=True):
        flat, (wk, w2) = _fcol(U)
        lam = np.ascontiguousarray(lam, np.float64)
        res = np.zeros(max(w2, 1))
        vec = np.empty(self.n * w2) if want_vectors else None
        check(lib().flz_ritz_rotate(self.ctx.handle, self.handle, flat, lam, w2, scale, res,
                                    _ptr(vec) if want_vectors else None))
        return res[:w2], (_from_fcol(vec, self.n, w2) if want_vectors else None)
