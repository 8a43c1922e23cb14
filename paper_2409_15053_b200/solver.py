"""Python mirror of the reference's solver API over the host layer of libflz
(include/flz_solver.h).  Names follow speig (lanczos.hpp / filter.hpp / sparse.hpp) so the
parity tests read like the reference's own tests.  Every compute call lands in libflz.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import FlzConfig, FlzStats, check, lib
from .device import _fcol, _from_fcol, _ptr


def LanczosConfig(block_size=3, tol=1e-10, max_dim=0, check_every=10, seed=20177, extra_ritz=5,
                  bounds_steps=50, degree=0, epsilon=0.255, max_degree=1000,
                  collect_diagnostics=False, return_vectors=True,
                  jackson_damping=False) -> FlzConfig:
    """speig::LanczosConfig defaults (lanczos.hpp:14-29); degree<=0 / None = automatic.
    ``return_vectors=False`` (extension) keeps the eigenvectors off the host;
    ``jackson_damping=True`` (extension, the reference has no damping) Jackson-damps the
    filter coefficients on the host."""
    return FlzConfig(block_size, tol, max_dim, check_every, seed, extra_ritz, bounds_steps,
                     int(degree or 0), epsilon, max_degree, int(collect_diagnostics),
                     int(return_vectors), int(jackson_damping))


@dataclass
class EigenResult:
    eigenvalues: np.ndarray
    residuals: np.ndarray
    eigenvectors: np.ndarray | None
    stats: dict = field(default_factory=dict)


class SparseSymMatrix:
    """speig::SparseSymMatrix (sparse.hpp:21-60): validated host CSR + lazy device copy."""

    def __init__(self, handle):
        self.handle = handle
        n, nnz = C.c_int64(), C.c_int64()
        lib().flz_hostmatrix_dims(handle, C.byref(n), C.byref(nnz))
        self.n, self.nnz = n.value, nnz.value

    @classmethod
    def from_entries(cls, n, rows, cols, values):
        rows = np.ascontiguousarray(rows, np.int64)
        h = C.c_void_p()
        check(lib().flz_hostmatrix_from_triplets(n, len(rows), rows,
                                                 np.ascontiguousarray(cols, np.int64),
                                                 np.ascontiguousarray(values, np.float64),
                                                 C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr(cls, n, row_ptr, col_idx, values, check_symmetry=True):
        h = C.c_void_p()
        check(lib().flz_hostmatrix_from_csr(n, np.ascontiguousarray(row_ptr, np.int64),
                                            np.ascontiguousarray(col_idx, np.int32),
                                            np.ascontiguousarray(values, np.float64),
                                            int(check_symmetry), C.byref(h)))
        return cls(h)

    @classmethod
    def from_local_rows(cls, n_global, row_begin, row_end, row_ptr, col_idx, values):
        """Distributed construction: this rank's row slab (row_ptr starts at 0)."""
        h = C.c_void_p()
        check(lib().flz_hostmatrix_from_local_rows(
            n_global, row_begin, row_end, np.ascontiguousarray(row_ptr, np.int64),
            np.ascontiguousarray(col_idx, np.int32), np.ascontiguousarray(values, np.float64),
            C.byref(h)))
        return cls(h)

    @classmethod
    def load_matrix_market(cls, path):
        h = C.c_void_p()
        check(lib().flz_hostmatrix_load_mm(str(path).encode(), C.byref(h)))
        return cls(h)

    def save_matrix_market(self, path):
        check(lib().flz_hostmatrix_save_mm(self.handle, str(path).encode()))

    @classmethod
    def load_binary(cls, path):
        """Binary CSR image written by save_binary (or by the FLZ_MM_CACHE of the loader)."""
        h = C.c_void_p()
        check(lib().flz_hostmatrix_load_bin(str(path).encode(), C.byref(h)))
        return cls(h)

    def save_binary(self, path):
        check(lib().flz_hostmatrix_save_bin(self.handle, str(path).encode()))

    def layout(self):
        """Device layout (uploads the matrix if needed): bytes the fused Clenshaw step streams
        for the matrix, and the nonzeros held at uniform-offset positions."""
        mb, ue = C.c_int64(), C.c_int64()
        check(lib().flz_hostmatrix_layout(self.handle, C.byref(mb), C.byref(ue)))
        out = {"matrix_bytes": mb.value, "uniform_entries": ue.value, "step_bytes": []}
        info = (C.c_int64 * 4)()
        name = C.create_string_buffer(96)
        for r in (1, 2, 3, 4):   # bytes one fused step of r columns streams, and its kernel
            check(lib().flz_hostmatrix_k1_info(self.handle, r, info, name, 96))
            out["step_bytes"].append(int(info[0]))
            if r == 3:
                out["kernel"] = name.value.decode()
                out["dense_blocks"], out["dense_entries"] = int(info[1]), int(info[2])
        return out

    def csr(self):
        rp = np.empty(self.n + 1, np.int64)
        ci = np.empty(self.nnz, np.int32)
        va = np.empty(self.nnz, np.float64)
        check(lib().flz_hostmatrix_csr(self.handle, rp, ci, va))
        return rp, ci, va

    def spmm_block(self, X):
        flat, (n, r) = _fcol(X)
        out = np.empty_like(flat)
        check(lib().flz_hostmatrix_spmm(self.handle, flat, n, r, out))
        return _from_fcol(out, n, r)

    def filter_apply(self, coeffs, lo, hi, X):
        flat, (n, r) = _fcol(X)
        cf = np.ascontiguousarray(coeffs, np.float64)
        out = np.empty_like(flat)
        check(lib().flz_hostmatrix_filter_apply(self.handle, cf, len(cf) - 1, lo, hi, flat, n, r,
                                                out))
        return _from_fcol(out, n, r)

    def __del__(self):
        try:
            lib().flz_hostmatrix_free(self.handle)
        except Exception:
            pass


def matvec_count() -> int:
    return int(lib().flz_matvec_count())


def indicator_coefficients(a, b, degree):
    out = np.empty(degree + 1)
    check(lib().flz_indicator_coefficients(a, b, degree, out))
    return out


def jackson_factors(degree):
    """Jackson kernel factors g_0..g_degree (extension: the reference has no damping)."""
    out = np.empty(degree + 1)
    check(lib().flz_jackson_factors(degree, out))
    return out


def select_degree(a, b, eps=0.255, max_degree=1000):
    cl = C.c_int(0)
    m = lib().flz_select_degree(a, b, eps, max_degree, C.byref(cl))
    if m < 0:
        check(m)
    return m, bool(cl.value)


def clenshaw(coeffs, t):
    c = np.ascontiguousarray(coeffs, np.float64)
    return float(lib().flz_clenshaw(c, len(c), t))


def build_filter(lo, hi, alpha, beta, degree=0, eps=0.255, max_degree=1000):
    """-> (coeffs, alpha_s, beta_s, clamped), build_filter (filter.cpp:163-184)."""
    a, b, cl = C.c_double(), C.c_double(), C.c_int()
    m = lib().flz_build_filter(lo, hi, alpha, beta, int(degree or 0), eps, max_degree, None, 0,
                               C.byref(a), C.byref(b), C.byref(cl))
    if m < 0:
        check(m)
    coeffs = np.empty(m + 1)
    lib().flz_build_filter(lo, hi, alpha, beta, m, eps, max_degree, _ptr(coeffs), m + 1, None,
                           None, None)
    return coeffs, a.value, b.value, bool(cl.value)


def init_block(n, r, seed=20177):
    Q = np.empty(n * r)
    check(lib().flz_init_block(n, r, seed, Q))
    return _from_fcol(Q, n, r)


def estimate_spectral_bounds(A: SparseSymMatrix, steps=50, seed=20177):
    lo, hi = C.c_double(), C.c_double()
    check(lib().flz_estimate_bounds(A.handle, steps, seed, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def sym_band_eig(bands, want_vectors=True):
    bands = np.ascontiguousarray(bands, np.float64)
    sb, dim = bands.shape[0] - 1, bands.shape[1]
    values = np.empty(dim)
    vec = np.empty(dim * dim) if want_vectors else None
    check(lib().flz_sym_band_eig(dim, sb, bands.ravel(), values,
                                 _ptr(vec) if want_vectors else None))
    return values, (_from_fcol(vec, dim, dim) if want_vectors else None)


def band_ritz_rows(bands, rows):
    bands = np.ascontiguousarray(bands, np.float64)
    sb, dim = bands.shape[0] - 1, bands.shape[1]
    rows = np.ascontiguousarray(rows, np.int64)
    values = np.empty(dim)
    out = np.empty(max(len(rows), 1) * dim)
    check(lib().flz_band_ritz_rows(dim, sb, bands.ravel(), len(rows), rows, values, _ptr(out)))
    return values, out[: len(rows) * dim].reshape(dim, len(rows)).T


def band_eigenvectors(bands, values, pick):
    bands = np.ascontiguousarray(bands, np.float64)
    sb, dim = bands.shape[0] - 1, bands.shape[1]
    pick = np.ascontiguousarray(pick, np.int64)
    vec = np.empty(dim * max(len(pick), 1))
    res, ortho = C.c_double(), C.c_double()
    check(lib().flz_band_eigenvectors(dim, sb, bands.ravel(),
                                      np.ascontiguousarray(values, np.float64), len(pick), pick,
                                      vec, C.byref(res), C.byref(ortho)))
    return _from_fcol(vec[: dim * len(pick)], dim, len(pick)), res.value, ortho.value


class LanczosFactorization:
    """speig::LanczosFactorization + expand + check_convergence (lanczos.cpp:105-405)."""

    def __init__(self, A: SparseSymMatrix, start, max_cols, coeffs=None, bounds=(0.0, 1.0),
                 interval=(0.0, 1.0)):
        flat, (n, r) = _fcol(start)
        self.A, self.n, self.r = A, n, r
        m = -1 if coeffs is None else len(coeffs) - 1
        cf = np.ascontiguousarray(coeffs if coeffs is not None else [0.0], np.float64)
        h = C.c_void_p()
        check(lib().flz_fact_create(A.handle, cf, m, bounds[0], bounds[1], interval[0],
                                    interval[1], flat, r, int(max_cols), C.byref(h)))
        self.handle = h

    def expand(self, nblocks):
        added = lib().flz_fact_expand(self.handle, nblocks)
        if added < 0:
            check(added)
        return added

    @property
    def block_count(self):
        return int(lib().flz_fact_block_count(self.handle))

    def get(self):
        k, r, n = self.block_count, self.r, self.n
        basis = np.empty(n * (k * r + r))
        D = np.empty(max(k, 1) * r * r)
        S = np.empty(max(k, 1) * r * r)
        dead = np.empty(k * r + r, np.uint8)
        check(lib().flz_fact_get(self.handle, _ptr(basis), _ptr(D), _ptr(S), _ptr(dead)))
        return (_from_fcol(basis, n, k * r + r), D[: k * r * r].reshape(k, r, r),
                S[: k * r * r].reshape(k, r, r), dead)

    def ortho_error(self):
        out = C.c_double()
        check(lib().flz_fact_ortho_error(self.handle, C.byref(out)))
        return out.value

    def flags(self):
        return int(lib().flz_fact_flags(self.handle))

    def check(self, alpha, beta, tol=1e-10, extra_ritz=5):
        dim = self.block_count * self.r
        values, est = np.empty(dim), np.empty(dim)
        wanted, dead = np.empty(dim, np.uint8), np.empty(dim, np.uint8)
        conv = lib().flz_fact_check(self.handle, alpha, beta, tol, extra_ritz, values, est, wanted,
                                    dead)
        if conv < 0:
            check(conv)
        return bool(conv), values, est, wanted, dead

    def __del__(self):
        try:
            lib().flz_fact_free(self.handle)
        except Exception:
            pass


class _ResultOwner:
    """Keeps a flz_result alive for as long as NumPy views of its eigenvectors exist."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            lib().flz_result_free(self.handle)
        except Exception:
            pass


def _solve(A: SparseSymMatrix, alpha, beta, cfg, plain, want_vectors):
    cfg = cfg or LanczosConfig()
    if not want_vectors and cfg.return_vectors:   # do not even download them
        cfg = FlzConfig(*[getattr(cfg, k) for k, _ in FlzConfig._fields_])
        cfg.return_vectors = 0
    h = C.c_void_p()
    check(lib().flz_solve(A.handle, alpha, beta, C.byref(cfg), int(plain), C.byref(h)))
    owner = _ResultOwner(h)
    cnt = int(lib().flz_result_count(h))
    ev, res = np.empty(cnt), np.empty(cnt)
    st = FlzStats()
    check(lib().flz_result_get(h, _ptr(ev), _ptr(res), None, C.byref(st)))
    vec = None
    if want_vectors and cfg.return_vectors:
        rows = int(lib().flz_result_rows(h))
        if cnt * rows:
            # zero-copy view of the result's own storage; the view keeps the result alive
            buf = (C.c_double * (rows * cnt)).from_address(lib().flz_result_vectors(h))
            buf._owner = owner
            vec = np.frombuffer(buf, dtype=np.float64).reshape(cnt, rows).T
        else:
            vec = np.empty((rows, cnt))
    stats = {k: getattr(st, k) for k, _ in FlzStats._fields_}
    return EigenResult(ev, res, vec, stats)


def filtered_lanczos(A, alpha, beta, cfg=None, want_vectors=True) -> EigenResult:
    """speig::filtered_lanczos (lanczos.hpp:183-184)."""
    return _solve(A, alpha, beta, cfg, False, want_vectors)


def plain_lanczos(A, alpha, beta, cfg=None, want_vectors=True) -> EigenResult:
    """speig::plain_lanczos (lanczos.hpp:185-186)."""
    return _solve(A, alpha, beta, cfg, True, want_vectors)
