"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes front-end for the two CPU oracles of the filter-and-Lanczos path:

* ``load("ref")``  -> oracle/_ref/libspeig_ref.so: the UNMODIFIED reference library
  (``/root/reference/proj/src``) behind the C ABI of ``oracle_abi.h`` (kind "reference");
* ``load("port")`` -> oracle/_build/libflz_oracle.so: the plain-C restatement
  ``flz_oracle.c`` (kind "port").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2409_15053_b200`` never does (tests/test_boundary.py greps for it).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/proj"

_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class OrcConfig(C.Structure):
    """Mirror of ``orc_config`` / ``speig::LanczosConfig`` (lanczos.hpp:14-29)."""

    _fields_ = [
        ("block_size", C.c_int32),
        ("tol", C.c_double),
        ("max_dim", C.c_int32),
        ("check_every", C.c_int32),
        ("seed", C.c_uint64),
        ("extra_ritz", C.c_int32),
        ("bounds_steps", C.c_int32),
        ("degree", C.c_int32),
        ("epsilon", C.c_double),
        ("max_degree", C.c_int32),
        ("collect_diagnostics", C.c_int32),
    ]


class OrcStats(C.Structure):
    """Mirror of ``orc_stats`` / ``speig::SolveStats`` (lanczos.hpp:136-155)."""

    _fields_ = [
        ("block_steps", C.c_int32),
        ("basis_vectors", C.c_int32),
        ("degree", C.c_int32),
        ("mv_iteration", C.c_uint64),
        ("mv_bounds", C.c_uint64),
        ("mv_total", C.c_uint64),
        ("time_total_s", C.c_double),
        ("time_preproc_s", C.c_double),
        ("time_orth_s", C.c_double),
        ("time_mv_s", C.c_double),
        ("checks", C.c_int32),
        ("converged", C.c_int32),
        ("breakdown_replacements", C.c_int32),
        ("degree_clamped", C.c_int32),
        ("norm_estimate", C.c_double),
        ("lambda_min_est", C.c_double),
        ("lambda_max_est", C.c_double),
        ("ortho_error", C.c_double),
    ]


def make_config(block_size=3, tol=1e-10, max_dim=0, check_every=10, seed=20177, extra_ritz=5,
                bounds_steps=50, degree=0, epsilon=0.255, max_degree=1000,
                collect_diagnostics=False) -> OrcConfig:
    """Reference defaults (lanczos.hpp:14-29); degree<=0 means automatic."""
    return OrcConfig(block_size, tol, max_dim, check_every, seed, extra_ritz, bounds_steps,
                     int(degree or 0), epsilon, max_degree, int(collect_diagnostics))


class OracleError(RuntimeError):
    pass


@dataclass
class SolveResult:
    eigenvalues: np.ndarray
    residuals: np.ndarray
    eigenvectors: np.ndarray  # n x count, column-major semantics (Fortran-ordered array)
    stats: dict = field(default_factory=dict)


class Matrix:
    def __init__(self, orc: "Oracle", handle):
        self.orc, self.handle = orc, handle
        self.n = int(orc._f("matrix_dim")(handle))
        self.nnz = int(orc._f("matrix_nnz")(handle))

    def csr(self):
        rp = np.empty(self.n + 1, np.int64)
        ci = np.empty(self.nnz, np.int32)
        va = np.empty(self.nnz, np.float64)
        self.orc._f("matrix_csr")(self.handle, rp, ci, va)
        return rp, ci, va

    def __del__(self):
        try:
            self.orc._f("matrix_free")(self.handle)
        except Exception:
            pass


class Factorization:
    """LanczosFactorization + expand (lanczos.cpp:105-271)."""

    def __init__(self, orc, A: Matrix, start, max_cols, coeffs=None, bounds=(0.0, 1.0),
                 interval=(0.0, 1.0)):
        self.orc, self.A = orc, A
        start = np.asfortranarray(start, dtype=np.float64)
        self.n, self.r = start.shape
        m = -1 if coeffs is None else len(coeffs) - 1
        cf = np.ascontiguousarray(coeffs if coeffs is not None else [0.0], dtype=np.float64)
        self.handle = orc._f("fact_create")(A.handle, cf, m, bounds[0], bounds[1], interval[0],
                                            interval[1], start.ravel(order="F"), self.r,
                                            int(max_cols))
        if not self.handle:
            raise OracleError(orc.last_error())

    def expand(self, nblocks: int) -> int:
        added = self.orc._f("fact_expand")(self.handle, nblocks)
        if added < 0:
            raise OracleError(self.orc.last_error())
        return added

    @property
    def block_count(self) -> int:
        return int(self.orc._f("fact_block_count")(self.handle))

    def get(self):
        k, r, n = self.block_count, self.r, self.n
        basis = np.empty(n * (k * r + r), np.float64)
        D = np.empty(max(k, 1) * r * r, np.float64)
        S = np.empty(max(k, 1) * r * r, np.float64)
        dead = np.empty(k * r + r, np.uint8)
        self.orc._f("fact_get")(self.handle, basis, D, S, dead)
        return (basis.reshape((n, k * r + r), order="F"), D[: k * r * r].reshape(k, r, r),
                S[: k * r * r].reshape(k, r, r), dead)

    def ortho_error(self) -> float:
        return float(self.orc._f("fact_ortho_error")(self.handle))

    def flags(self) -> int:
        return int(self.orc._f("fact_flags")(self.handle))

    def check(self, alpha, beta, tol=1e-10, extra_ritz=5):
        dim = self.block_count * self.r
        values = np.empty(dim)
        est = np.empty(dim)
        wanted = np.empty(dim, np.uint8)
        dead = np.empty(dim, np.uint8)
        conv = self.orc._f("fact_check")(self.handle, alpha, beta, tol, extra_ritz, values, est,
                                         wanted, dead)
        if conv < 0:
            raise OracleError(self.orc.last_error())
        return bool(conv), values, est, wanted, dead

    def __del__(self):
        try:
            self.orc._f("fact_free")(self.handle)
        except Exception:
            pass


class Oracle:
    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path
        self._sig()
        self.kind = self._f("kind")().decode()

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _sig(self):
        d, i64, i32, vp = C.c_double, C.c_int64, C.c_int, C.c_void_p
        S = {
            "last_error": (C.c_char_p, []),
            "kind": (C.c_char_p, []),
            "set_backend": (i32, [i32]),
            "get_backend": (i32, []),
            "dot": (d, [_f64p, _f64p, i64]),
            "nrm2": (d, [_f64p, i64]),
            "axpy": (None, [d, _f64p, _f64p, i64]),
            "scal": (None, [d, _f64p, i64]),
            "csr_matvec": (None, [i64, _i64p, _i32p, _f64p, _f64p, _f64p]),
            "clenshaw_combine": (None, [i64, d, d, d, _f64p, _f64p, _f64p, _f64p, _f64p]),
            "indicator_coefficients": (i32, [d, d, i32, _f64p]),
            "select_degree": (i32, [d, d, d, i32, C.POINTER(C.c_int)]),
            "clenshaw": (d, [_f64p, i32, d]),
            "matrix_from_csr": (vp, [i64, _i64p, _i32p, _f64p]),
            "matrix_from_triplets": (vp, [i64, i64, _i64p, _i64p, _f64p]),
            "matrix_free": (None, [vp]),
            "matrix_dim": (i64, [vp]),
            "matrix_nnz": (i64, [vp]),
            "matrix_csr": (None, [vp, _i64p, _i32p, _f64p]),
            "matvec_count": (C.c_uint64, []),
            "filter_apply": (i32, [vp, _f64p, i32, d, d, _f64p, i32, _f64p]),
            "build_filter": (i32, [d, d, d, d, i32, d, i32, C.c_void_p, i32, C.POINTER(d),
                                   C.POINTER(d), C.POINTER(C.c_int)]),
            "init_block": (i32, [i64, i32, C.c_uint64, _f64p]),
            "estimate_bounds": (i32, [vp, i32, C.c_uint64, C.POINTER(d), C.POINTER(d)]),
            "sym_band_eig": (i32, [i64, i64, _f64p, _f64p, C.c_void_p]),
            "fact_create": (vp, [vp, _f64p, i32, d, d, d, d, _f64p, i32, i64]),
            "fact_free": (None, [vp]),
            "fact_expand": (i32, [vp, i32]),
            "fact_block_count": (i64, [vp]),
            "fact_get": (None, [vp, _f64p, _f64p, _f64p, _u8p]),
            "fact_ortho_error": (d, [vp]),
            "fact_flags": (i32, [vp]),
            "fact_check": (i32, [vp, d, d, d, i32, _f64p, _f64p, _u8p, _u8p]),
            "solve": (vp, [vp, d, d, C.POINTER(OrcConfig), i32]),
            "result_free": (None, [vp]),
            "result_count": (i64, [vp]),
            "result_get": (None, [vp, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(OrcStats)]),
        }
        for name, (res, args) in S.items():
            fn = self._f(name)
            fn.restype, fn.argtypes = res, args

    # ---- helpers -------------------------------------------------------
    def last_error(self) -> str:
        return self._f("last_error")().decode()

    def set_backend(self, name: str):
        if self._f("set_backend")(1 if name == "avx2" else 0) != 0:
            raise OracleError(self.last_error())

    def backend(self) -> str:
        return "avx2" if self._f("get_backend")() == 1 else "scalar"

    def matvec_count(self) -> int:
        return int(self._f("matvec_count")())

    def matrix_from_csr(self, n, row_ptr, col_idx, values) -> Matrix:
        h = self._f("matrix_from_csr")(n, np.ascontiguousarray(row_ptr, np.int64),
                                       np.ascontiguousarray(col_idx, np.int32),
                                       np.ascontiguousarray(values, np.float64))
        if not h:
            raise OracleError(self.last_error())
        return Matrix(self, h)

    def load_matrix_market(self, path):
        """(n, row_ptr, col_idx, values) as the reference's own Matrix Market loader builds them
        (reference build only).  Runs in a fresh interpreter without NumPy: the reference's
        iostream-based loader crashes when it is called in a process that has loaded NumPy's
        bundled runtime libraries first."""
        import subprocess, sys, tempfile
        code = (
            "import ctypes as C, sys\n"
            "L = C.CDLL(sys.argv[1])\n"
            "f = L.ref_matrix_load_mm; f.restype = C.c_void_p; f.argtypes = [C.c_char_p]\n"
            "h = f(sys.argv[2].encode())\n"
            "e = L.ref_last_error; e.restype = C.c_char_p\n"
            "if not h: sys.exit('ERR ' + e().decode())\n"
            "d = L.ref_matrix_dim; d.restype = C.c_int64; d.argtypes = [C.c_void_p]\n"
            "z = L.ref_matrix_nnz; z.restype = C.c_int64; z.argtypes = [C.c_void_p]\n"
            "n, nnz = d(h), z(h)\n"
            "rp = (C.c_int64 * (n + 1))(); ci = (C.c_int32 * max(nnz, 1))(); va = (C.c_double * max(nnz, 1))()\n"
            "g = L.ref_matrix_csr; g.restype = None; g.argtypes = [C.c_void_p] * 4\n"
            "g(h, rp, ci, va)\n"
            "open(sys.argv[3], 'wb').write(bytes(C.c_int64(n)) + bytes(C.c_int64(nnz)) + bytes(rp) + bytes(ci)[:4 * nnz] + bytes(va)[:8 * nnz])\n")
        with tempfile.NamedTemporaryFile(suffix=".bin") as out:
            r = subprocess.run([sys.executable, "-S", "-c", code, self.path, str(path), out.name],
                               capture_output=True, text=True, timeout=600)
            if r.returncode != 0:
                raise OracleError(r.stderr.strip()[-500:])
            raw = open(out.name, "rb").read()
        n, nnz = np.frombuffer(raw, np.int64, 2)
        rp = np.frombuffer(raw, np.int64, n + 1, 16)
        ci = np.frombuffer(raw, np.int32, nnz, 16 + 8 * (n + 1))
        va = np.frombuffer(raw, np.float64, nnz, 16 + 8 * (n + 1) + 4 * nnz)
        return int(n), rp, ci, va

    def matrix_from_triplets(self, n, rows, cols, values) -> Matrix:
        rows = np.ascontiguousarray(rows, np.int64)
        h = self._f("matrix_from_triplets")(n, len(rows), rows,
                                            np.ascontiguousarray(cols, np.int64),
                                            np.ascontiguousarray(values, np.float64))
        if not h:
            raise OracleError(self.last_error())
        return Matrix(self, h)

    def csr_matvec(self, n, row_ptr, col_idx, values, x):
        y = np.empty(n)
        self._f("csr_matvec")(n, np.ascontiguousarray(row_ptr, np.int64),
                              np.ascontiguousarray(col_idx, np.int32),
                              np.ascontiguousarray(values, np.float64),
                              np.ascontiguousarray(x, np.float64), y)
        return y

    def clenshaw_combine(self, s1, s2, b, w, y1, y2, x):
        out = np.empty_like(w)
        self._f("clenshaw_combine")(len(w), s1, s2, b, w, y1, y2, x, out)
        return out

    def indicator_coefficients(self, a, b, degree):
        out = np.empty(degree + 1)
        if self._f("indicator_coefficients")(a, b, degree, out) != 0:
            raise OracleError(self.last_error())
        return out

    def select_degree(self, a, b, eps=0.255, max_degree=1000):
        cl = C.c_int(0)
        m = self._f("select_degree")(a, b, eps, max_degree, C.byref(cl))
        if m < 0:
            raise OracleError(self.last_error())
        return m, bool(cl.value)

    def clenshaw(self, coeffs, t):
        c = np.ascontiguousarray(coeffs, np.float64)
        return float(self._f("clenshaw")(c, len(c), t))

    def build_filter(self, lo, hi, alpha, beta, degree=0, eps=0.255, max_degree=1000):
        """-> (coeffs, alpha_s, beta_s, clamped) following build_filter (filter.cpp:163-184)."""
        a, b, cl = C.c_double(), C.c_double(), C.c_int()
        m = self._f("build_filter")(lo, hi, alpha, beta, int(degree or 0), eps, max_degree, None, 0,
                                    C.byref(a), C.byref(b), C.byref(cl))
        if m < 0:
            raise OracleError(self.last_error())
        coeffs = np.empty(m + 1)
        self._f("build_filter")(lo, hi, alpha, beta, m, eps, max_degree,
                                coeffs.ctypes.data_as(C.c_void_p), m + 1, None, None, None)
        return coeffs, a.value, b.value, bool(cl.value)

    def filter_apply(self, A: Matrix, coeffs, lo, hi, X):
        X = np.asfortranarray(X, dtype=np.float64)
        n, r = X.shape
        Y = np.empty(n * r)
        cf = np.ascontiguousarray(coeffs, np.float64)
        if self._f("filter_apply")(A.handle, cf, len(cf) - 1, lo, hi, X.ravel(order="F"), r, Y):
            raise OracleError(self.last_error())
        return Y.reshape((n, r), order="F")

    def init_block(self, n, r, seed=20177):
        Q = np.empty(n * r)
        if self._f("init_block")(n, r, seed, Q) != 0:
            raise OracleError(self.last_error())
        return Q.reshape((n, r), order="F")

    def estimate_bounds(self, A: Matrix, steps=50, seed=20177):
        lo, hi = C.c_double(), C.c_double()
        if self._f("estimate_bounds")(A.handle, steps, seed, C.byref(lo), C.byref(hi)) != 0:
            raise OracleError(self.last_error())
        return lo.value, hi.value

    def sym_band_eig(self, bands, want_vectors=True):
        """bands: (sb+1, dim) array with bands[d, i] = M(i+d, i)."""
        bands = np.ascontiguousarray(bands, np.float64)
        sb, dim = bands.shape[0] - 1, bands.shape[1]
        values = np.empty(dim)
        vec = np.empty(dim * dim) if want_vectors else None
        rc = self._f("sym_band_eig")(dim, sb, bands.ravel(), values,
                                     vec.ctypes.data_as(C.c_void_p) if want_vectors else None)
        if rc != 0:
            raise OracleError(self.last_error())
        return values, (vec.reshape((dim, dim), order="F") if want_vectors else None)

    def factorization(self, A, start, max_cols, coeffs=None, bounds=(0.0, 1.0),
                      interval=(0.0, 1.0)) -> Factorization:
        return Factorization(self, A, start, max_cols, coeffs, bounds, interval)

    def solve(self, A: Matrix, alpha, beta, cfg: OrcConfig | None = None, plain=False,
              want_vectors=True) -> SolveResult:
        cfg = cfg or make_config()
        h = self._f("solve")(A.handle, alpha, beta, C.byref(cfg), int(plain))
        if not h:
            raise OracleError(self.last_error())
        try:
            cnt = int(self._f("result_count")(h))
            ev, res = np.empty(cnt), np.empty(cnt)
            vec = np.empty(A.n * cnt) if want_vectors else None
            st = OrcStats()
            self._f("result_get")(h, ev.ctypes.data_as(C.c_void_p), res.ctypes.data_as(C.c_void_p),
                                  vec.ctypes.data_as(C.c_void_p) if want_vectors else None,
                                  C.byref(st))
        finally:
            self._f("result_free")(h)
        stats = {k: getattr(st, k) for k, _ in OrcStats._fields_}
        return SolveResult(ev, res, vec.reshape((A.n, cnt), order="F") if want_vectors else None,
                           stats)


def build(which=("port", "ref"), quiet=True):
    """Compile the oracles (the checker, not the product).  ``ref`` is a no-op when
    /root/reference is absent (GPU box): the prebuilt oracle/_ref/*.so travels."""
    for target in which:
        subprocess.run(["make", "-C", HERE, target], check=True,
                       stdout=subprocess.DEVNULL if quiet else None)


def available(which: str) -> bool:
    return os.path.exists(_path(which))


def _path(which: str) -> str:
    if which == "ref":
        return os.path.join(HERE, "_ref", "libspeig_ref.so")
    if which == "port":
        return os.path.join(HERE, "_build", "libflz_oracle.so")
    raise ValueError(which)


_cache: dict = {}


def load(which: str = "ref") -> Oracle:
    """``ref`` = compiled unmodified reference, ``port`` = plain-C restatement."""
    if which not in _cache:
        if not available(which):
            build((which,))
        if not available(which):
            raise OracleError(f"oracle '{which}' is not built and cannot be built here")
        _cache[which] = Oracle(_path(which), "ref_" if which == "ref" else "orc_")
    return _cache[which]


def best() -> Oracle:
    """The real reference when its .so exists, else the port."""
    return load("ref") if (available("ref") or os.path.isdir(REF_SRC)) else load("port")
