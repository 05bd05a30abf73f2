"""TEST INFRASTRUCTURE ONLY — ctypes view of the REFERENCE's own MIDBF code.

oracle/_ref/libmidbf_ref.so is /root/reference/proj/src compiled unmodified
against the Eigen stand-in in oracle/shim/ (recipe: oracle/ref.mk; C ABI:
oracle/ref_capi.cpp).  Only tests/ and tests/golden/make_golden.py use it, to
pin the oracle restatement and the product against the reference's code.
The built files travel to the GPU box; /root/reference itself does not, so
build() is a no-op there when the files exist.

Arrays follow oracle.py: points row-major (N, dim) float64, complex vectors
complex128, multi-RHS column-major (N, nrhs).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import tempfile

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "_ref", "libmidbf_ref.so")
UNIT_TESTS = os.path.join(_HERE, "_ref", "ref_unit_tests")
REF_SRC = "/root/reference/proj"

KIND_FIO2D, KIND_FIO3D, KIND_LOWRANK, KIND_NUFFT, KIND_CONST, KIND_RANK1 = range(6)

i64 = C.c_int64
u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int64)


def available():
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC)


def build():
    """(Re)build oracle/_ref from the reference sources when they are here."""
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j16", "-f", os.path.join("oracle", "ref.mk")], cwd=_ROOT, check=True)
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} missing and {REF_SRC} absent: build it where the reference is")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC):
            build()
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mock_cheb_points.restype = i64
        L.ref_rand_subset.restype = i64
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(dptr)


def _ip(a):
    return a.ctypes.data_as(iptr)


def _check(rc):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise AssertionError(msg)
    raise RuntimeError(msg)


class Problem:
    """Points + kernel description, as the reference's entry evaluators see them."""

    def __init__(self, kind, X, Omega, A=None, B=None, const=0j, u=None, v=None):
        self.kind = kind
        self.X = np.ascontiguousarray(X, dtype=np.float64)
        self.Omega = np.ascontiguousarray(Omega, dtype=np.float64)
        self.dim = self.X.shape[1]
        self.A = None if A is None else np.ascontiguousarray(A, dtype=np.float64)
        self.B = None if B is None else np.ascontiguousarray(B, dtype=np.float64)
        self.rank = 0 if A is None else self.A.shape[1]
        self.const = np.array([complex(const).real, complex(const).imag])
        self.u = None if u is None else np.ascontiguousarray(u, dtype=np.complex128)
        self.v = None if v is None else np.ascontiguousarray(v, dtype=np.complex128)

    def _args(self):
        return (self.kind, _p(self.X), i64(len(self.X)), _p(self.Omega), i64(len(self.Omega)), self.dim,
                _p(self.A), _p(self.B), self.rank)

    def factorize(self, n0, k=30, eps=1e-9, t=5, seed=0, parallel=True, path=None):
        """bf::idbf_factorize + bf::save_factorization; returns the MIDBF001 path."""
        if path is None:
            fd, path = tempfile.mkstemp(suffix=".midbf")
            os.close(fd)
        uu = None if self.u is None else self.u.view(np.float64)
        vv = None if self.v is None else self.v.view(np.float64)
        _check(lib().ref_factorize(*self._args(), _p(self.const), _p(uu), _p(vv), i64(n0), i64(k), C.c_double(eps),
                                   i64(t), u64(seed), 1 if parallel else 0, str(path).encode()))
        return path

    def entries(self, rows, cols):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(len(rows), dtype=np.complex128)
        _check(lib().ref_entries(*self._args(), _ip(rows), _ip(cols), i64(len(rows)), _p(out.view(np.float64))))
        return out

    def direct_sum(self, f, rows=None):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        rows = np.arange(len(self.X), dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
        out = np.empty(len(rows), dtype=np.complex128)
        _check(lib().ref_direct_sum(*self._args(), _p(f.view(np.float64)), _ip(rows), i64(len(rows)),
                                    _p(out.view(np.float64))))
        return out

    def eps_b(self, path, f, nrows=256, seed=0):
        """metrics::eps_b (src/metrics.cpp:26-53) of the stored factorization."""
        f = np.ascontiguousarray(f, dtype=np.complex128)
        out = C.c_double()
        _check(lib().ref_eps_b(str(path).encode(), *self._args(), _p(f.view(np.float64)), i64(nrows), u64(seed),
                               C.byref(out)))
        return out.value


def apply(path, f, transpose=False):
    """bf::apply / apply_transpose of a MIDBF001 container."""
    f = np.asarray(f, dtype=np.complex128)
    vec = f.ndim == 1
    F2 = np.asfortranarray(f.reshape(f.shape[0], -1))
    inf = info(path)
    nout = inf["ncols"] if transpose else inf["nrows"]
    g = np.empty((nout, F2.shape[1]), dtype=np.complex128, order="F")
    _check(lib().ref_apply(str(path).encode(), F2.ctypes.data_as(dptr), i64(F2.shape[0]), i64(F2.shape[1]),
                           1 if transpose else 0, g.ctypes.data_as(dptr)))
    return g[:, 0] if vec else g


class Loaded:
    """bf::load_factorization once, bf::apply many times (Exec as stored)."""

    def __init__(self, path):
        self._h = C.c_void_p()
        _check(lib().ref_load(str(path).encode(), C.byref(self._h)))
        self.info = info(path)

    def apply(self, f, transpose=False):
        f = np.asarray(f, dtype=np.complex128)
        vec = f.ndim == 1
        F2 = np.asfortranarray(f.reshape(f.shape[0], -1))
        nout = self.info["ncols"] if transpose else self.info["nrows"]
        g = np.empty((nout, F2.shape[1]), dtype=np.complex128, order="F")
        _check(lib().ref_apply_h(self._h, F2.ctypes.data_as(dptr), i64(F2.shape[0]), i64(F2.shape[1]),
                                 1 if transpose else 0, g.ctypes.data_as(dptr)))
        return g[:, 0] if vec else g

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().ref_free(self._h)
            except Exception:
                pass
            self._h = None


def info(path):
    o = np.zeros(8, dtype=np.int64)
    _check(lib().ref_info(str(path).encode(), _ip(o)))
    keys = ("nrows", "ncols", "L", "h", "n0", "nfactors", "total_nnz", "max_factor_nnz")
    return {k: int(v) for k, v in zip(keys, o)}


def build_tree(X, n0, min_depth=0):
    X = np.ascontiguousarray(X, dtype=np.float64)
    perm = np.empty(len(X), dtype=np.int64)
    depth = i64()
    _check(lib().ref_tree(_p(X), i64(len(X)), X.shape[1], i64(n0), min_depth, _ip(perm), C.byref(depth)))
    return perm, depth.value


def pivoted_qr(A, max_rank=-1):
    A = np.asfortranarray(A, dtype=np.complex128)
    m, n = A.shape
    perm = np.empty(n, dtype=np.int64)
    rank = i64()
    R = np.zeros((min(m, n), n), dtype=np.complex128, order="F")
    _check(lib().ref_pqr(A.ctypes.data_as(dptr), i64(m), i64(n), i64(max_rank), _ip(perm), C.byref(rank),
                         R.ctypes.data_as(dptr)))
    r = rank.value
    Rr = np.frombuffer(R.reshape(-1, order="F").tobytes(), dtype=np.complex128)[: r * n].reshape((r, n), order="F")
    return perm, r, Rr


def cid_from_rows(A, k_max, eps):
    A = np.asfortranarray(A, dtype=np.complex128)
    m, n = A.shape
    skel = np.empty(min(m, n) + 1, dtype=np.int64)
    V = np.zeros(n * (min(m, n) + 1), dtype=np.complex128)
    rank = i64()
    _check(lib().ref_cid(A.ctypes.data_as(dptr), i64(m), i64(n), i64(k_max), C.c_double(eps), _ip(skel),
                         _p(V.view(np.float64)), C.byref(rank)))
    r = rank.value
    return skel[:r].copy(), V[: r * n].reshape((r, n), order="F").copy()


def mock_chebyshev_points(P, s, seed):
    P = np.ascontiguousarray(P, dtype=np.float64)
    out = np.empty(max(s, len(P)), dtype=np.int64)
    n = lib().ref_mock_cheb_points(_p(P), i64(len(P)), P.shape[1], i64(s), u64(seed), _ip(out))
    return out[:n].copy()


def rand_subset(n, k, seed):
    out = np.empty(max(k, 1), dtype=np.int64)
    m = lib().ref_rand_subset(i64(n), i64(k), u64(seed), _ip(out))
    return out[:m].copy()


def grid2d(n):
    out = np.empty((n * n, 2), dtype=np.float64)
    lib().ref_grid2d(i64(n), _p(out))
    return out


def run_unit_tests(args=(), timeout=900):
    """The reference's own doctest suites (hot-path files) on its own code."""
    lib()  # builds when the sources are here
    return subprocess.run([UNIT_TESTS, *args], capture_output=True, text=True, timeout=timeout)
