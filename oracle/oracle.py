"""TEST INFRASTRUCTURE ONLY — ctypes view of the CPU oracle.

The oracle (orc_core.cpp) restates the reference MIDBF path on the CPU.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module; the product package never does.

Arrays: point sets are row-major (N, dim) float64; complex vectors are
complex128 (column-major (N, nrhs) for multi-RHS, i.e. Fortran order).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libmidbf_oracle.so")

KIND_FIO2D, KIND_FIO3D, KIND_LOWRANK, KIND_NUFFT, KIND_CONST, KIND_RANK1 = range(6)

i64 = C.c_int64
u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int64)
vp = C.c_void_p


class KernelDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("dim", C.c_int), ("rank", C.c_int),
        ("nrows", i64), ("ncols", i64),
        ("X", dptr), ("Omega", dptr), ("A", dptr), ("B", dptr),
        ("u", dptr), ("v", dptr), ("cre", C.c_double), ("cim", C.c_double),
    ]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_chain.restype = u64
        L.orc_chain.argtypes = [u64, u64]
        L.orc_tree_level_size.restype = i64
        L.orc_fac_nnz_bound.restype = C.c_double
        L.orc_fac_eps.restype = C.c_double
        L.orc_id_rank.restype = i64
        L.orc_mock_cheb_rows.restype = i64
        L.orc_mock_cheb_points.restype = i64
        L.orc_rand_subset.restype = i64
        L.orc_rand_subset_seq.restype = i64
        L.orc_fio2d_phase.restype = C.c_double
        L.orc_fio3d_phase.restype = C.c_double
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(dptr)


def _ip(a):
    return a.ctypes.data_as(iptr)


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise AssertionError(msg)
    raise RuntimeError(msg)


def chain(a, b):
    return int(lib().orc_chain(u64(a), u64(b)))


class Kernel:
    """Entry evaluator K(i,j) = exp(2*pi*i*Phi(x_i, xi_j)) (or test kernels)."""

    def __init__(self, kind, X=None, Omega=None, A=None, B=None, u=None, v=None, const=0j, nrows=None, ncols=None):
        self.kind = kind
        self._keep = []
        d = KernelDesc()
        d.kind = kind
        if X is not None:
            X = np.ascontiguousarray(X, dtype=np.float64)
            Omega = np.ascontiguousarray(Omega, dtype=np.float64)
            self._keep += [X, Omega]
            d.X, d.Omega = _p(X), _p(Omega)
            d.dim = X.shape[1]
            nrows, ncols = X.shape[0], Omega.shape[0]
        if A is not None:
            A = np.ascontiguousarray(A, dtype=np.float64)
            B = np.ascontiguousarray(B, dtype=np.float64)
            self._keep += [A, B]
            d.A, d.B = _p(A), _p(B)
            d.rank = A.shape[1]
            nrows, ncols = A.shape[0], B.shape[0]
        if u is not None:
            u = np.ascontiguousarray(u, dtype=np.complex128)
            v = np.ascontiguousarray(v, dtype=np.complex128)
            self._keep += [u, v]
            d.u, d.v = _p(u.view(np.float64)), _p(v.view(np.float64))
            nrows, ncols = len(u), len(v)
        d.cre, d.cim = complex(const).real, complex(const).imag
        d.nrows, d.ncols = nrows, ncols
        self.desc = d
        self.nrows, self.ncols = nrows, ncols

    def entries(self, rows, cols):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty(len(rows), dtype=np.complex128)
        _check(lib().orc_entries(C.byref(self.desc), _ip(rows), _ip(cols), i64(len(rows)), _p(out.view(np.float64))))
        return out

    def dense(self):
        r, c = np.meshgrid(np.arange(self.nrows), np.arange(self.ncols), indexing="ij")
        return self.entries(r.ravel(), c.ravel()).reshape(self.nrows, self.ncols)

    def direct_sum(self, f, rows=None, threads=0):
        f = np.ascontiguousarray(f, dtype=np.complex128)
        rows = np.arange(self.nrows, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(len(rows), dtype=np.complex128)
        _check(lib().orc_direct_sum(C.byref(self.desc), _p(f.view(np.float64)), _ip(rows), i64(len(rows)),
                                    _p(out.view(np.float64)), 1, threads))
        return out

    def eps_b(self, g_b, f, nrows=256, seed=0):
        g_b = np.ascontiguousarray(g_b, dtype=np.complex128)
        f = np.ascontiguousarray(f, dtype=np.complex128)
        out = C.c_double()
        _check(lib().orc_eps_b(_p(g_b.view(np.float64)), i64(len(g_b)), C.byref(self.desc), _p(f.view(np.float64)),
                               i64(len(f)), i64(nrows), u64(seed), C.byref(out)))
        return out.value


class Tree:
    def __init__(self, X, n0, min_depth=0):
        X = np.ascontiguousarray(X, dtype=np.float64)
        h = vp()
        _check(lib().orc_tree_build(_p(X), i64(X.shape[0]), X.shape[1], i64(n0), min_depth, C.byref(h)))
        self._h = h
        L = lib()
        self.dim = X.shape[1]
        self.depth = L.orc_tree_depth(h)
        self.perm = np.empty(X.shape[0], dtype=np.int64)
        L.orc_tree_perm(h, _ip(self.perm))
        self.levels = []
        for lv in range(self.depth + 1):
            n = L.orc_tree_level_size(h, lv)
            code = np.empty(n, dtype=np.uint64)
            b, e, p, nc = (np.empty(n, dtype=np.int64) for _ in range(4))
            ch = np.empty((n, 8), dtype=np.int64)
            L.orc_tree_level(h, lv, code.ctypes.data_as(C.POINTER(C.c_uint64)), _ip(b), _ip(e), _ip(p), _ip(nc),
                             _ip(ch))
            self.levels.append(dict(code=code, begin=b, end=e, parent=p, nchild=nc, child=ch))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_tree_free(self._h)
            self._h = None


class Factorization:
    """Owned oracle factorization handle (reference bf::Factorization)."""

    def __init__(self, handle):
        self._h = handle
        info = np.empty(12, dtype=np.int64)
        lib().orc_fac_info(handle, _ip(info))
        (self.nrows, self.ncols, self.L, self.h, self.n0, self.nfactors, self.total_nnz, self.max_factor_nnz,
         self.k_max, self.t, self.seed, self.parallel) = [int(v) for v in info]
        self.eps = lib().orc_fac_eps(handle)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_fac_free(self._h)
            self._h = None

    def nnz_bound(self, c=4.0):
        return lib().orc_fac_nnz_bound(self._h, C.c_double(c))

    def perms(self):
        rp = np.empty(self.nrows, dtype=np.int64)
        cp = np.empty(self.ncols, dtype=np.int64)
        lib().orc_fac_perms(self._h, _ip(rp), _ip(cp))
        return rp, cp

    def factor(self, i):
        """(rows, cols, blocks[nb,4] (row_off,col_off,m,n), groups[ng,2])."""
        o = np.empty(4, dtype=np.int64)
        lib().orc_fac_factor(self._h, i, _ip(o))
        rows, cols, nb, ng = (int(v) for v in o)
        blocks = np.empty((nb, 4), dtype=np.int64)
        groups = np.empty((ng, 2), dtype=np.int64)
        lib().orc_fac_tables(self._h, i, _ip(blocks), _ip(groups))
        return rows, cols, blocks, groups

    def block(self, i, b, m, n):
        out = np.empty((m, n), dtype=np.complex128, order="F")
        lib().orc_fac_block(self._h, i, i64(b), out.ctypes.data_as(dptr))
        return out

    def apply(self, f, transpose=False, parallel=True, threads=0):
        f = np.asarray(f, dtype=np.complex128)
        vec = f.ndim == 1
        F2 = np.asfortranarray(f.reshape(f.shape[0], -1))
        out = np.empty((self.ncols if transpose else self.nrows, F2.shape[1]), dtype=np.complex128, order="F")
        _check(lib().orc_apply(self._h, F2.ctypes.data_as(dptr), i64(F2.shape[0]), i64(F2.shape[1]),
                               1 if transpose else 0, out.ctypes.data_as(dptr), 1 if parallel else 0, threads))
        return out[:, 0] if vec else out

    def apply_transpose(self, g, **kw):
        return self.apply(g, transpose=True, **kw)

    def dense(self):
        return self.apply(np.eye(self.ncols, dtype=np.complex128))

    def save(self, path):
        _check(lib().orc_save(self._h, str(path).encode()))


def load(path):
    h = vp()
    _check(lib().orc_load(str(path).encode(), C.byref(h)))
    return Factorization(h)


def factorize(kernel, X, Omega, n0, k=30, eps=1e-9, t=5, seed=0, parallel=True):
    """make_trees(X, Omega, n0) + bf::idbf_factorize (tests/test_butterfly.cpp:52-60)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Omega = np.ascontiguousarray(Omega, dtype=np.float64)
    h = vp()
    _check(lib().orc_factorize(C.byref(kernel.desc), _p(X), i64(X.shape[0]), _p(Omega), i64(Omega.shape[0]),
                               X.shape[1], i64(n0), i64(k), C.c_double(eps), i64(t), u64(seed),
                               1 if parallel else 0, C.byref(h)))
    return Factorization(h)


def factorize_trees(kernel, X, Omega, n0x, mdx, n0o, mdo, k=30, eps=1e-9, t=5, seed=0):
    X = np.ascontiguousarray(X, dtype=np.float64)
    Omega = np.ascontiguousarray(Omega, dtype=np.float64)
    h = vp()
    _check(lib().orc_factorize_trees(C.byref(kernel.desc), _p(X), i64(X.shape[0]), _p(Omega), i64(Omega.shape[0]),
                                     X.shape[1], i64(n0x), mdx, i64(n0o), mdo, i64(k), C.c_double(eps), i64(t),
                                     u64(seed), C.byref(h)))
    return Factorization(h)


def random_coefficients(n, seed):
    out = np.empty(n, dtype=np.complex128)
    lib().orc_random_coefficients(i64(n), u64(seed), _p(out.view(np.float64)))
    return out


def grid2d(n):
    X = np.empty((n * n, 2), dtype=np.float64)
    lib().orc_grid2d(i64(n), _p(X))
    return X


def fio2d_phase(x, xi):
    x = np.ascontiguousarray(x, dtype=np.float64)
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    return lib().orc_fio2d_phase(_p(x), _p(xi))


def fio3d_phase(x, xi):
    x = np.ascontiguousarray(x, dtype=np.float64)
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    return lib().orc_fio3d_phase(_p(x), _p(xi))


# ---- linear-algebra pins
def pivoted_qr(A, max_rank=-1):
    A = np.asfortranarray(A)
    cplx = np.iscomplexobj(A)
    A = np.asfortranarray(A, dtype=np.complex128 if cplx else np.float64)
    m, n = A.shape
    r = min(m, n)
    dt = A.dtype
    perm = np.empty(n, dtype=np.int64)
    R = np.zeros((r, n), dtype=dt, order="F")
    Q = np.zeros((m, r), dtype=dt, order="F")
    rank = i64()
    _check(lib().orc_pqr(A.ctypes.data_as(dptr), i64(m), i64(n), 1 if cplx else 0, i64(max_rank), _ip(perm),
                         R.ctypes.data_as(dptr), Q.ctypes.data_as(dptr), C.byref(rank)))
    k = rank.value
    # the C side wrote rank-sized column-major arrays at the start of the buffers
    Rk = np.frombuffer(R.tobytes(order="F")[: k * n * dt.itemsize], dtype=dt).reshape((k, n), order="F")
    Qk = np.frombuffer(Q.tobytes(order="F")[: m * k * dt.itemsize], dtype=dt).reshape((m, k), order="F")
    return Qk, Rk, perm, k


def id_rank(d, k_max, eps):
    d = np.ascontiguousarray(d, dtype=np.float64)
    return int(lib().orc_id_rank(_p(d), i64(len(d)), i64(k_max), C.c_double(eps)))


def cid_from_rows(blk, k_max, eps):
    blk = np.asfortranarray(blk, dtype=np.complex128)
    m, n = blk.shape
    r = min(m, n)
    skel = np.empty(r, dtype=np.int64)
    V = np.zeros(r * n, dtype=np.complex128)
    rank = i64()
    _check(lib().orc_cid(blk.ctypes.data_as(dptr), i64(m), i64(n), i64(k_max), C.c_double(eps), _ip(skel),
                         _p(V.view(np.float64)), C.byref(rank)))
    k = rank.value
    return skel[:k].copy(), V[: k * n].reshape((k, n), order="F"), k


def rid_from_cols(blk, k_max, eps):
    blk = np.asfortranarray(blk, dtype=np.complex128)
    m, n = blk.shape
    r = min(m, n)
    skel = np.empty(r, dtype=np.int64)
    W = np.zeros(m * r, dtype=np.complex128)
    rank = i64()
    _check(lib().orc_rid(blk.ctypes.data_as(dptr), i64(m), i64(n), i64(k_max), C.c_double(eps), _ip(skel),
                         _p(W.view(np.float64)), C.byref(rank)))
    k = rank.value
    return skel[:k].copy(), W[: m * k].reshape((m, k), order="F"), k


def mock_chebyshev_rows(pts, s):
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    out = np.empty(max(len(pts), s), dtype=np.int64)
    n = lib().orc_mock_cheb_rows(_p(pts), i64(len(pts)), i64(s), _ip(out))
    return out[:n].copy()


def mock_chebyshev_points(P, s, seed):
    P = np.ascontiguousarray(P, dtype=np.float64)
    out = np.empty(max(P.shape[0], s), dtype=np.int64)
    n = lib().orc_mock_cheb_points(_p(P), i64(P.shape[0]), P.shape[1], i64(s), u64(seed), _ip(out))
    return out[:n].copy()


def rand_subset_seq(seed, draws):
    """[(n, k), ...] drawn in order from one std::mt19937_64(seed)."""
    ns = np.array([d[0] for d in draws], dtype=np.int64)
    ks = np.array([d[1] for d in draws], dtype=np.int64)
    out = np.empty(max(1, int(np.minimum(ns, ks).sum())), dtype=np.int64)
    lib().orc_rand_subset_seq(u64(seed), i64(len(draws)), _ip(ns), _ip(ks), _ip(out))
    res, off = [], 0
    for n, k in draws:
        c = min(n, k)
        res.append(out[off: off + c].copy())
        off += c
    return res


def rand_subset(n, k, seed):
    out = np.empty(max(n, 1), dtype=np.int64)
    m = lib().orc_rand_subset(i64(n), i64(k), u64(seed), _ip(out))
    return out[:m].copy()
