"""B200-native MIDBF hot path: the butterfly apply (K1), the fused kernel-entry
sampler that feeds the interpolative decompositions (K3) and the direct-sum
oracle kernel (K4), all in hand-written sm_100a CUDA behind the C ABI of
``include/midbf_b200.h``.

This module is the Python mirror of the reference's C++ API
(``proj/include/midbf/butterfly.hpp``): ``idbf_factorize`` / ``apply`` /
``apply_transpose`` / ``save_factorization`` / ``load_factorization`` with the
same argument meaning and error classes (``ValueError`` for the reference's
``std::invalid_argument``, ``RuntimeError`` for ``std::runtime_error``).
The shared library ``libmidbf_b200.so`` is built in-tree by
``__graft_entry__.build()``; there is no CPU fallback — without it, or
without an sm_100 device, every device call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "KIND_FIO2D", "KIND_FIO3D", "KIND_LOWRANK", "KIND_NUFFT", "KIND_CONST", "KIND_RANK1",
    "Kernel", "Factorization", "DevicePlan", "idbf_factorize", "load_factorization", "save_factorization",
    "apply", "apply_transpose", "random_coefficients", "chain", "device_count", "lib", "MidbfCudaError",
    "LIB_PATH",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# MIDBF_LIB selects another build of the library (the checked build of
# tests/test_gpu_checked.py); default: the in-tree release build
LIB_PATH = os.environ.get("MIDBF_LIB") or os.path.join(_HERE, "libmidbf_b200.so")

KIND_FIO2D, KIND_FIO3D, KIND_LOWRANK, KIND_NUFFT, KIND_CONST, KIND_RANK1 = range(6)
MIDBF_OK, MIDBF_EINVAL, MIDBF_ELOGIC, MIDBF_ERUNTIME, MIDBF_ECUDA = 0, -1, -2, -3, -4

i64, u64, dptr, iptr, vp = C.c_int64, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_void_p


class MidbfCudaError(RuntimeError):
    """CUDA failure or no sm_100 device (MIDBF_ECUDA)."""


class _KernelDesc(C.Structure):  # midbf_kernel_desc
    _fields_ = [
        ("kind", C.c_int32), ("dim", C.c_int32), ("rank", C.c_int32),
        ("nrows", i64), ("ncols", i64),
        ("X", dptr), ("Omega", dptr), ("A", dptr), ("B", dptr),
        ("u", dptr), ("v", dptr), ("cre", C.c_double), ("cim", C.c_double),
    ]


_lib = None


def lib():
    """Load libmidbf_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_1908_09376_b200)")
        L = C.CDLL(LIB_PATH)
        L.midbf_last_error.restype = C.c_char_p
        L.midbf_chain.restype = u64
        L.midbf_chain.argtypes = [u64, u64]
        L.midbf_factorize.argtypes = [C.POINTER(vp), C.POINTER(_KernelDesc), i64, i64, C.c_double, i64, u64,
                                      C.c_int, C.c_int]
        L.midbf_apply.argtypes = [vp, vp, vp, i64, C.c_int, vp]
        L.midbf_apply_async.argtypes = [vp, vp, vp, i64, C.c_int, vp]
        L.midbf_fact_apply.argtypes = [vp, vp, vp, i64, C.c_int, vp]
        L.midbf_plan_set_flags.argtypes = [vp, C.c_uint]
        L.midbf_fact_plan.argtypes = [vp, C.c_uint, C.POINTER(vp)]
        L.midbf_plan_load.argtypes = [C.POINTER(vp), C.c_char_p, C.c_uint]
        L.midbf_plan_create.argtypes = [C.POINTER(vp), i64, i64, iptr, iptr, i64, iptr, iptr, iptr, dptr, C.c_uint]
        _lib = L
    return _lib


def _check(rc):
    if rc == MIDBF_OK:
        return
    msg = lib().midbf_last_error().decode()
    if rc == MIDBF_EINVAL:
        raise ValueError(msg)
    if rc == MIDBF_ELOGIC:
        raise AssertionError(msg)
    if rc == MIDBF_ECUDA:
        raise MidbfCudaError(msg)
    raise RuntimeError(msg)


def _p(a):
    return a.ctypes.data_as(dptr)


def _ip(a):
    return a.ctypes.data_as(iptr)


def chain(a, b):
    """Stream derivation of the reference (src/butterfly.cpp:20-27)."""
    return int(lib().midbf_chain(a, b))


def device_count():
    n = C.c_int()
    _check(lib().midbf_device_count(C.byref(n)))
    return n.value


def random_coefficients(n, seed):
    """Complex Gaussian f of the reference experiment (src/experiment.cpp:75-81)."""
    out = np.empty(n, dtype=np.complex128)
    _check(lib().midbf_random_coefficients(i64(n), u64(seed), _p(out.view(np.float64))))
    return out


class Kernel:
    """Typed kernel K(x, xi) = exp(2*pi*i*Phi) (midbf_kernel_desc).

    X, Omega: (N, dim) point sets (always required for factorization: they
    build the trees); A, B: real (N, r) low-rank phase factors; u, v / const:
    the reference's rank-one and constant test kernels.
    """

    def __init__(self, kind, X=None, Omega=None, A=None, B=None, u=None, v=None, const=0j):
        self._keep = []
        d = _KernelDesc()
        d.kind = kind
        nrows = ncols = 0
        if X is not None:
            X = np.ascontiguousarray(X, dtype=np.float64)
            Omega = np.ascontiguousarray(Omega, dtype=np.float64)
            self._keep += [X, Omega]
            d.X, d.Omega, d.dim = _p(X), _p(Omega), X.shape[1]
            nrows, ncols = X.shape[0], Omega.shape[0]
        if A is not None:
            A = np.ascontiguousarray(A, dtype=np.float64)
            B = np.ascontiguousarray(B, dtype=np.float64)
            self._keep += [A, B]
            d.A, d.B, d.rank = _p(A), _p(B), A.shape[1]
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
        self.kind, self.nrows, self.ncols = kind, nrows, ncols

    def sample(self, rows_list, cols_list):
        """K(rows_t, cols_t) for each task t in one fused GPU launch (K3)."""
        tasks, rid, cid, off = [], [], [], 0
        for r, c in zip(rows_list, cols_list):
            tasks.append((len(rid), len(r), len(cid), len(c), off))
            rid.extend(int(v) for v in r)
            cid.extend(int(v) for v in c)
            off += len(r) * len(c)
        T = np.ascontiguousarray(np.array(tasks, dtype=np.int64).reshape(-1, 5))
        R = np.ascontiguousarray(np.array(rid, dtype=np.int64))
        Cc = np.ascontiguousarray(np.array(cid, dtype=np.int64))
        out = np.empty(max(off, 1), dtype=np.complex128)
        _check(lib().midbf_sample(C.byref(self.desc), i64(len(tasks)), _ip(T), _ip(R), i64(len(R)), _ip(Cc),
                                  i64(len(Cc)), _p(out.view(np.float64)), i64(off)))
        blocks, at = [], 0
        for (_, nr, _, nc, _) in tasks:
            blocks.append(out[at:at + nr * nc].reshape((nr, nc), order="F"))
            at += nr * nc
        return blocks

    def direct_sum(self, f, rows=None):
        """g(rows) = sum_j K(rows, j) f(j) on the GPU (K4)."""
        f = np.ascontiguousarray(f, dtype=np.complex128)
        if rows is None:
            rp, n = None, self.nrows
        else:
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            rp, n = _ip(rows), len(rows)
        g = np.empty(n, dtype=np.complex128)
        _check(lib().midbf_direct_sum(C.byref(self.desc), _p(f.view(np.float64)), rp, i64(n), _p(g.view(np.float64))))
        return g

    @staticmethod
    def last_direct_sum_seconds():
        """Device seconds of this thread's last direct_sum (K4 + reduction)."""
        out = C.c_double()
        _check(lib().midbf_last_direct_sum_seconds(C.byref(out)))
        return out.value

    def eps_b(self, g_b, f, nrows=256, seed=0):
        """metrics::eps_b_of (src/metrics.cpp:26-48), direct sum on the GPU."""
        N = len(g_b)
        if nrows < 1:
            raise ValueError("eps_b: need at least one sampled row")
        if nrows >= N:
            S = np.arange(N, dtype=np.int64)
        else:
            S = _rand_subset(N, nrows, seed)
        gd = self.direct_sum(f, S)
        num = float(np.sum(np.abs(np.asarray(g_b)[S] - gd) ** 2))
        den = float(np.sum(np.abs(gd) ** 2))
        return float(np.sqrt(num)) if den == 0 else float(np.sqrt(num / den))


def _rand_subset(n, k, seed):
    # std::mt19937_64 + uniform_int_distribution partial Fisher-Yates
    # (src/linalg.cpp:390-400) is reproduced on the host side of the library.
    out = np.empty(k, dtype=np.int64)
    L = lib()
    L.midbf_rand_subset.restype = i64
    m = L.midbf_rand_subset(i64(n), i64(k), u64(seed), _ip(out))
    return out[:m]


class DevicePlan:
    """Device arena of one factorization (K1).  apply() takes host numpy
    arrays or device tensors (anything with data_ptr(); complex128)."""

    _apply_fn = None  # bound midbf_apply (apply_ptr)

    def __init__(self, handle, owner=None, owned=True):
        self._h = handle
        self._owner = owner
        self._owned = owned
        info = np.empty(8, dtype=np.int64)
        _check(lib().midbf_plan_info(handle, _ip(info)))
        (self.nrows, self.ncols, self.nfactors, self.total_nnz, self.arena_bytes, self.nstrips, self.directions,
         self.max_len) = (int(v) for v in info)
        self._flags0 = self.get_flags()

    @classmethod
    def load(cls, path, directions=1):
        h = vp()
        _check(lib().midbf_plan_load(C.byref(h), str(path).encode(), directions))
        return cls(h)

    @classmethod
    def from_tables(cls, nrows, ncols, row_perm, col_perm, factors, directions=1):
        """factors: list of (rows, cols, blocks[nb,4], groups[ng,2], [M_b ...]) in product order."""
        shape = np.array([[f[0], f[1], len(f[2]), len(f[3])] for f in factors], dtype=np.int64).reshape(-1, 4)
        blocks = np.ascontiguousarray(np.concatenate([np.asarray(f[2], np.int64).reshape(-1, 4) for f in factors]
                                                     + [np.zeros((0, 4), np.int64)]))
        groups = np.ascontiguousarray(np.concatenate([np.asarray(f[3], np.int64).reshape(-1, 2) for f in factors]
                                                     + [np.zeros((0, 2), np.int64)]))
        payload = np.concatenate([np.asarray(M, np.complex128).ravel(order="F") for f in factors for M in f[4]]
                                 + [np.zeros(1, np.complex128)])
        rp = np.ascontiguousarray(row_perm, dtype=np.int64)
        cp = np.ascontiguousarray(col_perm, dtype=np.int64)
        h = vp()
        _check(lib().midbf_plan_create(C.byref(h), nrows, ncols, _ip(rp), _ip(cp), len(factors), _ip(shape),
                                       _ip(blocks), _ip(groups), _p(payload.view(np.float64)), directions))
        return cls(h)

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None):
            try:
                lib().midbf_plan_destroy(self._h)
            except TypeError:  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    def set_flags(self, pdl=True, prefetch=True, graph=True, flow=True, dmma=True, dmma_flow=True, variant=3,
                  compress=True, lite=None, chain=True, coop=None, prologue=False, k2_mul4=False):
        """Kernel-path switches: persistent dataflow kernel (flow) for single
        RHS, else per-stage kernels chained with PDL (+ L2 prefetch); graphs;
        multi-RHS on the FP64 tensor cores (dmma), as one dataflow launch per
        64-RHS slice (dmma_flow) or one launch per stage.  variant: k1_flow
        layout 0 (4 warp pairs x 3 x 16 KB), 1 (8 x 2 x 8 KB), 3 chosen
        by the plan's size (default); 2 is retired and runs 1.  compress: k1_flow
        streams the identity-compressed panels (unit rows / columns of the ID
        blocks gathered from x instead).  lite: the dense-only k1_flow
        (True), the compressed one (False), or chosen by the plan's size
        (None, the default: dense-only below 200 MB of panels), so
        set_flags() alone restores a new plan's flags (0x3F | 1 << 17, the
        bench's default flags 131135).  chain: consecutive single-RHS applies
        on one stream launch as programmatic dependents (k1_flow streams its
        first panels while the previous apply drains; bit 17, default on).
        coop: the CTA-per-strip kernel k1_coop for single-RHS applies (True,
        bit 18), never (False, bit 19), or by size (None: small plans).
        prologue: k1_flow's 4-pair layout gathers the permuted input in a
        stage -1 prologue instead of in stage 0's x windows (bit 24).
        k2_mul4: k2_flow's 32- / 64-wide tiles multiply complex entries with
        four real DMMAs instead of Gauss's three (bit 26)."""
        f = (1 if pdl else 0) | (2 if prefetch else 0) | (4 if graph else 0) | (8 if flow else 0)
        f |= (0 if dmma else 2048) | (0 if dmma_flow else 8192) | ((variant & 3) << 4) | (0 if compress else 512)
        if chain:
            f |= 1 << 17
        if coop is True:
            f |= 1 << 18
        elif coop is False:
            f |= 1 << 19
        if prologue:
            f |= 1 << 24
        if k2_mul4:
            f |= 1 << 26
        if lite is True:
            f |= 1024
        elif lite is False and compress:
            f |= 65536
        _check(lib().midbf_plan_set_flags(self._h, f))

    def get_flags(self):
        out = C.c_uint()
        _check(lib().midbf_plan_get_flags(self._h, C.byref(out)))
        return out.value

    def reset_flags(self):
        """Restore the flags the plan was created with."""
        _check(lib().midbf_plan_set_flags(self._h, self._flags0))

    def launches(self, nrhs=1, transpose=False):
        """Kernel launches one apply issues."""
        out = i64()
        _check(lib().midbf_plan_launches(self._h, 1 if transpose else 0, i64(nrhs), C.byref(out)))
        return out.value

    def stages(self, transpose=False):
        out = np.zeros((64, 4), dtype=np.int64)
        _check(lib().midbf_plan_stages(self._h, 1 if transpose else 0, _ip(out), i64(64)))
        return [tuple(int(v) for v in r) for r in out if r[2] or r[3]]

    def flow_bytes(self, transpose=False):
        """Panel bytes k1_flow streams per stage (application order)."""
        n = len(self.stages(transpose))
        out = np.zeros(max(n, 1), dtype=np.int64)
        _check(lib().midbf_plan_flow_bytes(self._h, 1 if transpose else 0, _ip(out), i64(n)))
        return [int(v) for v in out[:n]]

    def k2_bytes(self, transpose=False):
        """Panel bytes the multi-RHS DMMA kernel multiplies per apply (32/64-wide tiles)."""
        out = i64()
        _check(lib().midbf_plan_k2_bytes(self._h, 1 if transpose else 0, C.byref(out)))
        return out.value

    def apply_ptr(self, f_ptr, g_ptr, nrhs=1, transpose=False, stream=0):
        """Raw-pointer apply (device or host pointers, cudaStream_t as int).
        The hot loop of a Python caller: the bound C function is cached and
        the ints go straight through its argtypes."""
        fn = self._apply_fn
        if fn is None:
            fn = self._apply_fn = lib().midbf_apply
        rc = fn(self._h, f_ptr, g_ptr, nrhs, 1 if transpose else 0, stream)
        if rc:
            _check(rc)

    def apply_async_ptr(self, f_ptr, g_ptr, nrhs=1, transpose=False, stream=0):
        """Pipelined host-operand apply (midbf_apply_async): returns after
        enqueueing; synchronize `stream` before reading g / reusing f."""
        _check(lib().midbf_apply_async(self._h, vp(f_ptr), vp(g_ptr), nrhs, 1 if transpose else 0, vp(stream)))

    def apply(self, f, transpose=False, out=None, stream=0):
        nout = self.ncols if transpose else self.nrows
        nin = self.nrows if transpose else self.ncols
        if hasattr(f, "data_ptr"):  # device tensor: (n,) or (n, nrhs), complex128 on a CUDA device
            import torch

            if f.dtype != torch.complex128:
                raise TypeError(f"apply: device operand must be complex128, got {f.dtype}")
            if not f.is_cuda:
                raise TypeError("apply: tensors must live on a CUDA device (host data: pass a numpy array)")
            if f.dim() not in (1, 2):
                raise ValueError("apply: operand must be a vector or an n x nrhs matrix")
            if f.shape[0] != nin:
                raise ValueError("input length does not match the factorization")  # src/butterfly.cpp:645
            nrhs = 1 if f.dim() == 1 else f.shape[1]
            # the ABI reads and writes column-major n x nrhs
            fc = f if f.dim() == 1 else f.t().contiguous().t()
            if fc.dim() == 1:
                fc = fc.contiguous()
            shape = (nout,) if f.dim() == 1 else (nout, nrhs)
            if out is None:
                out = torch.empty(shape[::-1], dtype=torch.complex128, device=f.device).t() if f.dim() == 2 \
                    else torch.empty(nout, dtype=torch.complex128, device=f.device)
            if out.dtype != torch.complex128 or not out.is_cuda or tuple(out.shape) != shape:
                raise ValueError(f"apply: out must be a complex128 CUDA tensor of shape {shape}")
            colmajor = out.dim() == 1 and out.is_contiguous() or (
                out.dim() == 2 and out.stride(0) == 1 and (out.stride(1) == nout or nrhs == 1))
            dst = out if colmajor else torch.empty(shape[::-1], dtype=torch.complex128, device=f.device).t()
            if dst.dim() == 1 and dst.stride(0) != 1:
                dst = torch.empty(nout, dtype=torch.complex128, device=f.device)
            self.apply_ptr(fc.data_ptr(), dst.data_ptr(), nrhs, transpose, stream)
            if dst is not out:
                out.copy_(dst)
            return out
        f = np.asarray(f, dtype=np.complex128)
        vec = f.ndim == 1
        F2 = np.asfortranarray(f.reshape(f.shape[0], -1))
        if F2.shape[0] != nin:
            raise ValueError("input length does not match the factorization")
        g = np.empty((nout, F2.shape[1]), dtype=np.complex128, order="F")
        self.apply_ptr(F2.ctypes.data, g.ctypes.data, F2.shape[1], transpose)
        return g[:, 0] if vec else g


class Factorization:
    """Host bf::Factorization (include/midbf/butterfly.hpp:53-70) whose
    apply runs on the GPU through a cached device plan."""

    def __init__(self, handle):
        self._h = handle
        info = np.empty(12, dtype=np.int64)
        eps = C.c_double()
        _check(lib().midbf_fact_info(handle, _ip(info), C.byref(eps)))
        (self.nrows, self.ncols, self.L, self.h, self.n0, self.nfactors, self.total_nnz, self.max_factor_nnz,
         self.k_max, self.t, self.seed, self.exec) = (int(v) for v in info)
        self.eps = eps.value

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().midbf_fact_destroy(self._h)
            except TypeError:  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    def factor_count(self):
        return self.nfactors

    def nnz_bound(self, c=4.0):
        return c * self.k_max * self.k_max / max(self.n0, 1) * max(self.nrows, self.ncols)

    def sample_stats(self):
        """(entries sampled on the GPU, sampler calls, seconds in the sampler)."""
        o = np.zeros(3, dtype=np.int64)
        _check(lib().midbf_fact_stats(self._h, _ip(o)))
        return int(o[0]), int(o[1]), o[2] * 1e-9

    def id_stats(self):
        """(IDs on the GPU, IDs handed back to the host, seconds in the device
        ID batches, seconds for the whole factorize)."""
        o = np.zeros(4, dtype=np.int64)
        _check(lib().midbf_fact_id_stats(self._h, _ip(o)))
        return int(o[0]), int(o[1]), o[2] * 1e-9, o[3] * 1e-9

    def kernel_stats(self):
        """Device time of the factorize's kernels (CUDA events): dict with
        K3 launches / entries / seconds and K5 launches / seconds."""
        o = np.zeros(5, dtype=np.int64)
        _check(lib().midbf_fact_kernel_stats(self._h, _ip(o)))
        return {"k3_launches": int(o[0]), "k3_entries": int(o[1]), "k3_seconds": o[2] * 1e-9,
                "k5_launches": int(o[3]), "k5_seconds": o[4] * 1e-9}

    def perms(self):
        rp = np.empty(self.nrows, dtype=np.int64)
        cp = np.empty(self.ncols, dtype=np.int64)
        _check(lib().midbf_fact_perms(self._h, _ip(rp), _ip(cp)))
        return rp, cp

    def factor(self, i):
        o = np.empty(4, dtype=np.int64)
        _check(lib().midbf_fact_factor(self._h, i64(i), _ip(o)))
        rows, cols, nb, ng = (int(v) for v in o)
        blocks = np.empty((nb, 4), dtype=np.int64)
        groups = np.empty((ng, 2), dtype=np.int64)
        _check(lib().midbf_fact_tables(self._h, i64(i), _ip(blocks), _ip(groups)))
        return rows, cols, blocks, groups

    def block(self, i, b):
        _, _, blocks, _ = self.factor(i)
        m, n = int(blocks[b, 2]), int(blocks[b, 3])
        out = np.empty((m, n), dtype=np.complex128, order="F")
        _check(lib().midbf_fact_block(self._h, i64(i), i64(b), out.ctypes.data_as(dptr)))
        return out

    def plan(self, directions=1):
        h = vp()
        _check(lib().midbf_fact_plan(self._h, directions, C.byref(h)))
        return DevicePlan(h, owner=self, owned=False)

    def apply(self, f, transpose=False):
        f = np.asarray(f, dtype=np.complex128)
        vec = f.ndim == 1
        F2 = np.asfortranarray(f.reshape(f.shape[0], -1))
        nin = self.nrows if transpose else self.ncols
        if F2.shape[0] != nin:
            raise ValueError("input length does not match the factorization")
        g = np.empty((self.ncols if transpose else self.nrows, F2.shape[1]), dtype=np.complex128, order="F")
        _check(lib().midbf_fact_apply(self._h, F2.ctypes.data, g.ctypes.data, F2.shape[1], 1 if transpose else 0,
                                      None))
        return g[:, 0] if vec else g

    def apply_transpose(self, g):
        return self.apply(g, transpose=True)

    def dense(self):
        return self.apply(np.eye(self.ncols, dtype=np.complex128))

    def save(self, path):
        _check(lib().midbf_fact_save(self._h, str(path).encode()))


def cid_batch(blocks, k_max, eps):
    """Column IDs of complex blocks on the GPU (K5, midbf_cid_batch).  Returns
    per block (skeleton, V, rank), or None where the device hands the block
    back (rank -1: the caller recomputes it with the host ID)."""
    blocks = [np.asfortranarray(b, dtype=np.complex128) for b in blocks]
    if not blocks:
        return []
    dims = np.array([b.shape for b in blocks], dtype=np.int64).reshape(-1)
    caps = [min(b.shape[0], b.shape[1], k_max if k_max > 0 else 1 << 62) for b in blocks]
    kcap = max(caps)
    packed = np.concatenate([b.reshape(-1, order="F") for b in blocks])
    ranks = np.empty(len(blocks), dtype=np.int64)
    skel = np.empty(len(blocks) * kcap, dtype=np.int64)
    vals = np.zeros(sum(c * b.shape[1] for c, b in zip(caps, blocks)), dtype=np.complex128)
    _check(lib().midbf_cid_batch(_p(packed.view(np.float64)), _ip(dims), i64(len(blocks)), i64(k_max),
                                 C.c_double(eps), _ip(ranks), _ip(skel), i64(kcap), _p(vals.view(np.float64))))
    out, off = [], 0
    for q, (c, b) in enumerate(zip(caps, blocks)):
        k, n = int(ranks[q]), b.shape[1]
        out.append(None if k < 0 else (skel[q * kcap: q * kcap + k].copy(),
                                       vals[off: off + k * n].reshape((k, n), order="F").copy(), k))
        off += c * n
    return out


# ---- low-rank phase production (csrc/host/lowrank.cpp)
def _dense(A):
    """Column-major flat copy (float64 view) of a real or complex matrix."""
    cplx = np.iscomplexobj(A)
    A = np.asarray(A, dtype=np.complex128 if cplx else np.float64)
    flat = np.ascontiguousarray(A.reshape(-1, order="F"))
    return flat.view(np.float64), A.shape, A.dtype, cplx


def _out(shape, dtype):
    return np.zeros(int(np.prod(shape)), dtype=dtype)


def _shaped(buf, shape):
    return buf.reshape(shape, order="F")


def thin_q(A):
    """la::thin_q: orthonormal basis of range(A), m x min(m, n)."""
    a, (m, n), dt, cplx = _dense(A)
    Q = _out((m, min(m, n)), dt)
    _check(lib().midbf_thin_q(_p(a), i64(m), i64(n), 1 if cplx else 0, _p(Q.view(np.float64))))
    return _shaped(Q, (m, min(m, n)))


def pinv(A, rel_cutoff=1e-12):
    """la::pinv -> (pseudoinverse, sigma_max / sigma_min)."""
    a, (m, n), dt, cplx = _dense(A)
    P = _out((n, m), dt)
    cond = C.c_double()
    _check(lib().midbf_pinv(_p(a), i64(m), i64(n), 1 if cplx else 0, C.c_double(rel_cutoff),
                            _p(P.view(np.float64)), C.byref(cond)))
    return _shaped(P, (n, m)), cond.value


def rsvd_dense(A, R0, C0, r, seed):
    """la::rsvd on a dense matrix (std::mt19937_64(seed) draws the enlarged
    index sets) -> U, S, V, rows_evaluated, cols_evaluated, ill_conditioned."""
    a, (m, n), dt, cplx = _dense(A)
    R0 = np.ascontiguousarray(R0, dtype=np.int64)
    C0 = np.ascontiguousarray(C0, dtype=np.int64)
    if R0.shape != C0.shape or R0.ndim != 1:  # one count crosses the ABI (src/linalg.cpp:142, equal sizes)
        raise ValueError("rsvd: row and column samples differ in size")
    U, V, S = _out((m, r), dt), _out((n, r), dt), np.zeros(r)
    info = np.zeros(4, dtype=np.int64)
    _check(lib().midbf_rsvd_dense(_p(a), i64(m), i64(n), 1 if cplx else 0, _ip(R0), _ip(C0), i64(len(R0)), i64(r),
                                  u64(seed), _p(U.view(np.float64)), _p(S), _p(V.view(np.float64)), _ip(info)))
    k = int(info[0])
    return _shaped(U, (m, r))[:, :k], S[:k], _shaped(V, (n, r))[:, :k], int(info[1]), int(info[2]), bool(info[3])


def lowrank_phase(kernel, r, q=2, seed=0):
    """phase::low_rank_phase_factorization of the kernel's closed-form phase
    (rows / columns of Phi on the GPU) -> U (nrows x k), V (ncols x k, scaled
    by S), rows_evaluated, cols_evaluated."""
    U, V = np.zeros(kernel.nrows * r), np.zeros(kernel.ncols * r)
    info = np.zeros(3, dtype=np.int64)
    _check(lib().midbf_lowrank_phase(C.byref(kernel.desc), i64(r), i64(q), u64(seed), _p(U), _p(V), _ip(info)))
    k = int(info[0])
    return (_shaped(U, (kernel.nrows, r))[:, :k], _shaped(V, (kernel.ncols, r))[:, :k], int(info[1]),
            int(info[2]))


def eps_K(kernel, U, V, nsamp=256, seed=0):
    """metrics::eps_K of a low-rank phase U V^T against the kernel (GPU entries)."""
    U = np.asarray(U, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    r = U.shape[1] if U.ndim == 2 else -1
    if U.shape != (kernel.nrows, r) or V.shape != (kernel.ncols, r):
        raise ValueError("eps_K: U must be nrows x r and V ncols x r")
    u, _, _, _ = _dense(U)
    v, _, _, _ = _dense(V)
    out = C.c_double()
    _check(lib().midbf_eps_K(C.byref(kernel.desc), _p(u), _p(v), i64(r), i64(nsamp), u64(seed), C.byref(out)))
    return out.value


def idbf_factorize(kernel, n0, k=30, eps=1e-9, t=5, seed=0, parallel=True, sampler="device", ids="device"):
    """bf::idbf_factorize on trees built at a common depth from the kernel's
    point sets.  sampler="device": every entry from the GPU sampler (K3);
    "host": the same descriptor evaluated on the CPU (reference EntryFn path).
    ids="device" (with the device sampler): the interpolative decompositions
    run on the GPU too (K5); "host": la::rid_from_cols / cid_from_rows on the
    CPU, bitwise the oracle's arithmetic."""
    if sampler not in ("device", "host") or ids not in ("device", "host"):
        raise ValueError("sampler and ids are 'device' or 'host'")
    mode = 1 if sampler == "host" else (2 if ids == "device" else 0)
    h = vp()
    _check(lib().midbf_factorize(C.byref(h), C.byref(kernel.desc), n0, k, eps, t, seed, 1 if parallel else 0, mode))
    return Factorization(h)


def load_factorization(path):
    h = vp()
    _check(lib().midbf_fact_load(C.byref(h), str(path).encode()))
    return Factorization(h)


def save_factorization(path, F):
    F.save(path)


def apply(F, f):
    return F.apply(f)


def apply_transpose(F, g):
    return F.apply(g, transpose=True)
