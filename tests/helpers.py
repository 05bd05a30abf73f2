"""Shared inputs for the parity tests (seeded, small enough for the oracle)."""
import os
import tempfile

import numpy as np

import oracle as O


def integer_grid(n, dim=2):
    """xi on the integer grid [-n/2, n/2)^dim (BASELINE.json configs)."""
    ax = np.arange(-n // 2, n // 2, dtype=np.float64)
    g = np.meshgrid(*([ax] * dim), indexing="ij")
    return np.stack(g, -1).reshape(-1, dim)


def unit_grid(n, dim=2):
    ax = np.arange(n, dtype=np.float64) / n
    g = np.meshgrid(*([ax] * dim), indexing="ij")
    return np.stack(g, -1).reshape(-1, dim)


def cvec(n, seed, cols=None):
    rng = np.random.default_rng(seed)
    shape = (n,) if cols is None else (n, cols)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    for side, v in (("result", a), ("expected", b)):
        bad = np.flatnonzero(~np.isfinite(v))
        if bad.size:  # name the side and the entries, not just a NaN norm
            raise AssertionError(f"{side} has {bad.size} non-finite entries of {v.size}, first {bad[:8].tolist()}")
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# (name, kind, X, Omega, n0, k, eps) cases covering the reference's test
# geometry: grids with xi = x, integer xi (BASELINE cfg0 shape), scattered
# points with odd depth, 3D x.xi, single leaf.
def cases():
    rng = np.random.default_rng(1234)
    out = []
    X16 = O.grid2d(16)
    out.append(("fio_n16", O.KIND_FIO2D, X16, X16, 64, 30, 1e-9))
    X32 = O.grid2d(32)
    out.append(("fio_n32", O.KIND_FIO2D, X32, X32, 64, 30, 1e-9))
    X64 = O.grid2d(64)
    out.append(("cfg0_intxi_n64", O.KIND_FIO2D, X64, integer_grid(64), 64, 20, 1e-9))
    Xr, Or = rng.random((1024, 2)), rng.random((1024, 2))
    out.append(("scattered_odd", O.KIND_FIO2D, Xr, Or, 16, 25, 1e-9))
    X3, O3 = rng.random((512, 3)), rng.random((512, 3))
    out.append(("nufft3d", O.KIND_NUFFT, X3, O3, 64, 40, 1e-9))
    Xs, Os = rng.random((50, 2)), rng.random((50, 2))
    out.append(("single_leaf", O.KIND_FIO2D, Xs, Os, 64, 30, 1e-9))
    Xg = unit_grid(8, 3)
    out.append(("fio3d_n8", O.KIND_FIO3D, Xg, integer_grid(8, 3), 64, 64, 1e-9))
    return out


def oracle_factorization(kind, X, Om, n0, k, eps, **kw):
    K = O.Kernel(kind, X=X, Omega=Om)
    return K, O.factorize(K, X, Om, n0, k=k, eps=eps, **kw)


def saved(F):
    fd, path = tempfile.mkstemp(suffix=".midbf")
    os.close(fd)
    F.save(path)
    return path
