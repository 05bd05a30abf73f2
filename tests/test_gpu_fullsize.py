"""Parity at BASELINE.json's full sizes.

cfg1 / cfg3 are factorized on the device (K3 entries, host IDs), handed to
the oracle as MIDBF001, and the device apply (K1, K2) must match the
oracle's restated reference apply to rel-L2 <= 1e-12.  Size-independent
identities (adjoint, linearity) are checked on the device alone, and the
Omega = X companion is checked against the direct sum (K4)."""
import os
import tempfile

import numpy as np
import pytest

import oracle as O
import paper_1908_09376_b200 as M
from helpers import cvec, integer_grid, rel, unit_grid

pytestmark = pytest.mark.gpu


def _device_factorization(kind, X, Om, n0, k):
    K = M.Kernel(kind, X=X, Omega=Om)
    F = M.idbf_factorize(K, n0, k=k, eps=1e-9, t=5, seed=M.chain(0, 0x666163))
    return K, F


@pytest.fixture(scope="module")
def cfg1(gpu):
    X, Om = unit_grid(256, 2), integer_grid(256, 2)
    K, F = _device_factorization(M.KIND_FIO2D, X, Om, 64, 30)
    fd, path = tempfile.mkstemp(suffix=".midbf")
    os.close(fd)
    F.save(path)
    Fo = O.load(path)
    plan = M.DevicePlan.load(path, directions=3)
    os.unlink(path)
    return K, F, Fo, plan


def test_cfg1_structure_matches_appendix_b(cfg1):
    K, F, Fo, plan = cfg1
    assert (F.L, F.h, F.nfactors) == (5, 3, 7)
    assert F.total_nnz == 22364160  # every ID saturates at k for integer xi
    assert F.max_factor_nnz <= F.nnz_bound(4.0)
    entries, calls, _ = F.sample_stats()
    assert entries == 93388800 and calls == 7
    ndev, nback, _, _ = F.id_stats()
    assert ndev == 6144 and nback == 0  # every ID on the device (K5)


def test_cfg1_apply_matches_oracle(cfg1):
    K, F, Fo, plan = cfg1
    f = O.random_coefficients(65536, O.chain(0, 0x66))
    go = Fo.apply(f)
    assert rel(F.apply(f), go) <= 1e-12  # k1_flow through the C++ drop-in
    assert rel(plan.apply(f), go) <= 1e-12  # MIDBF001 -> device plan
    g = cvec(65536, 5)
    assert rel(plan.apply(g, transpose=True), Fo.apply_transpose(g)) <= 1e-12


def test_cfg4_multi_rhs_matches_oracle(cfg1):
    K, F, Fo, plan = cfg1
    X = cvec(65536, 6, cols=64)
    assert rel(plan.apply(X), Fo.apply(X)) <= 1e-12  # K2 (DMMA)


def test_cfg1_identities_on_device(cfg1):
    K, F, Fo, plan = cfg1
    f, g = cvec(65536, 7), cvec(65536, 8)
    lhs, rhs = plan.apply(f) @ g, f @ plan.apply(g, transpose=True)
    assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(f) * np.linalg.norm(g)
    a, b = 0.3 - 1.1j, -2.0 + 0.7j
    assert rel(plan.apply(a * f + b * g), a * plan.apply(f) + b * plan.apply(g)) <= 1e-12
    assert np.array_equal(plan.apply(f), plan.apply(f))


def test_cfg1_unit_xi_companion_accuracy(gpu, record_property):
    """Omega = X (the reference's convention, src/experiment.cpp:41-42): the
    factorization is accurate against the direct sum (K4) on 256 sampled
    rows, as metrics::eps_b does (src/metrics.cpp:26-48), at the paper's
    scale (4.12e-9 at n=256, k=30; its phase is the recovered
    one, ours the explicit phase).  The device-sampled factorization (K3 + K5)
    and the host-sampled one (the reference's EntryFn path, host IDs) pick
    different skeletons where pivots tie but must meet the same
    tolerance."""
    X = unit_grid(256, 2)
    K, F = _device_factorization(M.KIND_FIO2D, X, X.copy(), 64, 30)
    f = M.random_coefficients(65536, M.chain(0, 0x66))
    rows_seed = M.chain(0, 0x657062)
    eps_dev = K.eps_b(F.apply(f), f, nrows=256, seed=rows_seed)
    Fh = M.idbf_factorize(K, 64, k=30, eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="host")
    eps_host = K.eps_b(Fh.apply(f), f, nrows=256, seed=rows_seed)
    record_property("eps_b_device_sampled", eps_dev)
    record_property("eps_b_host_sampled", eps_host)
    print(f"cfg1_unitxi eps_b: device-sampled {eps_dev:.3e}, host-sampled {eps_host:.3e}")
    assert eps_dev <= 1e-7 and eps_host <= 1e-7
    assert max(eps_dev, eps_host) <= 10 * min(eps_dev, eps_host)
    assert F.total_nnz < 22364160  # adaptive ranks below k


@pytest.fixture(scope="module")
def cfg2(gpu):
    """BASELINE configs[2] exactly as bench.py builds it: n = 512, rank-8
    phase factors A, B (la::rsvd of the explicit phase, q = 2, V <- V S;
    src/phase_md.cpp:184-224, src/linalg.cpp:134-219) with entries only
    through them (metrics::phase_entry_fn, src/metrics.cpp:18-24), k = 30,
    9 factors, 1.73 GB; every entry sampled and every ID computed on the
    device."""
    import bench

    K, X, Om, fk, nrhs, desc = bench.workload("cfg2")
    F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163))
    fd, path = tempfile.mkstemp(suffix=".midbf")
    os.close(fd)
    F.save(path)
    Fo = O.load(path)
    plan = M.DevicePlan.load(path, directions=3)
    os.unlink(path)
    return K, F, Fo, plan


def test_cfg2_structure(cfg2):
    K, F, Fo, plan = cfg2
    assert (F.L, F.h, F.nfactors) == (6, 3, 9)
    assert F.total_nnz == Fo.total_nnz and F.max_factor_nnz <= F.nnz_bound(4.0)


def test_cfg2_apply_matches_oracle(cfg2):
    """Forward and transpose, three consecutive applies each (k1_flow
    alternates its two sentinel-armed stage-buffer sets between applies;
    cfg2 runs the 8-pair layout by size)."""
    K, F, Fo, plan = cfg2
    for s in (21, 22, 23):
        f = cvec(F.ncols, s)
        go = Fo.apply(f)
        assert rel(plan.apply(f), go) <= 1e-12
        g = cvec(F.nrows, s + 10)
        assert rel(plan.apply(g, transpose=True), Fo.apply_transpose(g)) <= 1e-12
    f = O.random_coefficients(F.ncols, O.chain(0, 0x66))
    assert rel(F.apply(f), Fo.apply(f)) <= 1e-12  # the C++ drop-in's cached plan


def test_cfg2_multi_rhs_matches_oracle(cfg2):
    K, F, Fo, plan = cfg2
    X = cvec(F.ncols, 24, cols=16)
    assert rel(plan.apply(X), Fo.apply(X)) <= 1e-12  # k2_flow (16-wide tiles)


def test_cfg3_apply_matches_oracle(gpu):
    X, Om = unit_grid(32, 3), integer_grid(32, 3)
    K, F = _device_factorization(M.KIND_FIO3D, X, Om, 64, 64)
    assert (F.L, F.nfactors) == (3, 5)
    fd, path = tempfile.mkstemp(suffix=".midbf")
    os.close(fd)
    F.save(path)
    Fo = O.load(path)
    os.unlink(path)
    f = cvec(32768, 9)
    assert rel(F.apply(f), Fo.apply(f)) <= 1e-12
    # consecutive applies alternate k1_flow's two sentinel-armed stage-buffer
    # sets (a single apply never re-arms); cfg3 runs the 8-pair variant
    for s in (10, 11, 12):
        f = cvec(32768, s)
        assert rel(F.apply(f), Fo.apply(f)) <= 1e-12
