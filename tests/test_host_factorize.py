"""Host logic of the product (trees, IDs, sweeps, factor assembly, MIDBF001)
against the oracle, on the CPU.  With the same (host-evaluated) entries the
product's factorization must be BITWISE the oracle's: same perms, block
tables, groups and block payloads."""
import filecmp

import numpy as np
import pytest

import oracle as O
import paper_1908_09376_b200 as M
from helpers import integer_grid, unit_grid


def _cases():
    rng = np.random.default_rng(99)
    yield "fio_n16", O.KIND_FIO2D, O.grid2d(16), O.grid2d(16), 64, 30, 1e-9
    yield "fio_n32", O.KIND_FIO2D, O.grid2d(32), O.grid2d(32), 64, 30, 1e-9
    yield "cfg0_intxi", O.KIND_FIO2D, O.grid2d(64), integer_grid(64), 64, 20, 1e-9
    yield "scattered_odd", O.KIND_FIO2D, rng.random((1024, 2)), rng.random((1024, 2)), 16, 25, 1e-9
    yield "nufft3d", O.KIND_NUFFT, rng.random((512, 3)), rng.random((512, 3)), 64, 40, 1e-9
    yield "fio3d", O.KIND_FIO3D, unit_grid(8, 3), integer_grid(8, 3), 64, 64, 1e-9
    yield "single_leaf", O.KIND_FIO2D, rng.random((50, 2)), rng.random((50, 2)), 64, 30, 1e-9
    yield "loose_eps", O.KIND_FIO2D, O.grid2d(16), O.grid2d(16), 64, 30, 1e-5


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: c[0])
def test_product_factorization_is_bitwise_oracle(case):
    name, kind, X, Om, n0, k, eps = case
    Fo = O.factorize(O.Kernel(kind, X=X, Omega=Om), X, Om, n0, k=k, eps=eps, seed=3)
    Fm = M.idbf_factorize(M.Kernel(kind, X=X, Omega=Om), n0, k=k, eps=eps, seed=3, sampler="host")
    assert (Fo.L, Fo.h, Fo.nfactors, Fo.total_nnz, Fo.max_factor_nnz) == (Fm.L, Fm.h, Fm.nfactors, Fm.total_nnz,
                                                                          Fm.max_factor_nnz)
    for a, b in zip(Fo.perms(), Fm.perms()):
        assert np.array_equal(a, b)
    for i in range(Fo.nfactors):
        ro, co, bo, go = Fo.factor(i)
        rm, cm, bm, gm = Fm.factor(i)
        assert (ro, co) == (rm, cm) and np.array_equal(bo, bm) and np.array_equal(go, gm)
        for b in range(len(bo)):
            assert np.array_equal(Fo.block(i, b, bo[b, 2], bo[b, 3]), Fm.block(i, b))


def test_structure_pins_on_the_product():
    """tests/test_butterfly.cpp:197-200 on the product's host factorization."""
    for n, nf in ((16, 3), (32, 5)):
        X = O.grid2d(n)
        F = M.idbf_factorize(M.Kernel(M.KIND_FIO2D, X=X, Omega=X), 64, k=30, sampler="host")
        assert F.nfactors == 2 * (F.L - F.h + 1) + 1 == nf
        assert F.max_factor_nnz <= F.nnz_bound(4.0)


def test_integer_xi_saturates_every_id():
    """cfg0's shape has exactly 471040 nnz."""
    F = M.idbf_factorize(M.Kernel(M.KIND_FIO2D, X=O.grid2d(64), Omega=integer_grid(64)), 64, k=20, sampler="host")
    assert F.total_nnz == 471040 and F.nfactors == 5


def test_midbf001_interop_both_ways(tmp_path):
    X = O.grid2d(32)
    Fm = M.idbf_factorize(M.Kernel(M.KIND_FIO2D, X=X, Omega=X), 64, k=30, seed=7, sampler="host")
    Fo = O.factorize(O.Kernel(O.KIND_FIO2D, X=X, Omega=X), X, X, 64, k=30, seed=7, parallel=True)
    pm, po = tmp_path / "m.midbf", tmp_path / "o.midbf"
    Fm.save(pm)
    Fo.save(po)
    # identical factorization + identical container layout -> identical bytes
    # (the exec flag differs: product runs OpenMP by default as well)
    assert filecmp.cmp(pm, po, shallow=False)
    back = O.load(pm)
    assert back.total_nnz == Fm.total_nnz
    again = M.load_factorization(po)
    assert again.total_nnz == Fo.total_nnz and again.seed == 7
    raw = pm.read_bytes()
    (tmp_path / "bad").write_bytes(b"XIDBF001" + raw[8:])
    with pytest.raises(RuntimeError):
        M.load_factorization(tmp_path / "bad")
    (tmp_path / "short").write_bytes(raw[:-16])
    with pytest.raises(RuntimeError):
        M.load_factorization(tmp_path / "short")


def test_reference_generators_match():
    """random_coefficients (src/experiment.cpp:75-81) and chain
    (src/butterfly.cpp:20-27) agree between product and oracle."""
    assert M.chain(0, 0x66) == O.chain(0, 0x66)
    assert np.array_equal(M.random_coefficients(1000, 5), O.random_coefficients(1000, 5))
