"""Explicit-phase low_rank_phase_factorization (rows/columns of Phi sampled on
the GPU) and metrics::eps_K (entries on the GPU) against the numpy
restatement in oracle/lowrank.py."""
import numpy as np
import pytest

import lowrank as OL
import oracle as O
import paper_1908_09376_b200 as M
from helpers import integer_grid, unit_grid

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fio32(gpu):
    X, Om = unit_grid(32, 2), integer_grid(32, 2)
    return X, Om, M.Kernel(M.KIND_FIO2D, X=X, Omega=Om), O.Kernel(O.KIND_FIO2D, X=X, Omega=Om)


def test_lowrank_phase_matches_oracle(fio32):
    X, Om, K, Ko = fio32
    N = len(X)
    U, V, rows, cols = M.lowrank_phase(K, 8, 2, seed=11)
    Uo, Vo, rows_o, cols_o = OL.lowrank_phase(lambda i: OL.fio2d_phase_block(X, Om, [i], np.arange(N))[0],
                                              lambda j: OL.fio2d_phase_block(X, Om, np.arange(N), [j])[:, 0],
                                              N, N, 8, 2, 11)
    assert (rows, cols) == (rows_o, cols_o)
    assert U.shape == (N, 8) and V.shape == (N, 8)
    P, Po = U @ V.T, Uo @ Vo.T
    assert np.linalg.norm(P - Po) <= 1e-10 * np.linalg.norm(Po)
    # a rank-8 surrogate of the FIO phase: small but nonzero residual
    Phi = OL.fio2d_phase_block(X, Om, np.arange(N), np.arange(N))
    assert np.linalg.norm(P - Phi) <= 1e-2 * np.linalg.norm(Phi)


def test_eps_K_matches_oracle(fio32):
    X, Om, K, Ko = fio32
    U, V, _, _ = M.lowrank_phase(K, 8, 2, seed=11)
    e = M.eps_K(K, U, V, 128, 7)
    eo = OL.eps_K(Ko.entries, U, V, 128, 7)
    assert abs(e - eo) <= 1e-10 * eo


def test_eps_K_all_rows_and_columns(gpu):
    """nsamp >= n takes every row / column (src/metrics.cpp:64-67)."""
    X, Om = unit_grid(12, 2), integer_grid(12, 2)
    K, Ko = M.Kernel(M.KIND_FIO2D, X=X, Omega=Om), O.Kernel(O.KIND_FIO2D, X=X, Omega=Om)
    U, V, _, _ = M.lowrank_phase(K, 6, 2, seed=4)
    e = M.eps_K(K, U, V, 1000, 3)
    assert abs(e - OL.eps_K(Ko.entries, U, V, 1000, 3)) <= 1e-10 * e


def test_dot_product_phase_has_exact_rank_three(gpu):
    """x.xi in 3D is rank 3 (the reference's recovered phase needs 4: recovery
    adds a constant, tests/test_phase_md.cpp:285-299)."""
    rng = np.random.default_rng(201)
    X, Xi = rng.random((512, 3)), rng.random((512, 3)) * 4
    K = M.Kernel(M.KIND_NUFFT, X=X, Omega=Xi)
    U3, V3, _, _ = M.lowrank_phase(K, 3, 2, seed=11)
    U2, V2, _, _ = M.lowrank_phase(K, 2, 2, seed=11)
    assert M.eps_K(K, U3, V3, 128, 7) <= 1e-12
    assert M.eps_K(K, U2, V2, 128, 7) >= 1e-2


def test_zero_phase_factorizes_to_an_exactly_zero_product(gpu):  # tests/test_phase_md.cpp:270-282
    rng = np.random.default_rng(61)
    K = M.Kernel(M.KIND_LOWRANK, A=np.zeros((90, 1)), B=np.zeros((90, 1)))
    U, V, _, _ = M.lowrank_phase(K, 3, 2, seed=5)
    assert U.shape[1] == 0 or np.abs(U @ V.T).max() <= 1e-14
    del rng
