"""Low-rank phase production on the host: la::thin_q,
la::pinv, la::rsvd against the reference's own pins
(tests/test_linalg.cpp:97-167) and against the numpy restatement in
oracle/lowrank.py (same index draws, same pivoted QR)."""
import numpy as np
import pytest

import lowrank as OL
import oracle as O
import paper_1908_09376_b200 as M


def _rank_k(rng, m, n, k, cplx=True):
    g = (lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)) if cplx else (lambda *s: rng.standard_normal(s))
    return g(m, k) @ g(k, n)


def test_thin_q_spans_the_input_columns():  # tests/test_linalg.cpp:97-104
    A = _rank_k(np.random.default_rng(14), 25, 8, 8)
    Q = M.thin_q(A)
    assert Q.shape == (25, 8)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(8)) <= 1e-12
    assert np.linalg.norm(Q @ (Q.conj().T @ A) - A) <= 1e-11 * np.linalg.norm(A)


def test_pinv_satisfies_the_moore_penrose_identities():  # :106-114
    A = _rank_k(np.random.default_rng(15), 12, 9, 4)
    P, cond = M.pinv(A)
    n = np.linalg.norm
    assert n(A @ P @ A - A) <= 1e-10 * n(A)
    assert n(P @ A @ P - P) <= 1e-10 * n(P)
    assert n((A @ P).conj().T - A @ P) <= 1e-10
    assert n((P @ A).conj().T - P @ A) <= 1e-10
    assert cond > 1e10  # rank 4 of 9: the thin SVD's smallest value is ~0
    Pn, _ = OL.pinv(A)
    assert n(P - Pn) <= 1e-10 * n(Pn)


def test_pinv_of_zero_is_zero():
    P, cond = M.pinv(np.zeros((3, 5)))
    assert P.shape == (5, 3) and not P.any() and np.isinf(cond)


def test_rsvd_of_all_ones_finds_the_exact_top_singular_value():  # :116-127
    A = np.ones((64, 64))
    R0, C0 = O.rand_subset_seq(7, [(64, 1), (64, 1)])
    U, S, V, _, _, _ = M.rsvd_dense(A, R0, C0, 1, 7)
    assert S.shape == (1,) and abs(S[0] - 64.0) <= 64.0 * 1e-12
    assert np.linalg.norm(U * S @ V.T - A) <= 1e-10 * np.linalg.norm(A)


def test_rsvd_recovers_an_exact_low_rank_matrix():  # :129-151
    m, n, r, q = 60, 50, 3, 2
    rng = np.random.default_rng(21)
    A = sum(np.outer(rng.standard_normal(m), rng.standard_normal(n)) for _ in range(r))
    R0, C0 = O.rand_subset_seq(21, [(m, q * r), (n, q * r)])
    U, S, V, rows, cols, ill = M.rsvd_dense(A, R0, C0, r, 21)
    assert np.linalg.norm(U * S @ V.T - A) <= 1e-9 * np.linalg.norm(A)
    assert not ill
    assert rows <= 3 * q * r and cols <= 2 * q * r  # bounded sampling


def test_rsvd_complex_uses_the_u_s_vh_convention():  # :153-167
    m, n, r, q = 40, 45, 5, 2
    A = _rank_k(np.random.default_rng(22), m, n, r)
    R0, C0 = O.rand_subset_seq(22, [(m, q * r), (n, q * r)])
    U, S, V, _, _, _ = M.rsvd_dense(A, R0, C0, r, 22)
    assert np.linalg.norm(U * S @ V.conj().T - A) <= 1e-9 * np.linalg.norm(A)


def test_rsvd_of_zero_is_empty():  # numerically zero slabs (src/linalg.cpp:168-174)
    R0, C0 = O.rand_subset_seq(3, [(30, 4), (20, 4)])
    U, S, V, _, _, _ = M.rsvd_dense(np.zeros((30, 20)), R0, C0, 2, 3)
    assert S.size == 0


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,n,r,q", [(80, 70, 4, 2), (120, 90, 8, 3), (50, 200, 6, 2)])
def test_rsvd_matches_the_oracle_restatement(cplx, m, n, r, q):
    """Same draws, same pivoted QR: same skeletons, singular values, product
    and sampling counts as the numpy restatement of rsvd_impl."""
    rng = np.random.default_rng(m + n + r)
    k = r + 3
    U0 = _rank_k(rng, m, k, k, cplx)
    V0 = _rank_k(rng, k, n, k, cplx)
    A = (U0 * 0.6 ** np.arange(k)) @ V0  # decaying spectrum past rank r
    seed = 1000 + m
    R0, C0 = O.rand_subset_seq(seed, [(m, q * r), (n, q * r)])
    U, S, V, rows, cols, ill = M.rsvd_dense(A, R0, C0, r, seed)
    Uo, So, Vo, rows_o, cols_o, ill_o = OL.rsvd_dense(A, R0, C0, r, seed)
    assert (rows, cols, ill) == (rows_o, cols_o, ill_o)
    assert np.allclose(S, So, rtol=1e-10, atol=0)
    P, Po = U * S @ V.conj().T, Uo * So @ Vo.conj().T
    assert np.linalg.norm(P - Po) <= 1e-10 * np.linalg.norm(Po)
