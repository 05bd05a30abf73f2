"""Pin the CPU oracle against the reference's own known-answer tests.

The reference ships no golden vectors and cannot be compiled here (SURVEY.md
section 8c), so the oracle is trusted only through the assertions of
proj/tests/test_linalg.cpp, test_tree.cpp, test_kernels.cpp and
test_butterfly.cpp, ported here line by line (cited per test)."""
import numpy as np
import pytest

import oracle as O
from helpers import cvec, rel

# ------------------------------------------------------------ linalg pins


def test_pivoted_qr_reconstructs_and_orders_diagonal():  # test_linalg.cpp:33-54
    rng = np.random.default_rng(11)
    A = rng.standard_normal((40, 25))
    Q, R, perm, rank = O.pivoted_qr(A)
    assert rank == 25
    assert np.linalg.norm(A[:, perm] - Q @ R) <= 1e-12 * np.linalg.norm(A)
    assert np.linalg.norm(Q.T @ Q - np.eye(25)) <= 1e-12
    d = np.diag(R)
    assert (d >= 0).all()
    assert all(d[i] <= d[i - 1] + 1e-10 * d[0] for i in range(1, 25))
    assert d[0] == pytest.approx(np.linalg.norm(A, axis=0).max(), rel=1e-12)


def test_pivoted_qr_diagonal_and_tie_orders():  # test_linalg.cpp:56-71
    A = np.diag([3.0, 7.0, 1.0, 5.0, 2.0])
    assert list(O.pivoted_qr(A)[2]) == [1, 3, 0, 4, 2]
    assert list(O.pivoted_qr(np.eye(3))[2]) == [0, 1, 2]


def _rank_k(m, n, k, rng):
    A = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
    B = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
    return A @ B


def test_pivoted_qr_max_rank_and_zero_tail():  # test_linalg.cpp:73-82
    K = _rank_k(30, 20, 4, np.random.default_rng(12))
    Q, R, perm, rank = O.pivoted_qr(K, 3)
    assert rank == 3 and Q.shape[1] == 3
    Q, R, perm, rank = O.pivoted_qr(K)
    for i in range(4, rank):
        assert abs(R[i, i]) <= 1e-10 * abs(R[0, 0])


def test_complex_qr_real_nonnegative_diagonal():  # test_linalg.cpp:84-95
    A = _rank_k(20, 15, 15, np.random.default_rng(13))
    Q, R, perm, rank = O.pivoted_qr(A)
    assert np.linalg.norm(A[:, perm] - Q @ R) <= 1e-11 * np.linalg.norm(A)
    for i in range(rank):
        assert abs(R[i, i].imag) <= 1e-14 and R[i, i].real >= 0


def test_id_rank_known_answers():  # test_linalg.cpp:169-178
    d = [1.0, 1e-2, 1e-4, 1e-9, 1e-16]
    assert O.id_rank(d, 10, 1e-3) == 3
    assert O.id_rank(d, 2, 1e-3) == 2
    assert O.id_rank(d, 10, 0.0) == 4
    assert O.id_rank(d, 3, 0.0) == 3
    assert O.id_rank([0.0] * 4, 4, 0.0) == 0


def test_column_id_exact_on_rank_deficient():  # test_linalg.cpp:180-200
    rng = np.random.default_rng(31)
    K = _rank_k(80, 40, 6, rng)
    rows = rng.choice(80, 18, replace=False)
    skel, V, k = O.cid_from_rows(K[rows], 6, 0.0)
    assert k == 6 and len(skel) == 6
    assert np.abs(V[:, skel] - np.eye(6)).max() <= 1e-12
    assert np.linalg.norm(K[:, skel] @ V - K) <= 1e-9 * np.linalg.norm(K)


def test_row_id_is_transpose_dual():  # test_linalg.cpp:202-224
    rng = np.random.default_rng(32)
    K = _rank_k(50, 70, 5, rng)
    cols = rng.choice(70, 15, replace=False)
    slab = K[:, cols]
    skel, W, k = O.rid_from_cols(slab, 5, 0.0)
    assert k == 5
    assert np.abs(W[skel, :] - np.eye(5)).max() <= 1e-12
    assert np.linalg.norm(W @ K[skel] - K) <= 1e-9 * np.linalg.norm(K)
    dskel, dV, _ = O.cid_from_rows(slab.T, 5, 0.0)
    assert list(dskel) == list(skel)
    assert np.linalg.norm(dV.T - W) <= 1e-14


def test_adaptive_id_truncates_noise():  # test_linalg.cpp:226-235
    rng = np.random.default_rng(33)
    K = _rank_k(30, 60, 4, rng)
    noise = _rank_k(30, 60, 30, rng)
    K = K + 1e-12 * (noise / np.linalg.norm(noise)) * np.linalg.norm(K)
    _, _, k = O.cid_from_rows(K, 20, 1e-8)
    assert 4 <= k <= 6


def test_mock_chebyshev_rows():  # test_linalg.cpp:237-250
    assert list(O.mock_chebyshev_rows(np.arange(10.0), 4)) == [0, 3, 6, 9]
    assert list(O.mock_chebyshev_rows([0.0, 1.0], 1)) == [0]
    assert list(O.mock_chebyshev_rows([0.0, 1.0], 5)) == [0, 1]


def test_mock_chebyshev_points_seeded_sorted_distinct():  # test_linalg.cpp:252-269
    P = np.random.default_rng(41).random((100, 2))
    a = O.mock_chebyshev_points(P, 17, 5)
    b = O.mock_chebyshev_points(P, 17, 5)
    assert list(a) == list(b) and len(a) == 17
    assert list(a) == sorted(set(a.tolist()))
    assert a.min() >= 0 and a.max() < 100


def test_mock_chebyshev_node_counts():  # c^d <= t*k
    P = np.random.default_rng(1).random((2000, 2))
    # k=20, t=5: 10x10 nodes, no top-up -> exactly 100 picks
    assert len(O.mock_chebyshev_points(P, 100, 0)) == 100
    P3 = np.random.default_rng(2).random((3000, 3))
    assert len(O.mock_chebyshev_points(P3, 320, 0)) == 320  # 6^3 = 216 nodes + 104 random


def test_rand_subset():  # test_linalg.cpp:271-281
    s = O.rand_subset(30, 12, 51)
    assert len(s) == 12 and len(set(s.tolist())) == 12
    assert s.min() >= 0 and s.max() < 30
    assert len(O.rand_subset(5, 9, 51)) == 5


# --------------------------------------------------------------- tree pins


def check_structure(T, X, n0):  # test_tree.cpp:25-73
    n = len(X)
    assert sorted(T.perm.tolist()) == list(range(n))
    assert len(T.levels) == T.depth + 1 and len(T.levels[0]["begin"]) == 1
    for lv in range(T.depth + 1):
        L = T.levels[lv]
        cursor = 0
        for i in range(len(L["begin"])):
            assert L["begin"][i] == cursor and L["end"][i] > L["begin"][i]
            cursor = L["end"][i]
            if i:
                assert L["code"][i] > L["code"][i - 1]
            if lv == T.depth:
                assert L["end"][i] - L["begin"][i] <= n0
            if lv:
                up = T.levels[lv - 1]
                p = L["parent"][i]
                assert up["code"][p] == L["code"][i] >> np.uint64(T.dim)
                assert up["begin"][p] <= L["begin"][i] and up["end"][p] >= L["end"][i]
                assert up["child"][p][int(L["code"][i]) & ((1 << T.dim) - 1)] == i
        assert cursor == n
        if lv < T.depth:
            D = T.levels[lv + 1]
            for i in range(len(L["begin"])):
                kids = [c for c in L["child"][i] if c >= 0]
                assert len(kids) == L["nchild"][i]
                assert sum(D["end"][c] - D["begin"][c] for c in kids) == L["end"][i] - L["begin"][i]


def test_tree_16x16_grid_one_split():  # test_tree.cpp:76-96
    X = O.grid2d(16)
    T = O.Tree(X, 64)
    assert T.depth == 1 and len(T.levels[1]["begin"]) == 4
    check_structure(T, X, 64)
    for q in range(4):
        L = T.levels[1]
        assert L["end"][q] - L["begin"][q] == 64 and L["code"][q] == q
        for p in range(L["begin"][q], L["end"][q]):
            o = T.perm[p]
            assert (X[o, 0] >= 0.5) == bool((q >> 1) & 1)
            assert (X[o, 1] >= 0.5) == bool(q & 1)


def test_tree_single_point_and_min_depth():  # test_tree.cpp:98-115
    T = O.Tree(np.array([[0.3, 0.7]]), 64)
    assert T.depth == 0 and T.levels[0]["end"][0] == 1 and T.perm[0] == 0
    T = O.Tree(O.grid2d(16), 64, 2)
    assert T.depth == 2 and len(T.levels[2]["begin"]) == 16
    assert all(e - b == 16 for b, e in zip(T.levels[2]["begin"], T.levels[2]["end"]))


def test_tree_prunes_empty_cells():  # test_tree.cpp:117-131
    X = np.random.default_rng(7).uniform(0, 0.24, (130, 2))
    X[0] = [0.9, 0.9]
    T = O.Tree(X, 64)
    assert T.depth >= 1 and len(T.levels[1]["begin"]) < 4
    check_structure(T, X, 64)


def test_tree_3d_octant_order():  # test_tree.cpp:133-155
    X = np.array([[0.25 + 0.5 * b1, 0.25 + 0.5 * b2, 0.25 + 0.5 * b3]
                  for b1 in (0, 1) for b2 in (0, 1) for b3 in (0, 1)])
    T = O.Tree(X, 1)
    assert T.depth == 1
    for q in range(8):
        assert T.levels[1]["code"][q] == q and T.perm[T.levels[1]["begin"][q]] == q


@pytest.mark.parametrize("dim", [2, 3])
def test_tree_random_invariants(dim):  # test_tree.cpp:157-168
    X = np.random.default_rng(11).random((500, dim))
    T = O.Tree(X, 32)
    assert T.depth >= 1
    check_structure(T, X, 32)


def test_tree_coincident_points_rejected():  # test_tree.cpp:170-175
    X = np.array([[0.5, 0.5], [0.5, 0.5], [0.9, 0.1]])
    with pytest.raises(ValueError):
        O.Tree(X, 1)
    O.Tree(X, 2)


# ------------------------------------------------------------- kernel pins


def test_fio2d_phase_known_values():  # test_kernels.cpp:27-37
    assert O.fio2d_phase([0, 0], [0, 0]) == pytest.approx(0.0)
    assert O.fio2d_phase([0, 0], [1, 0]) == pytest.approx(0.125, rel=1e-14)
    assert O.fio2d_phase([0.25, 0.25], [1, 0]) == pytest.approx(0.4375, rel=1e-13)
    assert O.fio2d_phase([0.25, 0.25], [0, 1]) == pytest.approx(0.375, rel=1e-13)


def test_fio3d_phase_reduces_to_formula():  # BASELINE.json configs[3]
    x, xi = np.array([0.25, 0.25, 0.25]), np.array([1.0, 0.0, 0.0])
    a1 = (2 + 1 * 1 * 1) / 16  # sin(pi/2)^3
    assert O.fio3d_phase(x, xi) == pytest.approx(0.25 + a1, rel=1e-13)


def test_grid2d_layout():  # test_kernels.cpp:67-75
    X = O.grid2d(4)
    assert X.shape == (16, 2) and X[0, 0] == 0.0
    assert X[7, 0] == pytest.approx(0.25) and X[7, 1] == pytest.approx(0.75)
    assert X[15, 0] == pytest.approx(0.75) and X.max() < 1.0


# ---------------------------------------------------------- butterfly pins


def _fio(X, Om):
    return O.Kernel(O.KIND_FIO2D, X=X, Omega=Om)


def test_constant_kernel():  # test_butterfly.cpp:68-91
    X = O.grid2d(8)
    K = O.Kernel(O.KIND_CONST, X=X, Omega=X, const=1.0)
    F = O.factorize(K, X, X, 16, k=1, eps=0.0)
    f = cvec(64, 11)
    assert rel(F.apply(f), K.direct_sum(f)) <= 1e-12
    _, _, blocks, _ = F.factor(0)  # U^1: four 16 x 1 blocks
    assert len(blocks) == 4 and (blocks[:, 2] == 16).all() and (blocks[:, 3] == 1).all()


def test_zero_kernel_exact():  # test_butterfly.cpp:93-109
    rng = np.random.default_rng(21)
    X, Om = rng.random((150, 2)), rng.random((150, 2))
    K = O.Kernel(O.KIND_CONST, X=X, Omega=Om, const=0j)
    F = O.factorize(K, X, Om, 32, k=5, eps=1e-9)
    assert np.abs(F.apply(cvec(150, 3))).max() == 0.0
    assert np.abs(F.apply_transpose(cvec(150, 4))).max() == 0.0


def test_rank_one_depth_three():  # test_butterfly.cpp:111-125
    rng = np.random.default_rng(31)
    X, Om = rng.random((1024, 2)), rng.random((1024, 2))
    K = O.Kernel(O.KIND_RANK1, u=cvec(1024, 33), v=cvec(1024, 34))
    F =O.factorize(K, X, Om, 16, k=6, eps=1e-12)
    assert F.L >= 3 and F.nfactors == 2 * (F.L - F.h + 1) + 1
    f = cvec(1024, 35)
    assert rel(F.apply(f), K.direct_sum(f)) <= 1e-10


@pytest.mark.parametrize("n", [16, 32])
def test_apply_matches_dense(n):  # test_butterfly.cpp:187-207
    X = O.grid2d(n)
    K = _fio(X, X)
    F = O.factorize(K, X, X, 64, k=30, eps=1e-9)
    assert F.nfactors == 2 * (F.L - F.h + 1) + 1 == {16: 3, 32: 5}[n]
    assert F.max_factor_nnz <= F.nnz_bound(4.0)
    f = cvec(n * n, 41 + n)
    assert rel(F.apply(f), K.direct_sum(f)) <= 1e-5
    g = cvec(n * n, 43 + n)
    assert rel(F.apply_transpose(g), K.dense().T @ g) <= 1e-5


def test_octree_3d():  # test_butterfly.cpp:209-226
    rng = np.random.default_rng(51)
    X, Om = rng.random((512, 3)), rng.random((512, 3))
    K = O.Kernel(O.KIND_NUFFT, X=X, Omega=Om)
    F = O.factorize(K, X, Om, 64, k=40, eps=1e-9)
    assert F.nfactors == 2 * (F.L - F.h + 1) + 1
    assert F.max_factor_nnz <= F.nnz_bound(16.0)
    f = cvec(512, 53)
    assert rel(F.apply(f), K.direct_sum(f)) <= 5e-6


def test_scattered_odd_depth():  # test_butterfly.cpp:228-241
    rng = np.random.default_rng(61)
    X, Om = rng.random((1024, 2)), rng.random((1024, 2))
    K = _fio(X, Om)
    F = O.factorize(K, X, Om, 16, k=25, eps=1e-9)
    assert F.L >= 3 and F.nfactors == 2 * (F.L - F.h + 1) + 1
    f = cvec(1024, 63)
    assert rel(F.apply(f), K.direct_sum(f)) <= 1e-4


def test_linearity_adjoint_mismatch():  # test_butterfly.cpp:243-273
    X = O.grid2d(16)
    F = O.factorize(_fio(X, X), X, X, 64, k=30, eps=1e-9)
    f1, f2 = cvec(256, 71), cvec(256, 72)
    a, b = 0.3 - 1.1j, -2.0 + 0.7j
    assert rel(F.apply(a * f1 + b * f2), a * F.apply(f1) + b * F.apply(f2)) <= 1e-12
    assert np.abs(F.apply(np.zeros(256, complex))).max() == 0.0
    with pytest.raises(ValueError):
        F.apply(np.zeros(257, complex))
    f, g = cvec(256, 81), cvec(256, 82)
    assert abs(F.apply(f) @ g - f @ F.apply_transpose(g)) <= 1e-10 * np.linalg.norm(f) * np.linalg.norm(g)


def test_parallel_is_bitwise_serial():  # test_butterfly.cpp:275-308
    X = O.grid2d(32)
    K = _fio(X, X)
    Fs = O.factorize(K, X, X, 64, k=25, eps=1e-9, parallel=False)
    Fp = O.factorize(K, X, X, 64, k=25, eps=1e-9, parallel=True)
    for i in range(Fs.nfactors):
        a, b = Fs.factor(i), Fp.factor(i)
        assert (a[2] == b[2]).all()
        for j, (m, n) in enumerate(a[2][:, 2:]):
            assert np.array_equal(Fs.block(i, j, m, n), Fp.block(i, j, m, n))
    f = cvec(1024, 91)
    assert np.array_equal(Fs.apply(f, parallel=False), Fp.apply(f, parallel=True))
    batch = np.sin(0.1 * np.add.outer(np.arange(1024), np.arange(3))) + 1j * np.cos(0.2 * np.arange(1024))[:, None]
    got = Fp.apply(batch)
    for c in range(3):
        assert np.abs(got[:, c] - Fp.apply(batch[:, c])).max() <= 1e-12


def test_complementary_low_rank():  # test_butterfly.cpp:310-335
    X = O.grid2d(64)
    K = _fio(X, X)
    T = O.Tree(X, 64)
    assert T.depth == 3
    rng = np.random.default_rng(101)
    for lv in (1, 2):
        rn, cn = T.levels[lv], T.levels[T.depth - lv]
        for _ in range(2):
            a = rng.integers(len(rn["begin"]))
            b = rng.integers(len(cn["begin"]))
            rows = T.perm[rn["begin"][a]:rn["end"][a]]
            cols = T.perm[cn["begin"][b]:cn["end"][b]]
            rr, cc = np.meshgrid(rows, cols, indexing="ij")
            blk = K.entries(rr.ravel(), cc.ravel()).reshape(len(rows), len(cols))
            s = np.linalg.svd(blk, compute_uv=False)
            assert (s > 1e-9 * s[0]).sum() <= 35


def test_looser_tolerance_shrinks():  # test_butterfly.cpp:337-352
    X = O.grid2d(16)
    K = _fio(X, X)
    Ft = O.factorize(K, X, X, 64, k=30, eps=1e-9)
    Fl = O.factorize(K, X, X, 64, k=30, eps=1e-5)
    assert Fl.total_nnz < Ft.total_nnz
    f = cvec(256, 111)
    gd = K.direct_sum(f)
    assert rel(Fl.apply(f), gd) <= 1e-3
    assert rel(Ft.apply(f), gd) < rel(Fl.apply(f), gd)


def test_depth_mismatch_rejected():  # test_butterfly.cpp:354-362
    X = O.grid2d(16)
    with pytest.raises(ValueError):
        O.factorize_trees(_fio(X, X), X, X, 64, 0, 16, 0)


def test_single_leaf_exact():  # test_butterfly.cpp:364-378
    rng = np.random.default_rng(121)
    X, Om = rng.random((50, 2)), rng.random((50, 2))
    K = _fio(X, Om)
    F = O.factorize(K, X, Om, 64)
    assert F.nfactors == 3
    f = cvec(50, 123)
    assert rel(F.apply(f), K.direct_sum(f)) <= 1e-13
    Kd = K.dense()
    assert np.linalg.norm(F.dense() - Kd) / np.linalg.norm(Kd) <= 1e-13


def test_midbf001_round_trip(tmp_path):  # butterfly_io.hpp:2-28
    X = O.grid2d(32)
    F = O.factorize(_fio(X, X), X, X, 64, k=30, eps=1e-9, seed=5)
    p = tmp_path / "f.midbf"
    F.save(p)
    G = O.load(p)
    assert (G.nrows, G.ncols, G.L, G.h, G.n0, G.k_max, G.t, G.seed) == (F.nrows, F.ncols, F.L, F.h, F.n0, F.k_max,
                                                                          F.t, F.seed)
    f = cvec(1024, 1)
    assert np.array_equal(G.apply(f), F.apply(f))
    raw = p.read_bytes()
    (tmp_path / "bad").write_bytes(b"MIDBF002" + raw[8:])
    with pytest.raises(RuntimeError):
        O.load(tmp_path / "bad")
    (tmp_path / "trunc").write_bytes(raw[:-8])
    with pytest.raises(RuntimeError):
        O.load(tmp_path / "trunc")
    (tmp_path / "trail").write_bytes(raw + b"\0")
    with pytest.raises(RuntimeError):
        O.load(tmp_path / "trail")
