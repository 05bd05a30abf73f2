"""K5 — batched interpolative decompositions on the GPU
against the oracle's restated la::cid_from_rows (src/linalg.cpp:266-286,
pivoted QR :23-107, id_rank :249-264), and device-ID factorizations against
host-ID factorizations and the direct sum."""
import numpy as np
import pytest

import oracle as O
import paper_1908_09376_b200 as M
from helpers import cvec, rel

pytestmark = pytest.mark.gpu


def _decaying(rng, m, n, rate):
    """m x n complex block with singular values rate**i (well-separated
    pivots, so the device and host QR choose the same skeleton)."""
    r = min(m, n)
    U, _ = np.linalg.qr(rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r)))
    return (U * rate ** np.arange(r)) @ V.conj().T


@pytest.mark.parametrize("k_max,eps", [(30, 1e-9), (30, 0.0), (0, 1e-6), (8, 1e-12)])
def test_cid_batch_matches_oracle(gpu, k_max, eps):
    rng = np.random.default_rng(7)
    # up to 256 rows: k5_id<8>; 257..512 rows (3D blocks, cfg3 320 x 512): k5_id<16>
    shapes = [(150, 64), (150, 120), (40, 30), (7, 200), (256, 512), (1, 5), (64, 1),
              (320, 512), (512, 320), (300, 10)]
    blocks = [_decaying(rng, m, n, 0.55) for m, n in shapes]
    got = M.cid_batch(blocks, k_max, eps)
    for B, g in zip(blocks, got):
        sk, V, k = O.cid_from_rows(B, k_max, eps)
        assert g is not None
        gsk, gV, gk = g
        assert gk == k and np.array_equal(gsk, sk)
        # R11^-1 amplifies rounding by ~1/sigma_k = 0.55^-k (summation
        # orders differ between the warp reductions and the host loops)
        tol = max(1e-9, 1e-14 / 0.55 ** k)
        assert np.abs(gV - V).max() <= tol * max(1.0, np.abs(V).max())
        if k:  # the ID reproduces the block from its skeleton columns
            assert rel(B[:, gsk] @ gV, B) <= 10 * 0.55 ** k + 1e-12


def test_cid_batch_hands_back_what_it_cannot_finish(gpu):
    rng = np.random.default_rng(8)
    rank2 = rng.standard_normal((60, 2)) @ rng.standard_normal((2, 50)) + 0j  # tiny diagonals inside k_max
    big = rng.standard_normal((600, 10)) + 0j                                  # m > 512
    zero = np.zeros((20, 30), complex)
    out = M.cid_batch([rank2, big, zero, _decaying(rng, 30, 40, 0.5)], 10, 1e-9)
    assert out[0] is None and out[1] is None  # host fallback cases
    assert out[2][2] == 0                     # zero block: rank 0 (id_rank, src/linalg.cpp:251)
    assert out[3] is not None and out[3][2] == min(10, O.cid_from_rows(_decaying(np.random.default_rng(8), 30, 40, 0.5), 10, 1e-9)[2])


@pytest.mark.parametrize("n", [16, 32])
def test_device_id_factorization_matches_host_ids(gpu, n):
    X = O.grid2d(n)
    K = M.Kernel(M.KIND_FIO2D, X=X, Omega=X)
    Fd = M.idbf_factorize(K, 64, k=30, eps=1e-9, ids="device")
    Fh = M.idbf_factorize(K, 64, k=30, eps=1e-9, ids="host")
    ndev, nback, _, _ = Fd.id_stats()
    assert ndev > 0 and nback == 0
    assert Fd.total_nnz == Fh.total_nnz and Fd.nfactors == Fh.nfactors
    f = cvec(n * n, 3)
    assert rel(Fd.apply(f), Fh.apply(f)) <= 1e-10
    gd = K.direct_sum(f)
    assert rel(Fd.apply(f), gd) <= 1e-5  # tests/test_butterfly.cpp:202


def test_device_ids_saturate_for_integer_xi(gpu):
    from helpers import integer_grid
    X = O.grid2d(64)
    K = M.Kernel(M.KIND_FIO2D, X=X, Omega=integer_grid(64))
    F = M.idbf_factorize(K, 64, k=20, eps=1e-9, ids="device")
    assert F.total_nnz == 471040  # every ID at its cap
    assert F.id_stats()[1] == 0


def test_rank_one_kernel_falls_back_to_host_ids(gpu):
    """u v^T is rank one: every capped QR sees tiny diagonals, the device
    hands the blocks back, and the result equals the host-ID factorization."""
    rng = np.random.default_rng(5)
    X, Om = rng.random((400, 2)), rng.random((400, 2))
    u, v = cvec(400, 1), cvec(400, 2)
    K = M.Kernel(M.KIND_RANK1, X=X, Omega=Om, u=u, v=v)
    Fd = M.idbf_factorize(K, 32, k=6, eps=1e-9, ids="device")
    Fh = M.idbf_factorize(K, 32, k=6, eps=1e-9, ids="host")
    assert Fd.id_stats()[1] > 0
    f = cvec(400, 4)
    assert rel(Fd.apply(f), Fh.apply(f)) <= 1e-13
    assert rel(Fd.apply(f), u * (v @ f)) <= 1e-12  # tests/test_butterfly.cpp:86-90
