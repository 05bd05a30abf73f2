"""K3 (fused entry sampler) and K4 (direct sum) on the GPU against the oracle,
and the device-sampled factorization against the direct sum."""
import numpy as np
import pytest

import oracle as O
import paper_1908_09376_b200 as M
from helpers import cvec, integer_grid, rel, unit_grid

pytestmark = pytest.mark.gpu


def _kernels():
    rng = np.random.default_rng(3)
    X64 = O.grid2d(64)
    yield "fio2d_intxi", O.KIND_FIO2D, dict(X=X64, Omega=integer_grid(64))
    yield "fio2d_unit", O.KIND_FIO2D, dict(X=X64, Omega=X64)
    yield "fio3d", O.KIND_FIO3D, dict(X=unit_grid(16, 3), Omega=integer_grid(16, 3))
    A, B = rng.standard_normal((4096, 8)), rng.standard_normal((4096, 8)) * 8
    yield "lowrank", O.KIND_LOWRANK, dict(A=A, B=B)
    yield "nufft", O.KIND_NUFFT, dict(X=rng.random((4096, 3)), Omega=rng.random((4096, 3)) * 16)
    u, v = cvec(4096, 1), cvec(4096, 2)
    yield "rank1", O.KIND_RANK1, dict(u=u, v=v)


@pytest.mark.parametrize("name,kind,kw", list(_kernels()), ids=lambda x: x if isinstance(x, str) else "")
def test_sampler_matches_oracle_entries(gpu, name, kind, kw):
    Ko, Km = O.Kernel(kind, **kw), M.Kernel(kind, **kw)
    rng = np.random.default_rng(9)
    rows = [rng.choice(Ko.nrows, size=s, replace=False) for s in (64, 7, 150)]
    cols = [rng.choice(Ko.ncols, size=s, replace=False) for s in (150, 64, 1)]
    blocks = Km.sample(rows, cols)
    for r, c, B in zip(rows, cols, blocks):
        rr, cc = np.meshgrid(r, c, indexing="ij")
        ref = Ko.entries(rr.ravel(), cc.ravel()).reshape(len(r), len(c))
        # Phi is evaluated with the reference's exact operation order; only
        # sincos may differ (CUDA vs glibc) by a few ulp.
        assert np.abs(B - ref).max() <= 4e-15, name


@pytest.mark.parametrize("name,kind,kw", list(_kernels()), ids=lambda x: x if isinstance(x, str) else "")
def test_direct_sum_matches_oracle(gpu, name, kind, kw):
    Ko, Km = O.Kernel(kind, **kw), M.Kernel(kind, **kw)
    f = cvec(Ko.ncols, 17)
    rows = np.random.default_rng(4).choice(Ko.nrows, 256, replace=False)
    assert rel(Km.direct_sum(f, rows), Ko.direct_sum(f, rows)) <= 1e-12


def test_direct_sum_all_rows(gpu):
    X = O.grid2d(32)
    Ko, Km = O.Kernel(O.KIND_FIO2D, X=X, Omega=X), M.Kernel(M.KIND_FIO2D, X=X, Omega=X)
    f = cvec(1024, 18)
    assert rel(Km.direct_sum(f), Ko.direct_sum(f)) <= 1e-12


@pytest.mark.parametrize("n", [16, 32])
def test_device_sampled_factorization_accuracy(gpu, n):
    """tests/test_butterfly.cpp:187-206 with every entry sampled on the GPU."""
    X = O.grid2d(n)
    Km = M.Kernel(M.KIND_FIO2D, X=X, Omega=X)
    F = M.idbf_factorize(Km, 64, k=30, eps=1e-9, sampler="device")
    assert F.nfactors == 2 * (F.L - F.h + 1) + 1
    assert F.nfactors == {16: 3, 32: 5}[n]
    assert F.max_factor_nnz <= F.nnz_bound(4.0)
    entries, calls, _ = F.sample_stats()
    assert entries > 0 and calls >= 3
    f = cvec(n * n, 41 + n)
    gd = Km.direct_sum(f)
    assert rel(F.apply(f), gd) <= 1e-5
    g = cvec(n * n, 43 + n)
    Ko = O.Kernel(O.KIND_FIO2D, X=X, Omega=X)
    assert rel(F.apply_transpose(g), Ko.dense().T @ g) <= 1e-5


def test_device_and_host_sampling_agree_on_integer_xi(gpu):
    """Every ID saturates for integer xi, so the
    device-sampled and host-sampled factorizations have the same structure and
    the same accuracy against the direct sum."""
    X, Om = O.grid2d(64), integer_grid(64)
    Km = M.Kernel(M.KIND_FIO2D, X=X, Omega=Om)
    Fd = M.idbf_factorize(Km, 64, k=20, eps=1e-9, sampler="device")
    Fh = M.idbf_factorize(Km, 64, k=20, eps=1e-9, sampler="host")
    assert Fd.total_nnz == Fh.total_nnz == 471040
    f = cvec(4096, 5)
    gd = Km.direct_sum(f)
    ed, eh = rel(Fd.apply(f), gd), rel(Fh.apply(f), gd)
    assert abs(ed - eh) <= 0.05 * eh


def test_sampler_splits_blocks_larger_than_a_chunk(gpu):
    """A 64 x 66000 block exceeds the sampler's 4M-entry chunk and is split
    into column ranges; every entry must still land in place."""
    rng = np.random.default_rng(8)
    A, B = rng.standard_normal((128, 4)), rng.standard_normal((70000, 4))
    Ko, Km = O.Kernel(O.KIND_LOWRANK, A=A, B=B), M.Kernel(M.KIND_LOWRANK, A=A, B=B)
    rows = rng.choice(128, 64, replace=False)
    cols = rng.choice(70000, 66000, replace=False)
    small_r, small_c = rng.choice(128, 5, replace=False), rng.choice(70000, 7, replace=False)
    big, small = Km.sample([rows, small_r], [cols, small_c])
    for r, c, Bk in ((rows, cols, big), (small_r, small_c, small)):
        rr, cc = np.meshgrid(r, c, indexing="ij")
        ref = Ko.entries(rr.ravel(), cc.ravel()).reshape(len(r), len(c))
        assert np.abs(Bk - ref).max() <= 4e-15


@pytest.mark.parametrize("name,kind,kw", list(_kernels())[:5], ids=lambda x: x if isinstance(x, str) else "")
def test_staged_and_generic_sampling_bitwise_equal(gpu, name, kind, kw):
    """Blocks with <= 512 rows go through the shared-memory staged sampler
    (operands per row / per column staged once, columns in 128-wide tiles);
    taller blocks through the generic one.  The staged operands are the
    reference's own intermediates, so both paths give the same bits."""
    Ko, Km = O.Kernel(kind, **kw), M.Kernel(kind, **kw)
    rng = np.random.default_rng(21)
    rows = rng.choice(Ko.nrows, 600, replace=False)
    cols = rng.choice(Ko.ncols, 300, replace=False)
    tall, top, bottom = Km.sample([rows, rows[:300], rows[300:]], [cols, cols, cols])
    assert np.array_equal(tall[:300], top) and np.array_equal(tall[300:], bottom)
    rr, cc = np.meshgrid(rows, cols, indexing="ij")
    ref = Ko.entries(rr.ravel(), cc.ravel()).reshape(len(rows), len(cols))
    assert np.abs(tall - ref).max() <= 4e-15


def test_lowrank_wider_than_staging(gpu):
    """Rank 12 > the staging width (8): the generic sampler and direct sum."""
    rng = np.random.default_rng(22)
    A, B = rng.standard_normal((2048, 12)), rng.standard_normal((2048, 12)) * 4
    Ko, Km = O.Kernel(O.KIND_LOWRANK, A=A, B=B), M.Kernel(M.KIND_LOWRANK, A=A, B=B)
    rows, cols = rng.choice(2048, 70, replace=False), rng.choice(2048, 90, replace=False)
    (Bk,) = Km.sample([rows], [cols])
    rr, cc = np.meshgrid(rows, cols, indexing="ij")
    assert np.abs(Bk - Ko.entries(rr.ravel(), cc.ravel()).reshape(70, 90)).max() <= 4e-15
    f = cvec(2048, 23)
    sel = rng.choice(2048, 300, replace=False)
    assert rel(Km.direct_sum(f, sel), Ko.direct_sum(f, sel)) <= 1e-12


def test_factorize_reports_kernel_times(gpu):
    X = O.grid2d(32)
    Km = M.Kernel(M.KIND_FIO2D, X=X, Omega=integer_grid(32))
    F = M.idbf_factorize(Km, 64, k=20, eps=1e-9, sampler="device")
    ks = F.kernel_stats()
    assert ks["k3_launches"] >= 3 and ks["k3_entries"] == F.sample_stats()[0]
    assert ks["k3_seconds"] > 0 and ks["k5_launches"] >= 1 and ks["k5_seconds"] > 0


def test_sincos_over_argument_ranges(gpu):
    """The sampler's lean sincos (Cody-Waite + fdlibm kernels, |2 pi Phi| <
    1e6) and its CUDA-sincos fallback beyond, against glibc: phases from
    1e-3 to 1e7, both signs, and near multiples of 1/4 (reduction edges)."""
    rng = np.random.default_rng(31)
    mags = np.concatenate([10.0 ** rng.uniform(-3, 7, 3000), rng.integers(-4000, 4000, 1000) / 4.0])
    X = np.ones((1, 1))
    Om = (mags * rng.choice([-1.0, 1.0], mags.size)).reshape(-1, 1)
    Om[-1000:, 0] += rng.uniform(-1e-12, 1e-12, 1000)
    Ko, Km = O.Kernel(O.KIND_NUFFT, X=X, Omega=Om), M.Kernel(M.KIND_NUFFT, X=X, Omega=Om)
    cols = np.arange(Om.shape[0])
    (Bk,) = Km.sample([np.array([0])], [cols])
    ref = Ko.entries(np.zeros_like(cols), cols)
    assert np.abs(Bk[0] - ref).max() <= 4e-15
